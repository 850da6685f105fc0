# fused CholeskyQR pass: kernel tests, QR tests, parity subset, A/B bench, trace
mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 600 -k "cholqr or qr or chol" > gpurun_out/s3b_kern.log 2>&1; echo "kern rc=$?"; tail -5 gpurun_out/s3b_kern.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -k "not full_size" > gpurun_out/s3b_par.log 2>&1; echo "parity rc=$?"; tail -5 gpurun_out/s3b_par.log
for V in 0 1; do
  if [ $V = 1 ]; then export TTR_NO_CQR=1; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/s3b_bench_$V.json 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/s3b_bench_$V.json'));print('nocqr=$V', round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phase_ms'].items()}, round(d['roofline']['frac'],4))"
done
unset TTR_NO_CQR
TTR_TRACE=gpurun_out/s3b_trace_large.txt timeout 600 python tools/run_once.py large - 2 > /dev/null 2>&1; echo "trace rc=$?"
awk '/^# trace/{n++} n==2' gpurun_out/s3b_trace_large.txt | head -30
for W in single sum10 gmres; do
  timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/s3b_bench_$W.json 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/s3b_bench_$W.json'));print('$W', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phase_ms'].items()})"
done
