# fused CholeskyQR pass: A/B in the pipeline + parity subset
mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
for V in 0 1; do
  if [ $V = 1 ]; then export TTR_NO_CQR=1; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/s3l_bench_$V.json 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/s3l_bench_$V.json'));print('nocqr=$V', round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phase_ms'].items()}, round(d['roofline']['frac'],4))"
  for W in single sum10; do
    timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/s3l_bench_${W}_$V.json 2>&1
    python -c "
import json;d=json.load(open('gpurun_out/s3l_bench_${W}_$V.json'));print('$W nocqr=$V', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phase_ms'].items()})"
  done
done
unset TTR_NO_CQR
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -k "not full_size" > gpurun_out/s3l_par.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/s3l_par.log
