mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 600 -k "chol or qr" > gpurun_out/s3q_kern.log 2>&1; echo "kern rc=$?"; tail -2 gpurun_out/s3q_kern.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/s3q_bench.json 2>&1
python -c "
import json;d=json.load(open('gpurun_out/s3q_bench.json'));print(round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phase_ms'].items()})"
for W in single sum10; do
  timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/s3q_bench_$W.json 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/s3q_bench_$W.json'));print('$W', round(d['ms_per_step'],3), {k:round(x,3) for k,x in d['phase_ms'].items()})"
done
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -k "not full_size" > gpurun_out/s3q_par.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/s3q_par.log
timeout 900 python bench.py --workload large --batch 2 --streams 2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/s3q_bench_large_b2s2.json 2>&1; echo "conc rc=$?"; cut -c1-300 gpurun_out/s3q_bench_large_b2s2.json
