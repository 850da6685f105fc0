mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 600 -k "jacobi or svd" > gpurun_out/s3r_kern.log 2>&1; echo "kern rc=$?"; tail -2 gpurun_out/s3r_kern.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -k "deterministic" > gpurun_out/s3r_det.log 2>&1; echo "det parity rc=$?"; tail -2 gpurun_out/s3r_det.log
timeout 1200 python bench.py --algo deterministic --workload sum10 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/s3r_bench_det_sum10.json 2>&1; echo "det sum10 rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/s3r_bench_det_sum10.json').read().strip().splitlines()[-1]);print('det sum10', round(d['ms_per_step'],1), {k:round(v,1) for k,v in d['phase_ms'].items()})"
