mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 600 -k "jacobi or svd" > gpurun_out/s4d_kern.log 2>&1; echo "kern rc=$?"; tail -2 gpurun_out/s4d_kern.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_two_sided.py -x -q --timeout 1400 -k "deterministic or above_160 or rank_deficient" > gpurun_out/s4d_det.log 2>&1; echo "det parity rc=$?"; tail -2 gpurun_out/s4d_det.log
for W in sum10 gmres; do
timeout 1200 python bench.py --algo deterministic --workload $W --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/s4d_bench_det_$W.json 2>&1; echo "det $W rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/s4d_bench_det_$W.json').read().strip().splitlines()[-1]);print('det $W', round(d['ms_per_step'],1), {k:round(v,1) for k,v in d['phase_ms'].items()})"
done
TTR_TRACE=gpurun_out/s4d_trace_det.txt timeout 900 python tools/run_det.py sum10 2>&1 | tail -1
head -8 gpurun_out/s4d_trace_det.txt
