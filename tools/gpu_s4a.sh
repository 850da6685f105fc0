mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 600 -k "chol or qr" > gpurun_out/s4f_kern.log 2>&1; echo "kern rc=$?"; tail -2 gpurun_out/s4f_kern.log
timeout 300 python tools/chol_bench.py
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 1400 -k "deterministic" > gpurun_out/s4f_det.log 2>&1; echo "det parity rc=$?"; tail -2 gpurun_out/s4f_det.log
timeout 1200 python bench.py --algo deterministic --workload sum10 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/s4f_bench_det_sum10.json 2>&1; echo "det sum10 rc=$?"
timeout 1200 python bench.py --algo deterministic --workload gmres --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/s4f_bench_det_gmres.json 2>&1; echo "det gmres rc=$?"
for W in sum10 gmres; do python -c "
import json;d=json.loads(open('gpurun_out/s4f_bench_det_$W.json').read().strip().splitlines()[-1]);print('det $W', round(d['ms_per_step'],1), {k:round(v,1) for k,v in d['phase_ms'].items()})"; done
