mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 600 > gpurun_out/r2e_kern.log 2>&1; echo "kernels rc=$?"; tail -3 gpurun_out/r2e_kern.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2e_bench_tma.json 2>&1; echo "bench rc=$?"
TTR_NO_TMA=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2e_bench_notma.json 2>&1; echo "bench-notma rc=$?"
for f in tma notma; do python -c "
import json;d=json.load(open('gpurun_out/r2e_bench_$f.json'));print('$f', round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phase_ms'].items()}, round(d['roofline']['frac'],4))"; done
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -k "not (two_sided and full_size)" > gpurun_out/r2e_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2e_pytest.log
