mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 300 python tools/run_once.py large 8 2 | tail -1 | cut -c1-260
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -k "not (two_sided and full_size)" > gpurun_out/r2x_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2x_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2x_bench.json 2>&1; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/r2x_bench.json'));print(round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phase_ms'].items()}, round(d['roofline']['frac'],4))"
