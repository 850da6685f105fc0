mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 600 python tools/jac_bench.py 144 > gpurun_out/r2p_jac.txt 2>&1; TTR_JACOBI=cluster timeout 600 python tools/jac_bench.py 144 >> gpurun_out/r2p_jac.txt 2>&1; timeout 600 python tools/jac_bench.py 100 >> gpurun_out/r2p_jac.txt 2>&1; cat gpurun_out/r2p_jac.txt
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -k "not (two_sided and full_size)" > gpurun_out/r2p_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2p_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2p_bench.json 2>&1; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/r2p_bench.json'));print(round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phase_ms'].items()}, round(d['roofline']['frac'],4))"
