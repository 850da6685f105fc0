mkdir -p gpurun_out
rm -f paper_2110_04393_b200/csrc/build/linalg.o
TTR_EXTRA_FLAGS=-DTTR_CHOL_PROF python -m paper_2110_04393_b200.build > /dev/null
timeout 300 python tools/chol_prof.py > gpurun_out/r2g_chol_prof.txt 2>&1; echo "prof rc=$?"; cat gpurun_out/r2g_chol_prof.txt
rm -f paper_2110_04393_b200/csrc/build/linalg.o
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 600 > gpurun_out/r2g_kern.log 2>&1; echo "kernels rc=$?"; tail -3 gpurun_out/r2g_kern.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2g_bench.json 2>&1; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/r2g_bench.json'));print(round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phase_ms'].items()}, round(d['roofline']['frac'],4))"
