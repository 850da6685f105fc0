mkdir -p gpurun_out
T=${1:-ch2}
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_two_sided.py tests/test_gpu_gmres.py -q --timeout 900 -k "not full_size" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench.json 2>&1
python -c "
import json;d=json.load(open('gpurun_out/${T}_bench.json'));print(round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phase_ms'].items()})"
rm -rf paper_2110_04393_b200/csrc/build paper_2110_04393_b200/libttround.so
TTR_EXTRA_FLAGS=-DTTR_CHOL_PROF python -m paper_2110_04393_b200.build > /dev/null
TTR_CHOL=blk timeout 300 python tools/chol_prof.py
timeout 300 python tools/chol_prof.py
rm -rf paper_2110_04393_b200/csrc/build paper_2110_04393_b200/libttround.so
