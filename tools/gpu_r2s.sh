mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_two_sided.py -x -q --timeout 900 -k "not full_size" > gpurun_out/r2s_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2s_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2s_bench.json 2>&1; echo "bench rc=$?"
TTR_NO_PGEMM=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2s_bench_nopg.json 2>&1; echo "bench rc=$?"
for f in r2s_bench r2s_bench_nopg; do python -c "
import json;d=json.load(open('gpurun_out/$f.json'));print('$f', round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phase_ms'].items()}, round(d['roofline']['frac'],4))"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s_seq.csv python tools/run_once.py large 6 1 > /dev/null 2>&1
python tools/ncu_seq.py gpurun_out/r2s_seq.csv | grep "pgemm\|dgemm_tma_kernel<64, 48, 16, 4, 2, 4, 0, 1>" | head -8; rm -f gpurun_out/r2s_seq.csv
