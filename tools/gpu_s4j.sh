mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/s4j_bench.json 2>&1
python -c "
import json;d=json.load(open('gpurun_out/s4j_bench.json'));print(round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phase_ms'].items()}, round(d['roofline']['frac'],4))"
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size --clock-control none --csv --kernel-name-base demangled -k regex:proj_carry -c 2 --log-file gpurun_out/s4j_pc.csv python tools/run_once.py large 6 1 > /dev/null 2>&1
grep -o '"\(gpu__time_duration.sum\|sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active\|launch__grid_size\)","[a-zA-Z%]*","[0-9.,]*"' gpurun_out/s4j_pc.csv | head -6
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q --timeout 900 -k "not full_size and not deterministic" > gpurun_out/s4j_par.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/s4j_par.log
