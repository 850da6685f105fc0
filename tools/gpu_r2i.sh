mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "not full_size and not deterministic" > gpurun_out/r2i_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/r2i_parity.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2i_bench_fused.json 2>&1; echo "bench rc=$?"
TTR_NO_FUSE=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2i_bench_nofuse.json 2>&1; echo "bench-nofuse rc=$?"
for f in fused nofuse; do python -c "
import json;d=json.load(open('gpurun_out/r2i_bench_$f.json'));print('$f', round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phase_ms'].items()}, round(d['roofline']['frac'],4))"; done
