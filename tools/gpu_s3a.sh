# session-3 baseline: GPU suite, bench line (no CPU leg), per-launch-site trace of C5
mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/s3a_bench.json 2> gpurun_out/s3a_bench.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/s3a_bench.json'));print(round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phase_ms'].items()}, round(d['roofline']['frac'],4), d.get('e2e',{}).get('value'))"
TTR_TRACE=gpurun_out/s3a_trace_large.txt timeout 600 python tools/run_once.py large - 2 > /dev/null 2>&1; echo "trace rc=$?"
awk '/^# trace/{n++} n==2' gpurun_out/s3a_trace_large.txt | head -50
timeout 2400 python -m pytest tests -m gpu -q --timeout 1800 > gpurun_out/s3a_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s3a_pytest.log
