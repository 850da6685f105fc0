# concurrent roundings after the stream-ordered-free fix: tests, C5 with K in flight
mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_concurrency.py -x -q --timeout 600 > gpurun_out/s5b_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s5b_tests.log
for KR in "2 16" "2 0" "2 8" "3 16" "2 32"; do set -- $KR
  timeout 600 python bench.py --inflight $1 --reserve-sms $2 --steps 6 --warmup 3 --no-cpu --no-e2e > gpurun_out/s5b_inf$1_r$2.json 2>gpurun_out/s5b_inf$1_r$2.err
  python -c "
import json;d=json.loads(open('gpurun_out/s5b_inf$1_r$2.json').read().strip().splitlines()[-1]);print('inflight $1 reserve $2', round(d['value'],3), round(d['ms_per_step'],1), {k:round(v,1) for k,v in d['phase_ms'].items()}, round(d['roofline']['frac'],3))" || tail -3 gpurun_out/s5b_inf$1_r$2.err
done
timeout 600 python bench.py --batch 2 --streams 2 --reserve-sms 16 --steps 6 --warmup 3 --no-cpu > gpurun_out/s5b_b2_r16.json 2>gpurun_out/s5b_b2_r16.err
python -c "
import json;d=json.loads(open('gpurun_out/s5b_b2_r16.json').read().strip().splitlines()[-1]);print('b2 r16', round(d['value'],3), round(d['ms_per_step'],1))" || tail -3 gpurun_out/s5b_b2_r16.err
