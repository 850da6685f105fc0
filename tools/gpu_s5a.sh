# concurrent roundings (tt_ctx_set_concurrency): tests, then C5 with 2 roundings in
# flight at several SM reserves
mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_concurrency.py -x -q --timeout 600 > gpurun_out/s5a_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s5a_tests.log
for R in -1 0 8 16 24; do
  timeout 600 python bench.py --batch 2 --streams 2 --reserve-sms $R --steps 6 --warmup 3 --no-cpu > gpurun_out/s5a_b2_r$R.json 2>gpurun_out/s5a_b2_r$R.err
  python -c "
import json;d=json.loads(open('gpurun_out/s5a_b2_r$R.json').read().strip().splitlines()[-1]);print('b2 reserve $R', round(d['value'],3), round(d['ms_per_step'],1), round(d['config']['host_ms_per_step'],1))"
done
timeout 600 python bench.py --batch 4 --streams 4 --reserve-sms 16 --steps 4 --warmup 3 --no-cpu > gpurun_out/s5a_b4s4_r16.json 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/s5a_b4s4_r16.json').read().strip().splitlines()[-1]);print('b4s4 r16', round(d['value'],3), round(d['ms_per_step'],1))"
for W in sum10 single; do
 for R in -1 8; do
  timeout 600 python bench.py --workload $W --batch 8 --streams 2 --reserve-sms $R --steps 10 --warmup 3 --no-cpu > gpurun_out/s5a_${W}_b8_r$R.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/s5a_${W}_b8_r$R.json').read().strip().splitlines()[-1]);print('$W b8s2 r$R', round(d['value'],2), round(d['ms_per_step'],2))"
 done
done
for KR in "2 16" "2 8" "3 16"; do set -- $KR
  timeout 600 python bench.py --inflight $1 --reserve-sms $2 --steps 6 --warmup 3 --no-cpu --no-e2e > gpurun_out/s5a_inf$1_r$2.json 2>gpurun_out/s5a_inf$1_r$2.err
  python -c "
import json;d=json.loads(open('gpurun_out/s5a_inf$1_r$2.json').read().strip().splitlines()[-1]);print('inflight $1 reserve $2', round(d['value'],3), round(d['ms_per_step'],1), {k:round(v,1) for k,v in d['phase_ms'].items()}, round(d['roofline']['frac'],3))" || tail -3 gpurun_out/s5a_inf$1_r$2.err
done
