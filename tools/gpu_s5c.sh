# staggered free-running lanes (bench --inflight K): C5 throughput
mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
for KR in "2 16" "2 8" "3 16" "4 16" "2 0"; do set -- $KR
  timeout 600 python bench.py --inflight $1 --reserve-sms $2 --steps 8 --warmup 3 --no-cpu --no-e2e > gpurun_out/s5c_inf$1_r$2.json 2>gpurun_out/s5c_inf$1_r$2.err
  python -c "
import json;d=json.loads(open('gpurun_out/s5c_inf$1_r$2.json').read().strip().splitlines()[-1]);print('inflight $1 reserve $2', round(d['value'],3), round(d['ms_per_step'],1), {k:round(v,1) for k,v in d['phase_ms'].items()}, round(d['roofline']['frac'],3))" || tail -3 gpurun_out/s5c_inf$1_r$2.err
done
