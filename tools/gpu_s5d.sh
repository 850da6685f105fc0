# single-rounding latency under CUDA-graph replay (tt_plan, B = 1) vs eager
mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
for W in tiny single sum10 large; do
  timeout 900 python bench.py --workload $W --batch 1 --graph --streams 1 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/s5d_${W}_graph_b1.json 2>gpurun_out/s5d_${W}_graph_b1.err
  python -c "
import json;d=json.loads(open('gpurun_out/s5d_${W}_graph_b1.json').read().strip().splitlines()[-1]);print('$W graph b1', round(d['value'],2), round(d['ms_per_step'],3))" || tail -3 gpurun_out/s5d_${W}_graph_b1.err
done
timeout 600 python bench.py --workload single --steps 10 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100000 --csv --log-file gpurun_out/s5d_single_launches.csv python bench.py --workload single --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_agg.py gpurun_out/s5d_single_launches.csv 25 > gpurun_out/s5d_single_launches.txt 2>&1; head -25 gpurun_out/s5d_single_launches.txt
