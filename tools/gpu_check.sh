# quick state check on the GPU box: smoke, full GPU suite, default bench line, launch list
# usage: bash tools/gpu_check.sh <tag>
T=${1:-c1}
mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${T}_smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 1800 > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/${T}_bench.json
python -c "
import json;d=json.load(open('gpurun_out/${T}_bench.json'));print(round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phase_ms'].items()}, round(d['roofline']['frac'],4), d.get('e2e'))"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 100000 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
python tools/ncu_agg.py gpurun_out/${T}_launches.csv 30 > gpurun_out/${T}_launches.txt 2>&1; head -40 gpurun_out/${T}_launches.txt
