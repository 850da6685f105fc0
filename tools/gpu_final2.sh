# round-2 final evidence (v4): smoke, GPU suite, default bench line (+ oracle
# baseline, e2e), reference arm, launch list, per-config / two-sided / graph /
# deterministic lines.  Usage: bash tools/gpu_final2.sh <tag>
T=${1:-f2}
mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" | tee -a gpurun_out/${T}_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench_large.json 2> gpurun_out/${T}_bench_large.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/${T}_bench_large.json
timeout 2400 python -m pytest tests -m gpu -q --timeout 1800 > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_ref_large.json 2>&1; echo "ref rc=$?"
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 100000 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
python tools/ncu_agg.py gpurun_out/${T}_launches.csv 30 > gpurun_out/${T}_launches.txt 2>&1
for W in tiny single sum10 gmres; do
  timeout 900 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu > gpurun_out/${T}_bench_$W.json 2>&1; echo "bench $W rc=$?"
done
timeout 900 python bench.py --algo two_sided --steps 10 --warmup 3 --no-cpu > gpurun_out/${T}_bench_large_two_sided.json 2>&1; echo "bench 2s rc=$?"
timeout 600 python bench.py --workload tiny --batch 256 --graph --streams 16 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_tiny_graph_b256.json 2>&1; echo "tiny graph rc=$?"
timeout 600 python bench.py --workload single --batch 64 --graph --streams 16 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_single_graph_b64.json 2>&1; echo "single graph rc=$?"
for W in tiny single sum10 gmres; do
  timeout 900 python bench.py --algo deterministic --workload $W --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_det_$W.json 2>&1; echo "det $W rc=$?"
done
