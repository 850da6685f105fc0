# last confirmation of the round at the final commit: smoke, the whole GPU suite,
# the default bench line (oracle baseline, e2e + pipelined) and the reference arm.
T=${1:-f8}
mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" | tee -a gpurun_out/${T}_smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 1800 > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench_large.json 2> gpurun_out/${T}_bench_large.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/${T}_bench_large.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_ref_large.json 2>&1; echo "ref rc=$?"
