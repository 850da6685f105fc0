mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 600 python tools/jac_bench.py 144; TTR_JAC_SORT=1 timeout 600 python tools/jac_bench.py 144
timeout 300 python tools/run_once.py large 8 2 | tail -1 | cut -c1-200
TTR_JAC_SORT=1 timeout 300 python tools/run_once.py large 8 2 | tail -1 | cut -c1-200
