mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_plan.py -x -q --timeout 600 -k "even_ragged or plan or graph" > gpurun_out/r2w.log 2>&1; echo "rc=$?"; tail -15 gpurun_out/r2w.log
