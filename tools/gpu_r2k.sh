mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_gmres.py -x -q --timeout 600 > gpurun_out/r2k_gmres.log 2>&1; echo "gmres rc=$?"; tail -30 gpurun_out/r2k_gmres.log
