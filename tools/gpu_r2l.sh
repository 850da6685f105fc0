mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_sharded.py -x -q --timeout 600 > gpurun_out/r2l_slab.log 2>&1; echo "slab rc=$?"; tail -30 gpurun_out/r2l_slab.log
