mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
for i in 1 2; do timeout 600 python tools/jac_bench.py 144; TTR_JACOBI=cluster timeout 600 python tools/jac_bench.py 144; done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q --timeout 900 -k "not full_size" > gpurun_out/r2q_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2q_pytest.log
