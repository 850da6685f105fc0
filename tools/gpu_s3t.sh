mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 600 -k "chol or qr or jacobi" > gpurun_out/s3t_kern.log 2>&1; echo "kern rc=$?"; tail -2 gpurun_out/s3t_kern.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_two_sided.py -x -q --timeout 900 -k "deterministic or rho_gt or large_ell or 160" > gpurun_out/s3t_det.log 2>&1; echo "det parity rc=$?"; tail -2 gpurun_out/s3t_det.log
TTR_TRACE=gpurun_out/s3t_trace_det.txt timeout 900 python tools/run_det.py sum10 2>&1 | tail -1
head -8 gpurun_out/s3t_trace_det.txt
