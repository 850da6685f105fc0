mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
TTR_TRACE=gpurun_out/s3s_trace_det.txt timeout 900 python tools/run_det.py sum10 2>&1 | tail -2
head -30 gpurun_out/s3s_trace_det.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 600 -k "jacobi or svd" > gpurun_out/s3s_kern.log 2>&1; echo "kern rc=$?"; tail -2 gpurun_out/s3s_kern.log
