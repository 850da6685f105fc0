mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gmres.py -x -q --timeout 900 -k "deterministic" > gpurun_out/s3v_det.log 2>&1; echo "det parity rc=$?"; tail -3 gpurun_out/s3v_det.log
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 600 -k "chol" > gpurun_out/s3v_kern.log 2>&1; echo "kern rc=$?"; tail -2 gpurun_out/s3v_kern.log
for W in tiny single sum10 gmres; do
TTR_TRACE=gpurun_out/s3v_trace_det_$W.txt timeout 900 python tools/run_det.py $W 2>&1 | tail -1
done
head -8 gpurun_out/s3v_trace_det_sum10.txt
