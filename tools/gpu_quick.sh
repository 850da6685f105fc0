# quick check: kernel + two-sided tests, batched throughput of the small configs
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_two_sided.py -x -q --timeout 600 -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
tail -2 gpurun_out/pytest_quick.log
for s in 1 8; do
timeout 300 python bench.py --workload tiny --batch 256 --streams $s --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_tiny_batch_s$s.log 2>&1; echo "tiny s=$s rc=$?"; tail -1 gpurun_out/bench_tiny_batch_s$s.log | cut -c1-160
timeout 300 python bench.py --workload single --batch 64 --streams $s --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_single_batch_s$s.log 2>&1; echo "single s=$s rc=$?"; tail -1 gpurun_out/bench_single_batch_s$s.log | cut -c1-160
done
