mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_two_sided.py -x -q --timeout 900 -k "not full_size" > gpurun_out/pytest_2s.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_2s.log
tail -15 gpurun_out/pytest_2s.log
timeout 900 python bench.py --algo two_sided --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_2s.json 2> gpurun_out/bench_2s.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_2s.json; tail -5 gpurun_out/bench_2s.err
