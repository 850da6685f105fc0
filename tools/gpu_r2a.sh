# round 2, first GPU call: new tests, a timed bench with the full-size oracle baseline
mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_kernels.py -x -q --timeout 600 > gpurun_out/r2a_pytest_new.log 2>&1; echo "pytest-new rc=$?"; tail -3 gpurun_out/r2a_pytest_new.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "eps_threshold" > gpurun_out/r2a_pytest_eps.log 2>&1; echo "pytest-eps rc=$?"; tail -3 gpurun_out/r2a_pytest_eps.log
nproc > gpurun_out/r2a_host.txt; lscpu | grep -i "model name" >> gpurun_out/r2a_host.txt; free -g >> gpurun_out/r2a_host.txt
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?"; cut -c1-600 gpurun_out/r2a_bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2a_ref.json 2>&1; echo "ref rc=$?"; cut -c1-400 gpurun_out/r2a_ref.json
