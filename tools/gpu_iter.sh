# one iteration on the GPU box: tests, C5 timing, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python tools/run_once.py large - 3 > gpurun_out/run_large.log 2>&1; echo "run rc=$?"; tail -3 gpurun_out/run_large.log
if [ "${NCU:-1}" = "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches_large.csv python tools/run_once.py large - 1 > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
fi
