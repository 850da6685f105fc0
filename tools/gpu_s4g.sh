mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 2400 python -m pytest tests -m gpu -q --timeout 1800 > gpurun_out/s4g_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/s4g_pytest.log
