mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -k "not (two_sided and full_size)" > gpurun_out/r2h_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2h_pytest.log
