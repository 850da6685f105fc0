mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/run_once.py large - 2
timeout 300 python tools/run_once.py gmres - 2
timeout 600 python tools/diag_spectra.py large > gpurun_out/spectra_large.log 2>&1
