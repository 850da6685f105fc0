mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:chol_blk_kernel" -s 0 -c 10 -o /tmp/r2r_chol -f python tools/run_once.py large 6 1 > gpurun_out/r2r_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/r2r_chol.ncu-rep --page raw --csv > gpurun_out/r2r_chol_raw.csv 2>/dev/null
ls -la gpurun_out/r2r_chol_raw.csv
