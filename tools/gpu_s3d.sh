mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 300 python tools/cqr_bench.py 36864 144 20 2>&1 | tee gpurun_out/s3d_cqr_bench.txt
timeout 300 python tools/cqr_bench.py 32768 144 20 2>&1 | tail -5
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:cqr_pass_kernel" -s 3 -c 1 -o gpurun_out/s3d_cqr -f python tools/cqr_bench.py 36864 144 1 > gpurun_out/s3d_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/s3d_cqr.ncu-rep --page details --csv > gpurun_out/s3d_cqr_details.csv 2>&1
ncu -i gpurun_out/s3d_cqr.ncu-rep --page source --csv > gpurun_out/s3d_cqr_source.csv 2>&1
