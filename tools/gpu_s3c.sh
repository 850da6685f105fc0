# ncu --set full of the fused CholeskyQR pass kernels (reduced C5, d=6)
mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 600 python tools/run_once.py large 6 1 > /dev/null 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:cqr_pass_kernel" -s 8 -c 4 -o gpurun_out/s3c_cqr_tg -f python tools/run_once.py large 6 1 > gpurun_out/s3c_ncu1.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:cqr_gram_reduce" -s 4 -c 1 -o gpurun_out/s3c_cqr_g -f python tools/run_once.py large 6 1 > gpurun_out/s3c_ncu2.log 2>&1; echo "ncu2 rc=$?"
for N in tg g; do
ncu -i gpurun_out/s3c_cqr_$N.ncu-rep --page details --csv > gpurun_out/s3c_cqr_${N}_details.csv 2>&1
ncu -i gpurun_out/s3c_cqr_$N.ncu-rep --page source --csv > gpurun_out/s3c_cqr_${N}_source.csv 2>&1
done
ls -la gpurun_out/ | grep s3c
