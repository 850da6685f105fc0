mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 600 python tools/jac_bench.py 144 > gpurun_out/r2m_jac.txt 2>&1; cat gpurun_out/r2m_jac.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jacobi_cluster -s 2 -c 1 -o gpurun_out/r2m_jac -f python tools/jac_bench.py 144 > gpurun_out/r2m_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/r2m_jac.ncu-rep --page source --csv --print-source sass > gpurun_out/r2m_jac_sass.csv 2>/dev/null; echo "src rc=$?"
ncu -i gpurun_out/r2m_jac.ncu-rep --page source --csv > gpurun_out/r2m_jac_src.csv 2>/dev/null; echo "src2 rc=$?"
ncu -i gpurun_out/r2m_jac.ncu-rep --page details --csv > gpurun_out/r2m_jac_details.csv 2>&1
ls -la gpurun_out/r2m_*
