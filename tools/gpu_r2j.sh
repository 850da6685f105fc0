mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 300 python tools/run_once.py large 6 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2j_seq.csv python tools/run_once.py large 6 1 > gpurun_out/r2j_ncu.log 2>&1; echo "ncu seq rc=$?"
python tools/ncu_seq.py gpurun_out/r2j_seq.csv | grep "proj_carry\|dgemm_tma_kernel<128, 48" | head -8
timeout 900 ncu --set full --clock-control none --import-source on -k regex:proj_carry -s 1 -c 1 -o gpurun_out/r2j_pc -f python tools/run_once.py large 6 1 > gpurun_out/r2j_ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/r2j_pc.ncu-rep --page details --csv > gpurun_out/r2j_pc_details.csv 2>&1
grep -i "Duration\|Tensor\|DRAM Throughput\|Registers\|Achieved Occupancy\|Stall\|Warp Cycles Per Issued\|Issue Slots" gpurun_out/r2j_pc_details.csv | head -30
