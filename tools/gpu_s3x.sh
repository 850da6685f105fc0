# ncu --set full of the phase-1 W GEMM (TMA kernel: DRAM traffic for bench.py's
# roofline), the Y_n GEMM, a fused CholeskyQR pass and live Cholesky calls (reduced C5, d=6)
mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,sm__throughput.avg.pct_of_peak_sustained_elapsed
run() {  # name regex skip count
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$2" -s $3 -c $4 -o gpurun_out/s3x_$1 -f python tools/run_once.py large 6 1 > gpurun_out/s3x_ncu_$1.log 2>&1; echo "ncu $1 rc=$?"
  ncu -i gpurun_out/s3x_$1.ncu-rep --page raw --csv --metrics $M > gpurun_out/s3x_ncu_$1_raw.csv 2>&1
}
run wgemm 'dgemm_tma_kernel<\(int\)64, \(int\)48, \(int\)16, \(int\)4, \(int\)2, \(int\)4, \(bool\)0, \(bool\)1>' 2 1
run ygemm 'dgemm_tma_kernel<\(int\)128, \(int\)48, \(int\)16, \(int\)4, \(int\)2, \(int\)4, \(bool\)0, \(bool\)0>' 1 1
run cqr 'cqr_pass_kernel<\(bool\)0, \(bool\)1, \(bool\)1' 2 1
run chol 'chol_la_kernel' 26 3
for N in wgemm ygemm cqr chol; do echo "== $N"; cat gpurun_out/s3x_ncu_${N}_raw.csv | head -5 | cut -c1-600; done
