# ncu --set full of the CURRENT (32-wide k-step) phase-1 W GEMM, Y_n GEMM, the
# fused projection-and-carry, the Z GEMM and the Jacobi (reduced C5, d=6), after a
# plain run of the same command; plus the NCCL plumbing self-test.
mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "per_bond" --timeout 600 > gpurun_out/s6a_perbond.log 2>&1; echo "per-bond tests rc=$?"; tail -3 gpurun_out/s6a_perbond.log
timeout 600 python -m pytest tests/test_gpu_sharded.py -q -k nccl --timeout 300 > gpurun_out/s6a_nccl.log 2>&1; echo "nccl test rc=$?"; tail -3 gpurun_out/s6a_nccl.log
timeout 300 python tools/run_once.py large 6 1 > gpurun_out/s6a_plain.log 2>&1; echo "plain rc=$?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed
run() {  # name regex skip count
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$2" -s $3 -c $4 -o gpurun_out/s6a_$1 -f python tools/run_once.py large 6 1 > gpurun_out/s6a_ncu_$1.log 2>&1; echo "ncu $1 rc=$?"
  ncu -i gpurun_out/s6a_$1.ncu-rep --page raw --csv --metrics $M > gpurun_out/s6a_ncu_$1_raw.csv 2>&1
}
run wgemm 'dgemm_tma_kernel<\(int\)64, \(int\)48, \(int\)32, \(int\)4, \(int\)2, \(int\)3, \(bool\)0, \(bool\)1>' 2 1
run ygemm 'dgemm_tma_kernel<\(int\)128, \(int\)48, \(int\)32, \(int\)4, \(int\)2, \(int\)2, \(bool\)0, \(bool\)0>' 1 1
run projcarry 'proj_carry_kernel' 1 1
run zgemm 'pgemm_kernel' 2 1
run jacobi 'jacobi_cluster_kernel' 2 1
for N in wgemm ygemm projcarry zgemm jacobi; do echo "== $N"; cat gpurun_out/s6a_ncu_${N}_raw.csv | head -5 | cut -c1-700; done
# one-rank NCCL context: the sharded path's tests, then C5 with the exchange steps
# going through ncclAllReduce (summand shards and mode slabs)
timeout 900 python -m pytest tests/test_gpu_sharded.py -q -k "nccl" --timeout 600 > gpurun_out/s6a_nccl2.log 2>&1; echo "nccl ctx tests rc=$?"; tail -3 gpurun_out/s6a_nccl2.log
timeout 600 python bench.py --nccl-one-rank --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/s6a_bench_large_nccl1.json 2> gpurun_out/s6a_bench_large_nccl1.err; echo "bench nccl1 rc=$?"; cut -c1-200 gpurun_out/s6a_bench_large_nccl1.json
timeout 600 python bench.py --nccl-one-rank --shard slab --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/s6a_bench_large_slab_nccl1.json 2> gpurun_out/s6a_bench_large_slab_nccl1.err; echo "bench slab nccl1 rc=$?"; cut -c1-200 gpurun_out/s6a_bench_large_slab_nccl1.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/s6a_bench_torchrun1.json 2> gpurun_out/s6a_bench_torchrun1.err; echo "torchrun1 rc=$?"; cut -c1-200 gpurun_out/s6a_bench_torchrun1.json
