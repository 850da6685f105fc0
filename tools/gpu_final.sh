# round-2 final evidence: smoke, GPU suite, default bench line (+ full-size oracle
# baseline), reference arm, launch list of the bench command, ncu --set full of the
# top kernels, per-config / batched / two-sided / deterministic lines.
# Usage: bash tools/gpu_final.sh <tag>
T=${1:-f1}
mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" | tee -a gpurun_out/${T}_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench_large.json 2> gpurun_out/${T}_bench_large.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/${T}_bench_large.json
timeout 2400 python -m pytest tests -m gpu -q --timeout 1800 > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_ref_large.json 2>&1; echo "ref rc=$?"; cut -c1-300 gpurun_out/${T}_ref_large.json
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 100000 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
python tools/ncu_agg.py gpurun_out/${T}_launches.csv 30 > gpurun_out/${T}_launches.txt 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,sm__throughput.avg.pct_of_peak_sustained_elapsed
for spec in "wgemm|dgemm_tma_kernel<64, 48, 16, 4, 2, 4, 0, 1>|3" "zgemm|pgemm_kernel|3" "ygemm|dgemm_tma_kernel<128, 48, 16, 4, 2, 4, 0, 0>|1" "projcarry|proj_carry_kernel|1" "jacobi|jacobi_cluster_kernel|1" "chol|chol_la_kernel|6" "cqr|cqr_pass_kernel<0, 1, 1|2"; do
  IFS='|' read -r N RGX SKIP <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$RGX" -s $SKIP -c 1 -o gpurun_out/${T}_$N -f python tools/run_once.py large 6 1 > gpurun_out/${T}_ncu_$N.log 2>&1; echo "ncu full $N rc=$?"
  ncu -i gpurun_out/${T}_$N.ncu-rep --page raw --csv --metrics $M > gpurun_out/${T}_ncu_${N}_raw.csv 2>&1
done
for W in tiny single sum10 gmres; do
  timeout 900 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu > gpurun_out/${T}_bench_$W.json 2>&1; echo "bench $W rc=$?"
done
timeout 900 python bench.py --algo two_sided --steps 10 --warmup 3 --no-cpu > gpurun_out/${T}_bench_large_two_sided.json 2>&1; echo "bench 2s rc=$?"
timeout 600 python bench.py --workload tiny --batch 256 --graph --streams 16 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_tiny_graph_b256.json 2>&1; echo "tiny graph rc=$?"
timeout 600 python bench.py --workload single --batch 64 --graph --streams 16 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_single_graph_b64.json 2>&1; echo "single graph rc=$?"
for W in tiny single; do
  timeout 900 python bench.py --algo deterministic --workload $W --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_det_$W.json 2>&1; echo "det $W rc=$?"
done
timeout 1200 python bench.py --algo deterministic --workload sum10 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_det_sum10.json 2>&1; echo "det sum10 rc=$?"
