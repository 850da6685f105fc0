# round-end style evidence: tests, bench line, launch list of the bench command, full capture of the top phase-1 kernel
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_large.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_large.log | cut -c1-300
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 100000 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo "ncu launches rc=$?"
if [ "${NCU_FULL:-1}" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:dgemm_kernel<.int.64, .int.48" -s 20 -c 1 -o gpurun_out/prof_w -f python tools/run_once.py large - 1 > gpurun_out/ncu_w.log 2>&1; echo "ncu full rc=$?"
fi
for w in tiny single sum10 gmres; do timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_$w.log 2>&1; done
timeout 300 python bench.py --workload tiny --batch 256 --steps 3 --warmup 3 > gpurun_out/bench_tiny_batch.log 2>&1
timeout 300 python bench.py --workload single --batch 64 --steps 3 --warmup 3 > gpurun_out/bench_single_batch.log 2>&1
timeout 600 python bench.py --algo two_sided --no-cpu > gpurun_out/bench_large_two_sided.log 2>&1; echo "bench 2s rc=$?"
timeout 600 python bench.py --algo two_sided --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_plain_2s.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 100000 --csv --log-file gpurun_out/launches_bench_2s.csv python bench.py --algo two_sided --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_bench_2s.log 2>&1; echo "ncu 2s launches rc=$?"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
