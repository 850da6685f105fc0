# deterministic (Alg. 1 + 2 on the assembled sum) vs randomized on the configs where the assembled sum fits
mkdir -p gpurun_out
for w in tiny single sum10 gmres; do
timeout 600 python bench.py --algo deterministic --workload $w --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_det_$w.log 2>&1; echo "det $w rc=$?"; tail -1 gpurun_out/bench_det_$w.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['config']['workload'], j['value'], j['ms_per_step'], j['ranks_out'][:6])"
done
