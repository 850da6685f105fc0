mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_plan.py -x -q --timeout 600 > gpurun_out/r2u_plan.log 2>&1; echo "plan rc=$?"; tail -3 gpurun_out/r2u_plan.log
for W in "tiny 256" "single 64"; do set -- $W
  for br in 1 8 16; do
  timeout 600 python bench.py --workload $1 --batch $2 --graph --streams $br --steps 5 --warmup 3 --no-cpu > gpurun_out/r2u_${1}_graph_b$br.json 2>&1; echo "$1 graph branches $br rc=$?"; cut -c1-170 gpurun_out/r2u_${1}_graph_b$br.json
  done
done
