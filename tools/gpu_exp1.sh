# experiment: C5 throughput with independent roundings in flight / CUDA graph
mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 600 python bench.py --workload large --batch 2 --streams 2 --steps 4 --warmup 3 > gpurun_out/x1_b2s2.json 2>&1; echo "b2s2 rc=$?"; cut -c1-300 gpurun_out/x1_b2s2.json
timeout 600 python bench.py --workload large --batch 1 --graph --steps 5 --warmup 3 > gpurun_out/x1_g1.json 2>&1; echo "g1 rc=$?"; cut -c1-300 gpurun_out/x1_g1.json
timeout 600 python bench.py --workload large --batch 2 --graph --streams 2 --steps 4 --warmup 3 > gpurun_out/x1_g2.json 2>&1; echo "g2 rc=$?"; cut -c1-300 gpurun_out/x1_g2.json
timeout 600 python bench.py --workload large --batch 3 --streams 3 --steps 3 --warmup 3 > gpurun_out/x1_b3s3.json 2>&1; echo "b3s3 rc=$?"; cut -c1-300 gpurun_out/x1_b3s3.json
