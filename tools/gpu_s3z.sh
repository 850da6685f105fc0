mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 300 python tools/chol_bench.py
touch paper_2110_04393_b200/csrc/linalg.cu
TTR_EXTRA_FLAGS=-DTTR_CHOL_NOINV python -m paper_2110_04393_b200.build > /dev/null
echo "without inverse:"; timeout 300 python tools/chol_bench.py 2>&1 | tail -3
touch paper_2110_04393_b200/csrc/linalg.cu
