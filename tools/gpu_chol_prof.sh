# per-phase clock64 profile of both Cholesky kernels (library built with -DTTR_CHOL_PROF)
mkdir -p gpurun_out
rm -rf paper_2110_04393_b200/csrc/build paper_2110_04393_b200/libttround.so
TTR_EXTRA_FLAGS=-DTTR_CHOL_PROF python -m paper_2110_04393_b200.build > /dev/null
TTR_CHOL=blk timeout 300 python tools/chol_prof.py
timeout 300 python tools/chol_prof.py
rm -rf paper_2110_04393_b200/csrc/build paper_2110_04393_b200/libttround.so
