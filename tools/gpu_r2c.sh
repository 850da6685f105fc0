mkdir -p gpurun_out
rm -f paper_2110_04393_b200/csrc/build/linalg.o
TTR_EXTRA_FLAGS=-DTTR_CHOL_PROF python -m paper_2110_04393_b200.build > /dev/null
timeout 300 python tools/chol_prof.py > gpurun_out/r2c_chol_prof.txt 2>&1; echo "prof rc=$?"; cat gpurun_out/r2c_chol_prof.txt
rm -f paper_2110_04393_b200/csrc/build/linalg.o
python -m paper_2110_04393_b200.build > /dev/null
