# per-launch sequence of a reduced C5 rounding (d=6), plus the smoke
mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 300 python tools/run_once.py large 6 2 > gpurun_out/r2b_plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/r2b_plain.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_seq.csv python tools/run_once.py large 6 2 > gpurun_out/r2b_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_seq.py gpurun_out/r2b_seq.csv > gpurun_out/r2b_seq.txt; wc -l gpurun_out/r2b_seq.txt
