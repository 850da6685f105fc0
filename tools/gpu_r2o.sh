mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2o_seq.csv python tools/run_once.py large 6 1 > gpurun_out/r2o_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_seq.py gpurun_out/r2o_seq.csv | grep "ttr::" | awk '$2+0 > 30' | head -60
