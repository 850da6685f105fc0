# Cholesky launch durations (ncu, cold caches) of the new look-ahead kernel and the
# round-1 one on a reduced config 5 (d = 6), then one --set full capture each
mkdir -p gpurun_out
T=${1:-cn1}
IDX=${2:-20}
python -m paper_2110_04393_b200.build > /dev/null
for V in la blk; do
  if [ $V = blk ]; then export TTR_CHOL=blk; else unset TTR_CHOL; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name-base demangled -k "regex:chol_(la|blk)_kernel" --log-file gpurun_out/${T}_${V}_dur.csv python tools/run_once.py large 6 1 > /dev/null 2>&1; echo "ncu dur $V rc=$?"
  python tools/ncu_seq.py gpurun_out/${T}_${V}_dur.csv | awk '{print $2}' | tr '\n' ' '; echo
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:chol_(la|blk)_kernel" -s $IDX -c 1 -o /tmp/${T}_$V -f python tools/run_once.py large 6 1 > /dev/null 2>&1; echo "ncu full $V rc=$?"
  ncu -i /tmp/${T}_$V.ncu-rep --page details --csv > gpurun_out/${T}_${V}_details.csv 2>&1
  ncu -i /tmp/${T}_$V.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_${V}_source.csv 2>&1
  grep '"Duration"' gpurun_out/${T}_${V}_details.csv | cut -c1-300
done
