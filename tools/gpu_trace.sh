# in-pipeline per-launch-site time of one C5 rounding (TTR_TRACE) + the other configs
mkdir -p gpurun_out
T=${1:-tr1}
python -m paper_2110_04393_b200.build > /dev/null
rm -f gpurun_out/${T}_*.txt
for W in large single sum10; do
  TTR_TRACE=gpurun_out/${T}_$W.txt timeout 600 python tools/run_once.py $W - 2 > /dev/null 2>&1; echo "$W rc=$?"
  awk '/^# trace/{n++} n==2' gpurun_out/${T}_$W.txt | head -45
done
