# histogram of max|G - I| before the sweep QR's third pass (route 1) and the
# truncation's pass 4 (build with -DTTR_NEARID_PROF; status words 40-63)
mkdir -p gpurun_out
touch paper_2110_04393_b200/csrc/linalg.cu
TTR_EXTRA_FLAGS=-DTTR_NEARID_PROF python -m paper_2110_04393_b200.build > /dev/null
for W in large single sum10 gmres; do
  timeout 600 python tools/run_once.py $W - 1 2>&1 | tail -1 | python3 -c "
import sys
l=sys.stdin.read(); st=eval(l.split('status')[1])
print('$W sweep 3rd-pass max|G-I| 10^-b histogram b=0..19:', st[40:60], ' trunc pass-4 [0-4,5-9,10-14,15-19]:', st[60:64])"
done
touch paper_2110_04393_b200/csrc/linalg.cu
