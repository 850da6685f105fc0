mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
for W in tiny single sum10 gmres large; do
  timeout 600 python tools/run_once.py $W - 1 2>&1 | tail -1 | python3 -c "
import sys,re
l=sys.stdin.read(); st=eval(l.split('status')[1])
print('$W', 'cholqr2',st[8],'scholqr3',st[10],'scholqr4',st[15],'householder',st[11],'tsqr',st[14],'jacobi sweeps/calls',st[12],st[13],'clamped',st[16])"
done
