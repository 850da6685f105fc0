mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
for V in none r0 r2 both; do
  unset TTR_X_NO_ROUTE0 TTR_X_NO_ROUTE2
  case $V in r0) export TTR_X_NO_ROUTE0=1;; r2) export TTR_X_NO_ROUTE2=1;; both) export TTR_X_NO_ROUTE0=1 TTR_X_NO_ROUTE2=1;; esac
  for W in single gmres; do
    timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/s3n_${W}_$V.json 2>&1
    python -c "
import json;d=json.load(open('gpurun_out/s3n_${W}_$V.json'));print('$W $V', round(d['ms_per_step'],3), {k:round(x,3) for k,x in d['phase_ms'].items()})"
  done
done
