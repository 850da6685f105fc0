mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
for sc in 1 100 10000; do
  echo "tol scale $sc"; TTR_JAC_TOL=$sc timeout 600 python tools/jac_bench.py 144
  TTR_JAC_TOL=$sc timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2y_bench_$sc.json 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/r2y_bench_$sc.json'));print('bench', round(d['ms_per_step'],2), 'trunc', round(d['phase_ms']['truncation'],2))"
done
TTR_JAC_TOL=10000 timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -k "config5_full or config3 or config4 or closed_form or eps" > gpurun_out/r2y_parity.log 2>&1; echo "parity(1e4) rc=$?"; tail -3 gpurun_out/r2y_parity.log
