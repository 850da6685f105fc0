# Cholesky A/B: unit + parity tests on the new kernel, C5 phase timings for both
mkdir -p gpurun_out
T=${1:-ch1}
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q --timeout 900 -k "not full_size" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
for V in blk la; do
  if [ $V = blk ]; then export TTR_CHOL=blk; else unset TTR_CHOL; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_$V.json 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/${T}_bench_$V.json'));print('$V', round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phase_ms'].items()})"
done
unset TTR_CHOL
for W in tiny single sum10 gmres; do
  timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_$W.json 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/${T}_bench_$W.json'));print('$W', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phase_ms'].items()})"
done
