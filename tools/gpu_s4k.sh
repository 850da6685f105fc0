mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/s4l_bench.json 2>&1
python -c "
import json;d=json.load(open('gpurun_out/s4l_bench.json'));print(round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phase_ms'].items()}, round(d['roofline']['frac'],4))"
for W in single sum10; do
  timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/s4l_bench_$W.json 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/s4l_bench_$W.json'));print('$W', round(d['ms_per_step'],3))"
done
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 600 -k "dgemm or qr" > gpurun_out/s4l_kern.log 2>&1; echo "kern rc=$?"; tail -2 gpurun_out/s4l_kern.log
