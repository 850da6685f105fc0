# TMA stage-count sweep on C5 (bench, no CPU / e2e legs) + launch list of the default
mkdir -p gpurun_out
for st in 2 3 5; do
  rm -f paper_2110_04393_b200/csrc/build/gemm.o
  TTR_EXTRA_FLAGS="-DTTR_TMA_STAGES=$st" python -m paper_2110_04393_b200.build > /dev/null
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2f_bench_st$st.json 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/r2f_bench_st$st.json'));print('stages $st', round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phase_ms'].items()}, round(d['roofline']['frac'],4))"
done
rm -f paper_2110_04393_b200/csrc/build/gemm.o
python -m paper_2110_04393_b200.build > /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_seq.csv python tools/run_once.py large 6 1 > gpurun_out/r2f_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_seq.py gpurun_out/r2f_seq.csv > gpurun_out/r2f_seq.txt
