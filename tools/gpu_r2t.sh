mkdir -p gpurun_out
for st in 2 3; do
  rm -f paper_2110_04393_b200/csrc/build/pgemm.o
  TTR_EXTRA_FLAGS="-DTTR_PG_STAGES=$st" python -m paper_2110_04393_b200.build > /dev/null
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/seq_$st.csv python tools/run_once.py large 6 1 > /dev/null 2>&1
  echo "stages $st:"; python tools/ncu_seq.py /tmp/seq_$st.csv | grep "pgemm" | head -3
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2t_bench_$st.json 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/r2t_bench_$st.json'));print('bench', round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phase_ms'].items()}, round(d['roofline']['frac'],4))"
done
rm -f paper_2110_04393_b200/csrc/build/pgemm.o
