# ncu --set full of specific launches: PROF_SPECS="name|regex|skip|count;..."  on reduced C5 (d=6)
mkdir -p gpurun_out
timeout 300 python tools/run_once.py large ${PD:-6} 1 > gpurun_out/plain.log 2>&1 || { echo plain failed; exit 1; }
IFS=';' read -ra SPECS <<< "$PROF_SPECS"
for spec in "${SPECS[@]}"; do
  IFS='|' read -r name rgx skip count <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$rgx" -s $skip -c $count -o gpurun_out/prof_$name -f python tools/run_once.py large ${PD:-6} 1 > gpurun_out/ncu_$name.log 2>&1
  echo "ncu $name rc=$?"
done
