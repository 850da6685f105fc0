mkdir -p gpurun_out
python -m paper_2110_04393_b200.build > /dev/null
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 python tools/sanitize_small.py > gpurun_out/r2n_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/r2n_sanitizer_$tool.log
done
