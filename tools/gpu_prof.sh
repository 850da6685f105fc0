# ncu --set full captures of the given kernels on a reduced C5 (d=6)
mkdir -p gpurun_out
timeout 300 python tools/run_once.py large 6 1 > gpurun_out/plain.log 2>&1 && \
for k in $KERNELS; do
  timeout 600 ncu --set full --clock-control none --import-source on --warp-sampling-interval ${SAMPLING:-auto} -k regex:$k -s ${SKIP:-2} -c ${COUNT:-1} -o gpurun_out/prof_$k -f python tools/run_once.py large 6 1 > gpurun_out/ncu_$k.log 2>&1
  echo "ncu $k rc=$?"
done
