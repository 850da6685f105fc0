# ncu --set full of the two-sided path's dominant kernel (phase-1 W GEMM with the right sketch, rho = 192)
mkdir -p gpurun_out
timeout 600 python bench.py --algo two_sided --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/plain_2s.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:dgemm_kernel<.int.64, .int.64, .int.16, .int.2, .int.2, .int.4, .bool.0, .bool.1>" -s 20 -c 1 -o gpurun_out/prof_w2s -f python bench.py --algo two_sided --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_w2s.log 2>&1; echo "ncu rc=$?"
