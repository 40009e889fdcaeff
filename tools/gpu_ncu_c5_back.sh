# ncu --set full of the first two c5 backward walk launches
set -x
mkdir -p gpurun_out
timeout 2400 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:trace_kernel<.bool.1' -s 0 -c 2 \
  -o gpurun_out/ncu_c5_back python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
  > gpurun_out/ncu_c5_back.log 2>&1; echo "ncu exit $?"
grep PROF gpurun_out/ncu_c5_back.log | tail -5
