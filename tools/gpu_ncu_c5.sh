# ncu --set full of the first c5 walk launches (forward and backward, band order)
set -x
mkdir -p gpurun_out
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 0 -c 6 \
  -o gpurun_out/ncu_c5_full python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
  > gpurun_out/ncu_c5.log 2>&1; echo "ncu exit $?"
tail -5 gpurun_out/ncu_c5.log
ls -la gpurun_out
