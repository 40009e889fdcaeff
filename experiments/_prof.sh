CMD="python bench.py --config c3 --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 3"
$CMD > gpurun_out/prof_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 4 -c 1 -o gpurun_out/prof_v3 $CMD > gpurun_out/prof_ncu.log 2>&1
echo rc=$? > gpurun_out/status.txt
