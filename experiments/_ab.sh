timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "c1 or c2_ball or lattice or c3_graded or c4 or wide" > gpurun_out/gpu_tests.log 2>&1; echo tests=$? > gpurun_out/status.txt
for V in v3 v4; do TETPROJ_LIB_VARIANT=$V timeout 300 python bench.py --config c3 --no-cpu-baseline --e2e-steps 0 --steps 3 > gpurun_out/ab_$V.log 2>&1; done
CMD="python bench.py --config c3 --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 3"
$CMD > gpurun_out/prof_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 2 -c 1 -o gpurun_out/prof_v4b $CMD > gpurun_out/prof_ncu.log 2>&1
echo rc=$? >> gpurun_out/status.txt
