# round-2 evidence at HEAD: GPU suite, smoke, bench c3 (full line) + c5, launch list,
# ncu --set full of the walks on c3 and c5, the fp study with the MT oracle
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/gpu_tests.log 2>&1; echo "GPU_TESTS_EXIT $?" >> gpurun_out/gpu_tests.log
tail -4 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/ev_bench_c3.json 2> gpurun_out/ev_bench_c3.err; echo "bench c3 $?"
timeout 1500 python bench.py --config c5 --steps 3 > gpurun_out/ev_bench_c5.json 2> gpurun_out/ev_bench_c5.err; echo "bench c5 $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ev_launches_c3.log 2>&1; echo "launches $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 0 -c 3 -o gpurun_out/ev_ncu_c3 -f python bench.py --config c3 --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 3 > gpurun_out/ev_ncu_c3.log 2>&1; echo "ncu c3 $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 0 -c 1 -o gpurun_out/ev_ncu_c5_fwd -f python bench.py --config c5 --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 3 > gpurun_out/ev_ncu_c5_fwd.log 2>&1; echo "ncu c5 fwd $?"
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:trace_kernel<.bool.1' -s 0 -c 1 -o gpurun_out/ev_ncu_c5_back -f python bench.py --config c5 --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 3 > gpurun_out/ev_ncu_c5_back.log 2>&1; echo "ncu c5 back $?"
timeout 1800 python tests/campaigns/fp_study.py > gpurun_out/fp_study.out 2>&1; echo "fp study $?"
