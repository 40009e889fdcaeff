# A/B of the FT16 walk (default) vs the 32-B-record walk (TETPROJ_WALKER=rec):
# parity subset, bench c3 both ways, ncu --set full of the FT16 walks on c3
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "not full_size and not debug_build" > gpurun_out/ab_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/ab_tests.log
tail -3 gpurun_out/ab_tests.log
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_ft_c3.json 2> gpurun_out/ab_ft_c3.err; echo "ft $?"
TETPROJ_WALKER=rec timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_rec_c3.json 2> gpurun_out/ab_rec_c3.err; echo "rec $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 0 -c 3 -o gpurun_out/ncu_ft_c3 -f python bench.py --config c3 --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 3 > gpurun_out/ncu_ft_c3.log 2>&1; echo "ncu $?"
