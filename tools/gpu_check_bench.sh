# benches c3 + c5 (full lines), then the GPU suite and smoke (used to A/B a kernel change)
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/ab_c3.json 2> gpurun_out/ab_c3.err; echo "bench c3 $?"
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/ab_c5.json 2> gpurun_out/ab_c5.err; echo "bench c5 $?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo "GPU_TESTS_EXIT $?"
tail -3 gpurun_out/ab_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')"
