# full GPU check: every -m gpu test, smoke, the default bench line, the reference arm
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/check_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/check_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/check_smoke.log 2>&1; echo "smoke $?"; tail -1 gpurun_out/check_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/check_bench_c3.json 2> gpurun_out/check_bench_c3.err; echo "bench $?"
tail -c 600 gpurun_out/check_bench_c3.json
