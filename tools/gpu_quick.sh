# quick check after a walker change: parity subset, then bench variants
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "not full_size and not debug_build" > gpurun_out/quick_tests.log 2>&1; echo "TESTS_EXIT $?" | tee -a gpurun_out/quick_tests.log
tail -2 gpurun_out/quick_tests.log
bash tools/gpu_variants.sh "$@"
