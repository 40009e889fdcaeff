mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -k "large_single or through_plans" > gpurun_out/newtests.log 2>&1; echo "tests $?"; tail -5 gpurun_out/newtests.log
