# exact-heavy shape passing the ray's grid points to the exact path: parity, A/B on c4a
mkdir -p gpurun_out
TETPROJ_LIB_VARIANT=keepray timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q > gpurun_out/keepray_tests.log 2>&1; echo "tests $?"; tail -2 gpurun_out/keepray_tests.log
for i in 1 2; do CFG=c4a bash tools/gpu_variants.sh keepray; done
