# empty-block early exit: parity subset, then A/B (default = exit) on c3, c2, c4a, c5
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_plan.py -m gpu -x -q > gpurun_out/exit_tests.log 2>&1; echo "tests $?"; tail -2 gpurun_out/exit_tests.log
for c in c3 c2 c4a c5; do CFG=$c bash tools/gpu_variants.sh noexit; done
CFG=c3 bash tools/gpu_variants.sh noexit
