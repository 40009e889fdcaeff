# warp-level early exit + axis vote (no block barrier): parity on the variant, A/B
mkdir -p gpurun_out
TETPROJ_LIB_VARIANT=wvote timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q > gpurun_out/wvote_tests.log 2>&1; echo "tests $?"; tail -2 gpurun_out/wvote_tests.log
for c in c3 c4b c5 c2; do CFG=$c bash tools/gpu_variants.sh wvote; done
CFG=c3 bash tools/gpu_variants.sh wvote
