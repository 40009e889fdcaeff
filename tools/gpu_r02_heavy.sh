# exact-heavy shape: record walk + kept ray (default) vs FT16 walk + kept ray vs no kept ray
mkdir -p gpurun_out
TETPROJ_LIB_VARIANT=heavyft timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c4a or heavy or lattice or sliver or degenerate or vertices" > gpurun_out/heavyft_tests.log 2>&1; echo "tests $?"; tail -2 gpurun_out/heavyft_tests.log
for i in 1 2; do CFG=c4a bash tools/gpu_variants.sh heavyft nokeep; done
