# the all-kernels small case on the bounds-checked debug library (DBG_CHECK traps)
mkdir -p gpurun_out
TETPROJ_DEBUG_LIB=1 timeout 1200 python tools/sanitize_case.py > gpurun_out/dbg_case.log 2>&1; echo "debug-lib case $?"; tail -2 gpurun_out/dbg_case.log
