timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$? > gpurun_out/status.txt
for V in v5 v6 v7; do TETPROJ_LIB_VARIANT=$V timeout 300 python bench.py --config c3 --no-cpu-baseline --e2e-steps 0 --steps 3 > gpurun_out/ab_$V.log 2>&1; done
echo done >> gpurun_out/status.txt
