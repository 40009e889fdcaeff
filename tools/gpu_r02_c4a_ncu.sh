# ncu of c4a's exact-heavy walks (the shape its timed steps run: 4 blocks/SM, record walk)
mkdir -p gpurun_out
R=/tmp/c4a_ncu; mkdir -p $R
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k 'regex:trace_kernel<.bool.0, .int.2, .int.2, .int.4' -s 0 -c 1 -o $R/f -f python bench.py --config c4a --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 3 > gpurun_out/c4a_ncu_fwd.log 2>&1; echo "fwd $?"
python tools/ncu_summary.py $R/f.ncu-rep "c4a forward walk, exact-heavy shape (record walk, 4 blocks/SM, kept ray), all 16 angles" > gpurun_out/head_ncu_c4a_fwd_summary.json
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k 'regex:trace_kernel<.bool.1, .int.2, .int.2, .int.4' -s 0 -c 1 -o $R/b -f python bench.py --config c4a --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 3 > gpurun_out/c4a_ncu_back.log 2>&1; echo "back $?"
python tools/ncu_summary.py $R/b.ncu-rep "c4a backward walk, exact-heavy shape (record walk, 4 blocks/SM, kept ray), all 16 angles" > gpurun_out/head_ncu_c4a_back_summary.json
