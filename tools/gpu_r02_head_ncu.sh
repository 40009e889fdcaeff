# ncu captures of the walks at HEAD (summarised on the box) + the crossings of the captured launches
set -x
mkdir -p gpurun_out
R=/tmp/head_ncu; mkdir -p $R
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 0 -c 3 -o $R/c3 -f python bench.py --config c3 --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 3 > gpurun_out/head_ncu_c3.log 2>&1; echo "ncu c3 $?"
python tools/ncu_summary.py $R/c3.ncu-rep "c3 forward walk (FT16, 8 blocks/SM), chunk 0: 256 of 360 angles;c3 forward walk, chunk 1: 104 angles;c3 backward walk (FT16, 10 blocks/SM, evict-last REDs), chunk 0: 256 angles" > gpurun_out/head_ncu_c3_summary.json
ncu -i $R/c3.ncu-rep --page source --csv --print-source sass > $R/c3_src.csv 2>/dev/null; gzip -c $R/c3_src.csv > gpurun_out/head_ncu_c3_source.csv.gz
timeout 1500 ncu --set full --clock-control none -k regex:trace_kernel -s 0 -c 1 -o $R/c5f -f python bench.py --config c5 --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 3 > gpurun_out/head_ncu_c5_fwd.log 2>&1; echo "ncu c5 fwd $?"
python tools/ncu_summary.py $R/c5f.ncu-rep "c5 forward walk (FT16, band order), launch 0: 64 of 720 angles" > gpurun_out/head_ncu_c5_fwd_summary.json
timeout 1500 ncu --set full --clock-control none --kernel-name-base demangled -k 'regex:trace_kernel<.bool.1' -s 0 -c 1 -o $R/c5b -f python bench.py --config c5 --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 3 > gpurun_out/head_ncu_c5_back.log 2>&1; echo "ncu c5 back $?"
python tools/ncu_summary.py $R/c5b.ncu-rep "c5 backward walk (FT16, band order: 8 blocks/SM, bands of 4 angles), launch 0: 64 of 720 angles" > gpurun_out/head_ncu_c5_back_summary.json
for cfg in c2 c4b; do
  timeout 900 ncu --set full --clock-control none -k regex:trace_kernel -s 0 -c 1 -o $R/${cfg}f -f python bench.py --config $cfg --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 3 > gpurun_out/head_ncu_${cfg}_fwd.log 2>&1; echo "ncu $cfg fwd $?"
  python tools/ncu_summary.py $R/${cfg}f.ncu-rep "$cfg forward walk (FT16), launch 0 (all angles)" > gpurun_out/head_ncu_${cfg}_fwd_summary.json
  timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k 'regex:trace_kernel<.bool.1' -s 0 -c 1 -o $R/${cfg}b -f python bench.py --config $cfg --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 3 > gpurun_out/head_ncu_${cfg}_back.log 2>&1; echo "ncu $cfg back $?"
  python tools/ncu_summary.py $R/${cfg}b.ncu-rep "$cfg backward walk (FT16), launch 0 (all angles)" > gpurun_out/head_ncu_${cfg}_back_summary.json
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/head_launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/head_launches_c3.log 2>&1; echo "launches $?"
du -sh gpurun_out
timeout 900 python tools/launch_crossings.py > gpurun_out/head_launch_crossings.json 2> gpurun_out/head_launch_crossings.err; echo "crossings $?"
