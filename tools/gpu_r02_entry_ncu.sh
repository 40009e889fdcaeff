# c2 entry finder: launch list + ncu --set full of the raster and setup kernels
mkdir -p gpurun_out
R=/tmp/entry_ncu; mkdir -p $R
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/entry_launches_c2.csv python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/entry_launches_c2.log 2>&1; echo "launches $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:entry_ -s 0 -c 3 -o $R/c2e -f python bench.py --config c2 --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 3 > gpurun_out/entry_ncu_c2.log 2>&1; echo "ncu $?"
python tools/ncu_summary.py $R/c2e.ncu-rep "c2 entry_setup_kernel (90 angles);c2 entry_small_kernel;c2 entry_raster_kernel" > gpurun_out/entry_ncu_c2_summary.json
ncu -i $R/c2e.ncu-rep --page source --csv --print-source sass > $R/src.csv 2>/dev/null; gzip -c $R/src.csv > gpurun_out/entry_ncu_c2_source.csv.gz
