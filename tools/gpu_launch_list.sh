# ncu launch list (per-launch durations) of the c3 bench command
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 \
  > gpurun_out/launches_c3.log 2>&1; echo "ncu exit $?"
wc -l gpurun_out/launches_c3.csv
