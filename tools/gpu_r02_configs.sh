# bench lines for the other configs at HEAD, the 2-rank logic check (gloo, one
# GPU) and the per-rank work of the north-star 8-GPU c5 strong-scaling run
mkdir -p gpurun_out
for cfg in c2 c4a c4b; do
  timeout 900 python bench.py --config $cfg > gpurun_out/cf_bench_$cfg.json 2> gpurun_out/cf_bench_$cfg.err; echo "bench $cfg $?"
done
TETPROJ_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config c2 --steps 3 > gpurun_out/cf_two_rank_c2.json 2> gpurun_out/cf_two_rank_c2.err; echo "two-rank $?"
timeout 900 python bench.py --config c5 --angles 90 --steps 5 --no-cpu-baseline > gpurun_out/cf_c5_rank90.json 2> gpurun_out/cf_c5_rank90.err; echo "c5 per-rank $?"
