# final round-2 bench lines at HEAD (the driver's default command first)
mkdir -p gpurun_out
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/fb_c3.json 2> gpurun_out/fb_c3.err; echo "c3 $?"
timeout 1500 python bench.py --config c5 --steps 5 > gpurun_out/fb_c5.json 2> gpurun_out/fb_c5.err; echo "c5 $?"
timeout 900 python bench.py --config c5 --angles 90 --steps 5 --no-cpu-baseline > gpurun_out/fb_c5_rank90.json 2> gpurun_out/fb_c5_rank90.err; echo "c5/90 $?"
for cfg in c2 c4a c4b; do
  timeout 900 python bench.py --config $cfg > gpurun_out/fb_$cfg.json 2> gpurun_out/fb_$cfg.err; echo "$cfg $?"
done
timeout 900 python bench.py --impl reference --steps 3 > gpurun_out/fb_ref.json 2> gpurun_out/fb_ref.err; echo "ref $?"
TETPROJ_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config c2 --steps 3 > gpurun_out/fb_two_rank_c2.json 2> gpurun_out/fb_two_rank_c2.err; echo "two-rank $?"
bash tools/gpu_variants.sh bone fsep
