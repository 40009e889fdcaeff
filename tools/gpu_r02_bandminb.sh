mkdir -p gpurun_out
for i in 1 2; do CFG=c5 bash tools/gpu_variants.sh bb8 bb7 bb6 bb8g2 bb8g8; done
