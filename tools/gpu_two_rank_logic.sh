# bench.py multi-rank path (sharding, all-reduced backprojection, max-over-ranks timing, rank-0 JSON)
# with two ranks sharing the one GPU over gloo: a logic check, not a scaling number
set -x
mkdir -p gpurun_out
TETPROJ_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --config c2 \
  > gpurun_out/two_rank_c2.json 2> gpurun_out/two_rank_c2.err; echo "two-rank exit $?"
tail -c 1500 gpurun_out/two_rank_c2.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 --config c2 \
  > gpurun_out/two_rank_ref.json 2> gpurun_out/two_rank_ref.err; echo "two-rank ref exit $?"
cat gpurun_out/two_rank_ref.json | head -c 600
