# last round-2 check at HEAD: GPU suite, smoke, all bench lines
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/last_gpu_tests.log 2>&1; echo "GPU_TESTS_EXIT $?" >> gpurun_out/last_gpu_tests.log
tail -2 gpurun_out/last_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/last_smoke.txt 2>&1; tail -1 gpurun_out/last_smoke.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/last_c3.json 2> gpurun_out/last_c3.err; echo "c3 $?"
timeout 1500 python bench.py --config c5 --steps 5 > gpurun_out/last_c5.json 2> gpurun_out/last_c5.err; echo "c5 $?"
timeout 900 python bench.py --config c5 --angles 90 --steps 5 --no-cpu-baseline > gpurun_out/last_c5_rank90.json 2> gpurun_out/last_c5_rank90.err; echo "c5/90 $?"
for cfg in c2 c4a c4b; do
  timeout 900 python bench.py --config $cfg > gpurun_out/last_$cfg.json 2> gpurun_out/last_$cfg.err; echo "$cfg $?"
done
timeout 900 python bench.py --impl reference > gpurun_out/last_ref.json 2> gpurun_out/last_ref.err; echo "ref $?"
TETPROJ_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config c2 --steps 3 > gpurun_out/last_two_rank_c2.json 2> gpurun_out/last_two_rank_c2.err; echo "two-rank $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/last_launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/last_launches_c3.log 2>&1; echo "launches $?"
