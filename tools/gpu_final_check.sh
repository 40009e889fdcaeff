# round-end sanity: default bench line (c3, with cpu_baseline), c5 line, reference arm, smoke
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err; echo "bench c3 $?"
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/final_c5.json 2> gpurun_out/final_c5.err; echo "bench c5 $?"
timeout 300 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "bench ref $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')"
