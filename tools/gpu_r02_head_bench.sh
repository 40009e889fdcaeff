# HEAD evidence: full GPU suite, smoke, bench lines of every config, reference arm, two-rank logic
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/hb_gpu_tests.log 2>&1; echo "GPU_TESTS_EXIT $?" >> gpurun_out/hb_gpu_tests.log
tail -2 gpurun_out/hb_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/hb_smoke.txt 2>&1; tail -1 gpurun_out/hb_smoke.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/hb_c3.json 2> gpurun_out/hb_c3.err; echo "c3 $?"
timeout 1500 python bench.py --config c5 --steps 5 > gpurun_out/hb_c5.json 2> gpurun_out/hb_c5.err; echo "c5 $?"
timeout 900 python bench.py --config c5 --angles 90 --steps 5 --no-cpu-baseline > gpurun_out/hb_c5_rank90.json 2> gpurun_out/hb_c5_rank90.err; echo "c5/90 $?"
for cfg in c2 c4a c4b; do
  timeout 900 python bench.py --config $cfg > gpurun_out/hb_$cfg.json 2> gpurun_out/hb_$cfg.err; echo "$cfg $?"
done
timeout 900 python bench.py --impl reference > gpurun_out/hb_ref.json 2> gpurun_out/hb_ref.err; echo "ref $?"
TETPROJ_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config c2 --steps 3 > gpurun_out/hb_two_rank_c2.json 2> gpurun_out/hb_two_rank_c2.err; echo "two-rank $?"
for f in c3 c5 c5_rank90 c2 c4a c4b ref two_rank_c2; do python -c "
import json
d=json.loads(open('gpurun_out/hb_$f.json').read().strip().splitlines()[-1])
print('$f', '%.4g' % d.get('value'), '%.4g' % ((d.get('e2e') or {}).get('value') or 0), d.get('ms_per_step'), d.get('n_gpus'), (d.get('clocks') or {}).get('reasons'))" || echo "$f bad"; done
