# bench lines at HEAD (plans): c5, c5 rank share, c2/c4a/c4b, reference arm, two-rank logic, launch list
mkdir -p gpurun_out
timeout 1500 python bench.py --config c5 --steps 5 > gpurun_out/pe_c5.json 2> gpurun_out/pe_c5.err; echo "c5 $?"
timeout 900 python bench.py --config c5 --angles 90 --steps 5 --no-cpu-baseline > gpurun_out/pe_c5_rank90.json 2> gpurun_out/pe_c5_rank90.err; echo "c5/90 $?"
for cfg in c2 c4a c4b; do
  timeout 900 python bench.py --config $cfg > gpurun_out/pe_$cfg.json 2> gpurun_out/pe_$cfg.err; echo "$cfg $?"
done
timeout 900 python bench.py --impl reference > gpurun_out/pe_ref.json 2> gpurun_out/pe_ref.err; echo "ref $?"
TETPROJ_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config c2 --steps 3 > gpurun_out/pe_two_rank_c2.json 2> gpurun_out/pe_two_rank_c2.err; echo "two-rank $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pe_launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pe_launches_c3.log 2>&1; echo "launches $?"
for f in c5 c5_rank90 c2 c4a c4b ref two_rank_c2; do python -c "
import json,sys
d=json.loads(open('gpurun_out/pe_$f.json').read().strip().splitlines()[-1])
print('$f', d.get('value'), (d.get('e2e') or {}).get('value'), d.get('ms_per_step'), d.get('n_gpus'))" || echo "$f bad"; done
