# warp tile width re-sweep at HEAD (TETPROJ_TILE_W: 8 default, 4, 16)
mkdir -p gpurun_out
for c in c3 c5 c2; do for tw in 8 4 16 8; do
  TETPROJ_TILE_W=$tw timeout 900 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 > gpurun_out/tw_${c}_$tw.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/tw_${c}_$tw.json').read().strip().splitlines()[-1]); k=d['kernel_ms_per_step']
print('$c tw$tw', '%.4e'%d['value'], 'fwd %.2f back %.2f'%(k['forward'],k['backward']))"
done; done
