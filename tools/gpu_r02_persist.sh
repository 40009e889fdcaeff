# L2 persisting window over the walked table (TETPROJ_L2_PERSIST=1) vs off
mkdir -p gpurun_out
for c in c3 c5; do for P in 0 1; do
  TETPROJ_L2_PERSIST=$P timeout 900 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 > gpurun_out/persist_${c}_$P.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/persist_${c}_$P.json').read().strip().splitlines()[-1]); k=d['kernel_ms_per_step']
print('$c persist$P', '%.4e'%d['value'], 'fwd %.2f back %.2f'%(k['forward'],k['backward']))"
done; done
