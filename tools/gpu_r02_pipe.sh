# host-buffer pipeline chunk floor: c2 / c4a / c3 e2e at forced chunk sizes
mkdir -p gpurun_out
for c in c2 c4a; do
  for L in 0 19 20 21 22; do
    TETPROJ_PIPE_CHUNK_LOG=$L timeout 600 python bench.py --config $c --no-cpu-baseline --steps 5 --e2e-steps 5 > gpurun_out/pipe_${c}_$L.json 2> gpurun_out/pipe_${c}_$L.err; echo "$c $L $?"
  done
done
python - <<'PY'
import json
for c in ["c2", "c4a"]:
    for L in [0, 19, 20, 21, 22]:
        try:
            d = json.loads(open(f"gpurun_out/pipe_{c}_{L}.json").read().strip().splitlines()[-1])
            print(f"{c} log{L:2d} value {d['value']:.4e} e2e {d['e2e']['value']:.4e}")
        except Exception as e:
            print(c, L, "FAILED", e)
PY
