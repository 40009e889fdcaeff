# FT16 (default) vs rec walk on the other configs: c5 (HBM-resident), c2, c4b, c4a
mkdir -p gpurun_out
for cfg in c2 c4b c4a c5; do
  st=5; [ $cfg = c5 ] && st=3
  timeout 1200 python bench.py --config $cfg --steps $st --no-cpu-baseline --e2e-steps 0 > gpurun_out/abc_ft_$cfg.json 2> gpurun_out/abc_ft_$cfg.err; echo "ft $cfg $?"
  TETPROJ_WALKER=rec timeout 1200 python bench.py --config $cfg --steps $st --no-cpu-baseline --e2e-steps 0 > gpurun_out/abc_rec_$cfg.json 2> gpurun_out/abc_rec_$cfg.err; echo "rec $cfg $?"
done
python - <<'PY'
import json
for cfg in ("c2", "c4b", "c4a", "c5"):
    for w in ("ft", "rec"):
        try:
            d = json.loads(open(f"gpurun_out/abc_{w}_{cfg}.json").read().strip().splitlines()[-1])
            k = d["kernel_ms_per_step"]
            print(f"{cfg} {w:4s} {d['value']:.4e} fwd {k['forward']:.2f} back {k['backward']:.2f} entry {k['entry']:.2f} lost {d['lost']} stuck {d['stuck']}")
        except Exception as e:
            print(cfg, w, "FAILED", e)
PY
