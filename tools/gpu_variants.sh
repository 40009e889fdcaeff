# bench c3 for the default library and each named variant (tools/build_variants.py)
# usage: bash tools/gpu_variants.sh [config] v1 v2 ...
mkdir -p gpurun_out
cfg=${CFG:-c3}
timeout 600 python bench.py --config $cfg --no-cpu-baseline --e2e-steps 0 > gpurun_out/var_default_$cfg.json 2> gpurun_out/var_default_$cfg.err; echo "default $?"
for v in "$@"; do
  TETPROJ_LIB_VARIANT=$v timeout 600 python bench.py --config $cfg --no-cpu-baseline --e2e-steps 0 > gpurun_out/var_${v}_$cfg.json 2> gpurun_out/var_${v}_$cfg.err; echo "$v $?"
done
python - "$cfg" "$@" <<'PY'
import json, sys
cfg = sys.argv[1]
for v in ["default"] + sys.argv[2:]:
    try:
        d = json.loads(open(f"gpurun_out/var_{v}_{cfg}.json").read().strip().splitlines()[-1])
        k = d["kernel_ms_per_step"]
        print(f"{v:12s} {d['value']:.4e}  fwd {k['forward']:.2f}  back {k['backward']:.2f}  entry {k['entry']:.2f}  clk {d['clocks']['sm_mhz']}")
    except Exception as e:
        print(v, "FAILED", e)
PY
