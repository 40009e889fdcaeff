# plans: GPU tests, smoke, then bench with plan vs --no-plan on c2 / c3 / c4a
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_plan.py tests/test_solvers.py -m gpu -x -q > gpurun_out/plan_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/plan_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/plan_smoke.log 2>&1; echo "smoke $?"; tail -1 gpurun_out/plan_smoke.log
for c in c2 c3 c4a; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/plan_bench_$c.json 2> gpurun_out/plan_bench_$c.err; echo "$c plan $?"
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-plan > gpurun_out/noplan_bench_$c.json 2> gpurun_out/noplan_bench_$c.err; echo "$c noplan $?"
done
python - <<'PY'
import json
for c in ["c2", "c3", "c4a"]:
    for v in ["plan", "noplan"]:
        try:
            d = json.loads(open(f"gpurun_out/{v}_bench_{c}.json").read().strip().splitlines()[-1])
            k = d["kernel_ms_per_step"]
            print(f"{c} {v:7s} {d['value']:.4e} e2e {d['e2e']['value']:.4e} ms {d['ms_per_step']:.3f} entry {k['entry']:.3f} fwd {k['forward']:.2f} back {k['backward']:.2f} launches {d['gpu_launches']}")
        except Exception as e:
            print(c, v, "FAILED", e)
PY
