"""bench.py host-side contract (CPU only): the reference arm's JSON line, its
rank handling under a multi-rank launch, and the per-config ncu traffic table
behind roofline.traffic."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _build(oracle_lib):
    return oracle_lib


def _run(env_extra, *args):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                          cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)


def test_reference_arm_line():
    r = _run({}, "--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "3")
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["higher_is_better"] is True
    assert d["unit"] == "tet-crossings/s" and d["value"] > 0
    assert d["steps"] == 2 and d["warmup"] == 3 and d["vs_baseline"] is None
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_exit_silently():
    r = _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"},
             "--impl", "reference", "--config", "c1", "--gpus", "2")
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""


def test_ncu_traffic_per_config():
    sys.path.insert(0, ROOT)
    import bench
    table = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    for cfg in ("c3", "c5"):
        for k in ("forward", "backward"):
            per = table[cfg][k]["dram_bytes_per_crossing"]
            assert 0 < per < 96            # below the no-reuse sector traffic
            assert bench.ncu_traffic(cfg, k, 1e9) == pytest.approx(per * 1e9)
    assert bench.ncu_traffic("c2", "backward", 1e9) is None   # no capture: null, not a guess
