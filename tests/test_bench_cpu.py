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
    for cfg in ("c2", "c3", "c4b", "c5", "c4a"):
        for k in ("forward", "backward"):
            per = table[cfg][k]["dram_bytes_per_crossing"]
            assert 0 < per < 96            # below the no-reuse sector traffic
            assert bench.ncu_traffic(cfg, k, 1e9) == pytest.approx(per * 1e9)
    assert bench.ncu_traffic("c1", "backward", 1e9) is None    # no capture: null, not a guess


def test_gpus_flag_fails_loudly_without_the_gpus():
    """`bench.py --gpus 2` outside torchrun re-launches itself with 2 ranks --
    and refuses (non-zero exit, message) on a node with fewer GPUs."""
    r = _run({}, "--gpus", "2", "--steps", "1", "--warmup", "3", "--no-cpu-baseline")
    assert r.returncode != 0
    assert "needs 2 GPUs" in r.stderr


def test_rank_workload_weak_and_strong():
    sys.path.insert(0, ROOT)
    import bench
    # weak: every rank traces A angles of a ws*A scan
    w, full, g0, _ = bench.rank_workload("c2", 0, 4, 10, "weak")
    assert full.n_angles == 40 and g0.n_angles == 10
    # strong: the config's scan (or --angles total) split over the ranks
    w, full, g1, _ = bench.rank_workload("c2", 1, 4, None, "strong")
    assert full.n_angles == 90 and g1.n_angles in (22, 23)
    n = sum(bench.rank_workload("c2", r, 4, 90, "strong")[2].n_angles for r in range(4))
    assert n == 90


def test_roofline_fields_recompute_from_profiles():
    """Every roofline number follows from the live launch time and a file in
    profiles/: issue rate = warp instructions per crossing (ncu_issue.json) x
    crossings per launch / launch time, against SMs x 4 x clock."""
    sys.path.insert(0, ROOT)
    import bench
    iss = json.load(open(os.path.join(ROOT, "profiles", "ncu_issue.json")))["c3"]["backward"]
    rl = bench.roofline("c3", "backward", 3.0e9, 20.0, 1965.0)
    assert rl["bound"] == "issue" and rl["unit"] == "warp-inst/s"
    want = iss["warp_inst_per_crossing"] * 3.0e9 / 20e-3
    assert rl["achieved"] == pytest.approx(want)
    assert rl["peak"] == pytest.approx(bench.sm_count() * 4 * 1965e6)
    assert rl["frac"] == pytest.approx(want / rl["peak"])
    assert rl["hbm"]["achieved"] == pytest.approx(36 * 3.0e9 / 20e-3 / 1e9)
    # no capture for the config: the HBM view, labelled as such
    rl2 = bench.roofline("c1", "forward", 1e9, 10.0, 1965.0)
    assert rl2["bound"] == "hbm" and rl2["unit"] == "GB/s"


def test_reference_arm_config_matches_our_keys():
    r = _run({}, "--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "3")
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    for k in ("workload", "tets", "angles_total", "angles_per_gpu", "detector", "rays_per_step",
              "parallelism", "scaling"):
        assert k in d["config"], k
    assert d["config"]["rays_per_step"] == 4 * 8 * 8
