#!/usr/bin/env python
"""Benchmark: tet-crossings/s of one hot-path step (forward projection +
backprojection [+ all-reduce]) of the tetrahedral CT operator of
arXiv:1908.06909 on B200, per BASELINE.json's metric.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl reference]

One JSON line on rank 0.  A step = tet_project(mu) + tet_backproject(y) over
the rank's angles (weak scaling: every rank owns the same number of angles of
an N-times-denser circular scan; the backprojection is all-reduced over NCCL).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "tet-crossings/s (fwd+back step)"
BYTES_FWD = 52   # gathered bytes per crossing, forward
BYTES_BACK = 56  # gathered bytes per crossing, backward with f64 accumulator
# compulsory bytes per crossing: apex id + coords + exit id + mu
# forward; + f64 accumulator read-modify-write backward
COMPULSORY_FWD = 24
COMPULSORY_BACK = 36


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--angles", type=int, default=None, help="angles per rank (default: config)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def rank_workload(cfg, rank, ws, angles_per_rank=None):
    """Weak scaling: the full scan has ws*A equidistant angles and rank r owns
    angles r::ws (paper_1908_06909_b200.dist.AngleSharding).  Returns the
    workload, the FULL geometry, the rank's geometry and its detector rows."""
    from paper_1908_06909_b200.dist import AngleSharding
    from workloads import configs as CF
    w = CF.workload(cfg)
    A = angles_per_rank or w.geom.n_angles
    if cfg in ("c2", "c3", "c4b", "c5"):
        full = CF.workload(cfg, n_angles=A * ws).geom
    else:
        full = w.geom.subset(np.arange(min(A, w.geom.n_angles)))
    sh = AngleSharding(full.n_angles, rank, ws)
    geom = full.subset(sh.local_angles())
    y = CF.uniform_y(geom, 1000 + rank)
    return w, full, geom, y


class ClockSampler:
    """nvidia-smi sampling during the timed region (clocks + throttle reasons)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []      # (monotonic time, fields)
        self.proc = None
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # the sampler is live before the timed region starts
            deadline = time.monotonic() + 5.0
            while not self.rows and time.monotonic() < deadline:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        self.t0 = time.monotonic()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.monotonic(), [x.strip() for x in line.split(",")]))

    def stop(self):
        """End of the timed region: wait for the sample that covers it (a
        region shorter than the 50-ms period still gets one)."""
        self.t1 = time.monotonic()
        deadline = self.t1 + 1.0
        while self.proc and time.monotonic() < deadline and \
                not any(t >= self.t1 for t, _ in self.rows):
            time.sleep(0.01)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        t1 = self.t1 if self.t1 is not None else time.monotonic()
        # samples inside the timed region, plus the one that closes it
        inside = [r for t, r in self.rows if self.t0 <= t <= t1]
        after = [r for t, r in self.rows if t > t1][:1]
        rows = inside + after
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[4:8]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows), "samples_inside": len(inside)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def l2_gather_peak():
    """Measured random 32-B gather rate from L2 (experiments/microbench.py,
    profiles/r01_microbench.json): the second denominator of SURVEY §8(d)."""
    try:
        return float(json.load(open(os.path.join(ROOT, "profiles", "r01_microbench.json")))
                     ["gather32_L2_GBps"])
    except Exception:
        return None


def ncu_traffic(config, kernel, crossings_per_launch):
    """DRAM bytes per launch of the walk kernel: ncu's dram__bytes_read.sum +
    dram__bytes_write.sum per crossing (profiles/ncu_traffic.json, from one
    `ncu --set full` capture of this bench's launches of `config`) x
    crossings/launch; None for a config without a capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        per = json.load(open(p))[config][kernel]["dram_bytes_per_crossing"]
        return per * crossings_per_launch
    except Exception:
        return None


def cpu_baseline(w, geom, y, budget_s=15.0):
    """The oracle as it stands, on this host's cores, on a bounded sample of
    the same scan: an evenly strided subset of ray ids (all angles), sized
    from a short calibration run to ~budget_s seconds of fwd+back work."""
    from oracle import tetref as O
    om = O.OracleMesh.from_mesh(w.mesh)
    cores = len(os.sched_getaffinity(0))
    mu = w.mu.astype(np.float64)
    yflat = y.reshape(-1)

    def run(n):
        ids = np.linspace(0, geom.n_rays - 1, n).round().astype(np.int64)
        t0 = time.perf_counter()
        _, st = O.project(om, geom, mu, ray_ids=ids, nthreads=cores)
        _, st2 = O.backproject(om, geom, yflat[ids], ray_ids=ids, nthreads=cores)
        return time.perf_counter() - t0, st["crossings"] + st2["crossings"], n

    dt, cross, n = run(20000)
    n2 = int(min(geom.n_rays, max(20000, 20000 * budget_s / max(dt, 1e-3))))
    dt, cross, n = run(n2)
    return {"value": cross / dt, "unit": "tet-crossings/s", "cores": cores, "kind": "oracle",
            "sample": f"{n} of {geom.n_rays} rays (evenly strided over all angles), "
                      f"fwd+back, {dt:.1f} s", "crossings": int(cross), "seconds": dt}


def run_reference(args):
    """--impl reference: the oracle (CPU, host cores) timed on the same config."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    w, _, geom, y = rank_workload(args.config, 0, 1, args.angles)
    from oracle import tetref as O
    om = O.OracleMesh.from_mesh(w.mesh)
    cores = len(os.sched_getaffinity(0))
    n_ang = 2
    times, cross = [], []
    for step in range(args.warmup + args.steps):
        idx = np.array([(step * 37) % geom.n_angles, (step * 37 + 180) % geom.n_angles])
        sub = geom.subset(idx)
        t0 = time.perf_counter()
        _, st = O.project(om, sub, w.mu.astype(np.float64), nthreads=cores)
        _, st2 = O.backproject(om, sub, y[idx], nthreads=cores)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
            cross.append(st["crossings"] + st2["crossings"])
    value = sum(cross) / sum(times)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tet-crossings/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {w.desc}", "tets": w.mesh.n_tets,
                       "reference_step": f"{n_ang} of {geom.n_angles} angles per step"},
            "cpu_baseline": {"value": value, "unit": "tet-crossings/s", "cores": cores,
                             "kind": "oracle",
                             "sample": f"{n_ang} angles x {geom.n_v}x{geom.n_u} pixels per step"},
            "e2e": {"value": value, "unit": "tet-crossings/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    from paper_1908_06909_b200 import tetproj as T
    from paper_1908_06909_b200.dist import dist_backproject

    ws, rank, local = dist_env()
    # one process per GPU over NCCL; TETPROJ_DIST_BACKEND=gloo (testing the
    # multi-rank logic with several ranks on one GPU) maps ranks onto devices
    backend = os.environ.get("TETPROJ_DIST_BACKEND", "nccl")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if ws > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    if ws > 1 and rank != 0:
        dist.barrier()                      # rank 0 builds the mesh cache first
    w, full_geom, geom, y_np = rank_workload(args.config, rank, ws, args.angles)
    if ws > 1 and rank == 0:
        dist.barrier()
    torch.cuda.synchronize()
    t_create = time.perf_counter()
    tm = T.TetMesh.from_mesh(w.mesh, device=local)   # validate, snap, reorder, upload
    t_create = time.perf_counter() - t_create
    h = tm.handle
    mu = torch.from_numpy(w.mu).to(dev)
    y = torch.from_numpy(y_np).to(dev)
    proj = torch.empty((geom.n_angles, geom.n_v, geom.n_u), dtype=torch.float32, device=dev)
    x = torch.empty(w.mesh.n_tets, dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    # untimed: stats of one step (crossing counts are deterministic per geometry)
    st_f = T.tet_project(h, geom, mu, proj, stats=True)
    st_b = T.tet_backproject(h, geom, y, x, stats=True)
    assert st_f["lost"] == st_f["stuck"] == st_f["entry_conflicts"] == 0, st_f
    assert st_b["lost"] == st_b["stuck"] == 0, st_b

    def backward():
        if ws > 1:   # local A_r^T y_r, then all_reduce(SUM) over NCCL
            dist_backproject(tm, full_geom, y,
                             backproject=lambda g, yl: (T.tet_backproject(h, g, yl, x), x)[1])
        else:
            T.tet_backproject(h, geom, y, x)

    def step():
        T.tet_project(h, geom, mu, proj)
        backward()

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    T.tet_set_kernel_timing(h, True)
    T.tet_kernel_times(h)  # reset
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            flush.zero_()                    # L2 flush between timed steps (not timed)
            ev[i][0].record(stream)
            T.tet_project(h, geom, mu, proj)
            ev[i][1].record(stream)
            backward()
            ev[i][2].record(stream)
        torch.cuda.synchronize()
        clocks.stop()
        if ws > 1:
            dist.barrier()
    T.tet_set_kernel_timing(h, False)
    kt = T.tet_kernel_times(h)
    ms_f = [a.elapsed_time(b) for a, b, c in ev]
    ms_b = [b.elapsed_time(c) for a, b, c in ev]
    ms_step = [f + b for f, b in zip(ms_f, ms_b)]
    t_local = sum(ms_step) / 1e3
    crossings_local = (st_f["crossings"] + st_b["crossings"]) * args.steps
    vals = torch.tensor([t_local, sum(ms_f) / 1e3, sum(ms_b) / 1e3, crossings_local,
                         st_f["crossings"], st_b["crossings"], geom.n_rays, st_f["rays_hit"],
                         st_f["lost"] + st_b["lost"], st_f["stuck"] + st_b["stuck"],
                         st_f["exact_fallbacks"] + st_b["exact_fallbacks"]],
                        dtype=torch.float64, device=dev)
    if ws > 1:
        mx = vals[:3].clone()
        sm = vals[3:].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        vals = torch.cat([mx, sm])
    (t_max, tf_max, tb_max, cross_all, cf_all, cb_all, rays_all, hit_all, lost_all, stuck_all,
     exact_all) = vals.tolist()

    # ---- e2e: same metric through the public API with HOST buffers ----
    mu_h = torch.from_numpy(w.mu).pin_memory()
    y_h = torch.from_numpy(y_np).pin_memory()
    proj_h = torch.empty(proj.shape, dtype=torch.float32).pin_memory()
    x_h = torch.empty(x.shape, dtype=torch.float32).pin_memory()
    e2e_ms = []
    for i in range(args.e2e_steps + 1 if args.e2e_steps > 0 else 0):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        T.tet_project(h, geom, mu_h.numpy(), proj_h.numpy(), stream=stream.cuda_stream)
        T.tet_backproject(h, geom, y_h.numpy(), x_h.numpy(), stream=stream.cuda_stream)
        if ws > 1:
            xd = x_h.to(dev, non_blocking=True)
            dist.all_reduce(xd)
            x_h.copy_(xd)
        b.record(stream)
        torch.cuda.synchronize()
        if i > 0:
            e2e_ms.append(a.elapsed_time(b))
    e2e_t = torch.tensor([max(sum(e2e_ms), 1e-9) / 1e3], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = (cf_all + cb_all) * len(e2e_ms) / e2e_t.item() if e2e_ms else None

    if rank == 0:
        peak, peak_src = measured_peaks()
        tf, nf = kt["forward"]
        tb, nb = kt["backward"]
        te, ne = kt["entry"]
        tp, np_ = kt["permute"]
        per_launch_f = tf / max(nf, 1)
        per_launch_b = tb / max(nb, 1)
        # dominant kernel: the walk with the larger share of the step
        if tb >= tf:
            dom, bytes_unit, cross_unit, launches, tdom = "backward", BYTES_BACK, st_b["crossings"], nb, tb
        else:
            dom, bytes_unit, cross_unit, launches, tdom = "forward", BYTES_FWD, st_f["crossings"], nf, tf
        comp_unit = COMPULSORY_BACK if dom == "backward" else COMPULSORY_FWD
        l2pk = l2_gather_peak()
        algo_bytes_per_launch = bytes_unit * cross_unit / max(launches // args.steps, 1)
        achieved = algo_bytes_per_launch / (tdom / max(launches, 1) / 1e3) / 1e9
        achieved_c = achieved * comp_unit / bytes_unit
        # each timed entry region launches two kernels (setup + raster)
        n_launch_step = (nf + nb + 2 * ne + np_) / args.steps
        clk = clocks.summary()
        line = {
            "metric": METRIC,
            "value": cross_all / t_max,
            "unit": "tet-crossings/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": 1e3 * t_max / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: {w.desc}", "tets": w.mesh.n_tets,
                       "verts": w.mesh.n_verts, "hull_faces": w.mesh.n_bfaces,
                       "angles_per_gpu": geom.n_angles, "detector": [geom.n_v, geom.n_u],
                       "rays_per_step": int(rays_all), "parallelism": f"angles x{ws}",
                       "l2": "flushed between timed steps (256 MiB write, untimed)"},
            "fwd": {"crossings_per_s": cf_all * args.steps / tf_max,
                    "mrays_per_s": rays_all * args.steps / tf_max / 1e6,
                    "ms": 1e3 * tf_max / args.steps, "crossings": int(cf_all)},
            "back": {"crossings_per_s": cb_all * args.steps / tb_max,
                     "mrays_per_s": rays_all * args.steps / tb_max / 1e6,
                     "ms": 1e3 * tb_max / args.steps, "crossings": int(cb_all)},
            "rays_hit": int(hit_all), "lost": int(lost_all), "stuck": int(stuck_all),
            "exact_fallbacks_per_step": int(exact_all),
            "kernel_ms_per_step": {k: v[0] / args.steps for k, v in kt.items()},
            "mesh_create_s": t_create,
            "roofline": {"bound": "hbm", "kernel": f"trace_kernel<{dom}>",
                         "achieved": achieved_c, "peak": peak, "unit": "GB/s",
                         "frac": achieved_c / peak, "peak_source": peak_src,
                         "bytes_per_crossing": comp_unit,
                         "traffic": ncu_traffic(args.config, dom,
                                                cross_unit / max(launches // args.steps, 1)),
                         "per_launch_ms": per_launch_b if dom == "backward" else per_launch_f,
                         "note": "compulsory bytes per crossing (SURVEY 8(d)) x crossings per "
                                 "step / busy time of the walk-kernel class per step (union of its "
                                 "launch intervals, CUDA events on the launching streams: angle "
                                 "chunks alternate between two streams and may overlap); "
                                 "per_launch_ms = busy time / launches.  ncu DRAM traffic per "
                                 "crossing: c3 0.27 fwd / 0.22 back (L2-resident); c5 0.30 fwd "
                                 "(band order keeps a mesh slab in L2 across angles) / 2.9 back "
                                 "(0.39 TB/s, 6 % of HBM) within 3 % of c3's crossing rate: the walk "
                                 "is latency/issue-bound, not bandwidth-bound (DESIGN.md 5, "
                                 "Roofline); traffic = that per-crossing figure x crossings/launch",
                         "gathered_bytes_per_crossing": bytes_unit,
                         "gathered_achieved": achieved,
                         "gathered_frac": achieved / peak,
                         "l2_gather_peak_gbs": l2pk,
                         "l2_gather_frac": achieved / l2pk if l2pk else None},
            "e2e": {"value": e2e_value, "unit": "tet-crossings/s",
                    "h2d_bytes_per_step": int(w.mu.nbytes + y_np.nbytes),
                    "d2h_bytes_per_step": int(proj.numel() * 4 + x.numel() * 4)},
            "gpu_launches": int(round(n_launch_step * args.steps)),
            "clocks": clk,
        }
        if not args.no_cpu_baseline and ws == 1:
            line["cpu_baseline"] = cpu_baseline(w, geom, y_np)
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
