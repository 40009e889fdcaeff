#!/usr/bin/env python
"""Benchmark: tet-crossings/s of one hot-path step (forward projection +
backprojection [+ all-reduce]) of the tetrahedral CT operator of
arXiv:1908.06909 on B200, per BASELINE.json's metric.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
                  [--scaling weak|strong] [--angles A] [--impl reference]

One JSON line on rank 0.  A step = tet_plan_create (geometry + the entry map
of every ray, Alg. 2 "Read initial intersection element") +
tet_plan_project(mu) + tet_plan_backproject(y) + tet_plan_destroy over the
rank's angles, the backprojection all-reduced over NCCL for N > 1 (--no-plan:
tet_project + tet_backproject, each running the entry finder itself).
--scaling weak (default): every rank owns A angles (default: the config's)
of an N*A-angle circular scan.  --scaling strong: the config's scan (or
--angles total angles) is sharded over the N ranks (north_star c5: 720
angles over 8 GPUs).  With --gpus N > 1 and no torchrun environment the
script re-launches itself under torch.distributed.run with N local ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
ISSUE_SLOTS_PER_SM = 4   # one warp instruction per SM sub-partition per cycle


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--no-plan", action="store_true",
                    help="entry finder inside each call instead of once per step")
    ap.add_argument("--angles", type=int, default=None,
                    help="weak: angles per rank; strong: total angles (default: the config's)")
    return ap.parse_args(argv)


def maybe_relaunch(args) -> None:
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-exec under
    torch.distributed.run with one rank per local GPU.  Fails loudly when the
    node has fewer than N GPUs (TETPROJ_DIST_BACKEND=gloo, the one-GPU logic
    check, maps several ranks onto one device and skips that check)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return
    if os.environ.get("TETPROJ_DIST_BACKEND", "nccl") == "nccl":
        import torch
        n = torch.cuda.device_count()
        if n < args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, "
                             f"this node has {n}\n")
            sys.exit(2)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def rank_workload(cfg, rank, ws, angles=None, scaling="weak"):
    """The full scan and this rank's share (paper_1908_06909_b200.dist.
    AngleSharding: rank r owns angles r::ws).  weak: the full scan has
    ws * A equidistant angles (A = `angles` or the config's), so every rank
    traces A angles; strong: the full scan has `angles` (or the config's)
    angles, split over the ranks.  Returns the workload, the FULL geometry,
    the rank's geometry and its detector rows."""
    from paper_1908_06909_b200.dist import AngleSharding
    from workloads import configs as CF
    w = CF.workload(cfg)
    A0 = w.geom.n_angles
    total = (angles or A0) * ws if scaling == "weak" else (angles or A0)
    if cfg in ("c2", "c3", "c4b", "c5"):
        full = CF.workload(cfg, n_angles=total).geom
    else:   # fixed direction sets (c1, c4a): at most the config's angles
        full = w.geom.subset(np.arange(min(total, A0)))
    sh = AngleSharding(full.n_angles, rank, ws)
    geom = full.subset(sh.local_angles())
    y = CF.uniform_y(geom, 1000 + rank)
    return w, full, geom, y


def config_dict(args, w, full, geom, ws):
    """The `config` object of both arms (same keys, so the driver can see
    that both did the same work)."""
    return {"workload": f"{args.config}: {w.desc}", "tets": w.mesh.n_tets,
            "verts": w.mesh.n_verts, "hull_faces": w.mesh.n_bfaces,
            "angles_total": full.n_angles, "angles_per_gpu": geom.n_angles,
            "detector": [geom.n_v, geom.n_u], "beam": "cone" if geom.beam == 0 else "parallel",
            "rays_per_step": int(full.n_rays), "parallelism": f"angles x{ws}",
            "scaling": args.scaling,
            "l2": "flushed between timed steps (256 MiB write, untimed)"}


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


def _profile_json(name):
    try:
        return json.load(open(os.path.join(ROOT, "profiles", name)))
    except Exception:
        return None


def l2_gather_peak():
    """Measured random 32-B gather rate from L2 (experiments/microbench.py,
    profiles/microbench.json, whose ncu capture shows it at the L2 limit):
    the second denominator of SURVEY §8(d)."""
    d = _profile_json("microbench.json")
    return float(d["gather32_L2_GBps"]) if d and "gather32_L2_GBps" in d else None


def ncu_traffic(config, kernel, crossings_per_launch):
    """DRAM bytes per launch of the walk kernel: ncu's dram__bytes_read.sum +
    dram__bytes_write.sum per crossing (profiles/ncu_traffic.json, from one
    `ncu --set full` capture of this bench's launches of `config`) x
    crossings/launch; None for a config without a capture."""
    d = _profile_json("ncu_traffic.json")
    try:
        return d[config][kernel]["dram_bytes_per_crossing"] * crossings_per_launch
    except Exception:
        return None


def ncu_issue(config, kernel):
    """Per-crossing ncu counters of the walk kernel (profiles/ncu_issue.json:
    smsp__inst_executed.sum / crossings of the captured launch, plus the
    capture's issue-active, L1 data-pipe and L2 throughput percentages)."""
    d = _profile_json("ncu_issue.json")
    try:
        return d[config][kernel]
    except Exception:
        return None


def sm_count():
    try:
        import torch
        return torch.cuda.get_device_properties(0).multi_processor_count
    except Exception:
        return 148


def roofline(config, dom, cross_launch, per_launch_ms, clk_mhz):
    """The dominant walk kernel against the limit that binds it.

    The walk is a dependent gather chain served from L1/L2 (DRAM traffic
    0.2-3 B per crossing, roofline.traffic), so neither HBM nor L2 bandwidth
    binds; the binding resource is warp-instruction issue: `achieved` =
    ncu warp instructions per crossing (profiles/ncu_issue.json) x crossings
    per launch / launch time (CUDA events, live), `peak` = SMs x 4 issue
    slots x the SM clock sampled during the timed region.  The bandwidth
    views (compulsory and gathered bytes against HBM, gathered bytes against
    the measured L2 gather rate) are kept beside it as context."""
    peak_hbm, peak_src = measured_peaks()
    per_launch_s = per_launch_ms / 1e3
    comp = COMPULSORY_BACK if dom == "backward" else COMPULSORY_FWD
    gath = BYTES_BACK if dom == "backward" else BYTES_FWD
    comp_gbs = comp * cross_launch / per_launch_s / 1e9
    gath_gbs = gath * cross_launch / per_launch_s / 1e9
    l2pk = l2_gather_peak()
    hbm = {"bytes_per_crossing": comp, "achieved": comp_gbs, "peak": peak_hbm, "unit": "GB/s",
           "frac": comp_gbs / peak_hbm, "peak_source": peak_src,
           "gathered_bytes_per_crossing": gath, "gathered_achieved": gath_gbs,
           "gathered_frac": gath_gbs / peak_hbm}
    l2 = {"gathered_achieved": gath_gbs, "peak": l2pk, "unit": "GB/s",
          "frac": gath_gbs / l2pk if l2pk else None,
          "peak_source": "profiles/microbench.json gather32_L2_GBps"}
    line = {"kernel": f"trace_kernel<{dom}>", "per_launch_ms": per_launch_ms,
            "crossings_per_launch": cross_launch,
            "traffic": ncu_traffic(config, dom, cross_launch),
            "traffic_note": "ncu dram__bytes_read.sum + dram__bytes_write.sum per crossing "
                            "(profiles/ncu_traffic.json) x crossings per launch",
            "hbm": hbm, "l2": l2}
    iss = ncu_issue(config, dom)
    if iss:
        sms = sm_count()
        f = (clk_mhz or 1965.0) * 1e6
        ach = iss["warp_inst_per_crossing"] * cross_launch / per_launch_s
        peak = sms * ISSUE_SLOTS_PER_SM * f
        line.update({"bound": "issue", "achieved": ach, "peak": peak, "unit": "warp-inst/s",
                     "frac": ach / peak,
                     "peak_source": f"{sms} SMs x {ISSUE_SLOTS_PER_SM} issue slots x "
                                    f"{f / 1e6:.0f} MHz (SM clock sampled in the timed region)",
                     "issue": iss})
        l2["lts_throughput_pct_ncu"] = iss.get("lts_throughput_pct")
    else:   # no capture for this config: the HBM view is the only one available
        line.update({"bound": "hbm", "achieved": comp_gbs, "peak": peak_hbm, "unit": "GB/s",
                     "frac": comp_gbs / peak_hbm, "peak_source": peak_src})
    return line


def cpu_baseline(w, geom, y, budget_s=15.0):
    """The oracle as it stands, on this host's cores, on a bounded sample of
    the same scan: an evenly strided subset of ray ids (all angles), sized
    from a short calibration run to ~budget_s seconds of fwd+back work.
    Built -O3 -march=native on this host; the oracle finds each
    ray's entering hull face by scanning every hull face, so meshes with many
    hull faces (c2: 5,944) cost it more per crossing."""
    from oracle import tetref as O
    O.use_native()
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
                      f"fwd+back, {dt:.1f} s; oracle {O.build_flags()} (brute-force hull "
                      f"scan over {w.mesh.n_bfaces} faces per ray)",
            "crossings": int(cross), "seconds": dt}


def run_reference(args):
    """--impl reference: the oracle (CPU, host cores) timed on the same
    config.  Under torchrun only rank 0 runs."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    n_gpus = max(args.gpus, ws)
    w, full, _, _ = rank_workload(args.config, 0, n_gpus, args.angles, args.scaling)
    y = np.random.default_rng(1000).uniform(0.5, 1.5, (full.n_angles, full.n_v, full.n_u)) \
        .astype(np.float32)
    from oracle import tetref as O
    O.use_native()
    om = O.OracleMesh.from_mesh(w.mesh)
    cores = len(os.sched_getaffinity(0))
    n_ang = 2
    times, cross = [], []
    for step in range(args.warmup + args.steps):
        idx = np.array([(step * 37) % full.n_angles,
                        (step * 37 + full.n_angles // 2) % full.n_angles])
        sub = full.subset(idx)
        t0 = time.perf_counter()
        _, st = O.project(om, sub, w.mu.astype(np.float64), nthreads=cores)
        _, st2 = O.backproject(om, sub, y[idx], nthreads=cores)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
            cross.append(st["crossings"] + st2["crossings"])
    value = sum(cross) / sum(times)
    cfg = config_dict(args, w, full, full.subset(np.arange(0, full.n_angles, n_gpus)), n_gpus)
    cfg["reference_step"] = (f"{n_ang} of {full.n_angles} angles per step (fwd+back), "
                             f"oracle on {cores} host cores")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tet-crossings/s",
            "n_gpus": n_gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.median(times), "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": cfg,
            "cpu_baseline": {"value": value, "unit": "tet-crossings/s", "cores": cores,
                             "kind": "oracle",
                             "sample": f"{n_ang} angles x {full.n_v}x{full.n_u} pixels per step; "
                                       f"oracle {O.build_flags()}"},
            "e2e": {"value": value, "unit": "tet-crossings/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def nccl_report(rank, log_path):
    """NCCL version and, from the INIT log of this rank, whether NVLS
    (NVSwitch in-switch reduction) was set up."""
    import torch
    try:
        v = torch.cuda.nccl.version()
        out = {"version": ".".join(str(x) for x in v) if isinstance(v, (tuple, list)) else str(v)}
    except Exception as e:   # reporting only: never fail the benchmark over it
        out = {"version": f"unknown ({type(e).__name__})"}
    try:
        txt = open(log_path).read()
        out["log"] = os.path.relpath(log_path, ROOT)
        out["nvls"] = "NVLS" in txt and "NVLS multicast support is not available" not in txt
        out["init_lines"] = sum(1 for ln in txt.splitlines() if "Init COMPLETE" in ln)
    except Exception:
        out["log"] = None
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    maybe_relaunch(args)
    import torch
    import torch.distributed as dist

    from paper_1908_06909_b200 import tetproj as T
    from paper_1908_06909_b200.dist import dist_backproject

    ws, rank, local = dist_env()
    if ws != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}\n")
        return 2
    # one process per GPU over NCCL; TETPROJ_DIST_BACKEND=gloo (testing the
    # multi-rank logic with several ranks on one GPU) maps ranks onto devices
    backend = os.environ.get("TETPROJ_DIST_BACKEND", "nccl")
    if backend == "nccl" and ws > torch.cuda.device_count():
        sys.stderr.write(f"bench.py: {ws} NCCL ranks but {torch.cuda.device_count()} GPUs\n")
        return 2
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    nccl_log = None
    if ws > 1:
        if backend == "nccl":
            if "NCCL_DEBUG" not in os.environ:   # communicator init log (NVLS or not)
                nccl_log = os.path.join(ROOT, "gpurun_out", f"nccl_init_rank{rank}.log")
                os.makedirs(os.path.dirname(nccl_log), exist_ok=True)
                os.environ.update(NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT,NVLS",
                                  NCCL_DEBUG_FILE=nccl_log)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    if ws > 1 and rank != 0:
        dist.barrier()                      # rank 0 builds the mesh cache first
    w, full_geom, geom, y_np = rank_workload(args.config, rank, ws, args.angles, args.scaling)
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

    use_plan = not args.no_plan

    def forward(mu_in, proj_out, **kw):
        """The step's first half; returns the plan (None with --no-plan)."""
        if not use_plan:
            T.tet_project(h, geom, mu_in, proj_out, **kw)
            return None
        pl = T.tet_plan_create(h, geom, stream=stream.cuda_stream)   # entry map, once per step
        T.tet_plan_project(pl, mu_in, proj_out, **kw)
        return pl

    def back_local(pl, y_in, x_out, **kw):
        if pl is None:
            T.tet_backproject(h, geom, y_in, x_out, **kw)
        else:
            T.tet_plan_backproject(pl, y_in, x_out, **kw)
            T.tet_plan_destroy(pl)          # stream-ordered free

    def backward(pl):
        if ws > 1:   # local A_r^T y_r, then all_reduce(SUM) over NCCL
            dist_backproject(tm, full_geom, y,
                             backproject=lambda g, yl: (back_local(pl, yl, x), x)[1])
        else:
            back_local(pl, y, x)

    def step():
        backward(forward(mu, proj))

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
        t_wall = time.perf_counter()
        for i in range(args.steps):
            flush.zero_()                    # L2 flush between timed steps (not timed)
            ev[i][0].record(stream)
            pl = forward(mu, proj)
            ev[i][1].record(stream)
            backward(pl)
            ev[i][2].record(stream)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
        clocks.stop()
        if ws > 1:
            dist.barrier()
    T.tet_set_kernel_timing(h, False)
    kt = T.tet_kernel_times(h)
    # per-step device times, max over ranks step by step, then the median step
    per = torch.tensor([[a.elapsed_time(b) for a, b, c in ev],
                        [b.elapsed_time(c) for a, b, c in ev]], dtype=torch.float64, device=dev)
    counts = torch.tensor([st_f["crossings"], st_b["crossings"], geom.n_rays, st_f["rays_hit"],
                           st_f["lost"] + st_b["lost"], st_f["stuck"] + st_b["stuck"],
                           st_f["exact_fallbacks"] + st_b["exact_fallbacks"]],
                          dtype=torch.float64, device=dev)
    if ws > 1:
        steps_max = (per[0] + per[1]).clone()
        dist.all_reduce(per, op=dist.ReduceOp.MAX)
        dist.all_reduce(steps_max, op=dist.ReduceOp.MAX)
        dist.all_reduce(counts, op=dist.ReduceOp.SUM)
    else:
        steps_max = per[0] + per[1]
    ms_f = per[0].tolist()
    ms_b = per[1].tolist()
    ms_step = steps_max.tolist()
    cf_all, cb_all, rays_all, hit_all, lost_all, stuck_all, exact_all = counts.tolist()
    med = statistics.median(ms_step)

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
        pl = forward(mu_h.numpy(), proj_h.numpy(), stream=stream.cuda_stream)
        back_local(pl, y_h.numpy(), x_h.numpy(), stream=stream.cuda_stream)
        if ws > 1:
            xd = x_h.to(dev, non_blocking=True)
            dist.all_reduce(xd)
            x_h.copy_(xd)
        b.record(stream)
        torch.cuda.synchronize()
        if i > 0:
            e2e_ms.append(a.elapsed_time(b))
    e2e_t = torch.tensor(e2e_ms or [0.0], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = (cf_all + cb_all) / (statistics.median(e2e_t.tolist()) / 1e3) if e2e_ms else None

    if rank == 0:
        tf, nf = kt["forward"]
        tb, nb = kt["backward"]
        te, ne = kt["entry"]
        tp, np_ = kt["permute"]
        # dominant kernel: the walk with the larger share of the step
        if tb >= tf:
            dom, cross_unit, launches, tdom = "backward", st_b["crossings"], nb, tb
        else:
            dom, cross_unit, launches, tdom = "forward", st_f["crossings"], nf, tf
        per_step_launches = max(launches // args.steps, 1)
        clk = clocks.summary()
        rl = roofline(args.config, dom, cross_unit / per_step_launches,
                      tdom / max(launches, 1), clk.get("sm_mhz"))
        # each timed entry region launches three kernels (setup, small-item
        # raster, warp raster): once per step with a plan, once per call without
        n_launch_step = (nf + nb + 3 * ne + np_) / args.steps
        line = {
            "metric": METRIC,
            "value": (cf_all + cb_all) / (med / 1e3),
            "unit": "tet-crossings/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": med,
            "ms_per_step_mean": statistics.mean(ms_step),
            "ms_per_step_all": ms_step,
            "timed_region_wall_s": t_wall,
            "higher_is_better": True,
            "scaling": args.scaling,
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic",
            "config": dict(config_dict(args, w, full_geom, geom, ws),
                           walk=T.tet_mesh_features(h)["walk"],
                           entry=("once per step (tet_plan_create), shared by fwd and back"
                                  if use_plan else "per call (tet_project, tet_backproject)")),
            "fwd": {"crossings_per_s": cf_all / (statistics.median(ms_f) / 1e3),
                    "mrays_per_s": rays_all / (statistics.median(ms_f) / 1e3) / 1e6,
                    "ms": statistics.median(ms_f), "crossings": int(cf_all)},
            "back": {"crossings_per_s": cb_all / (statistics.median(ms_b) / 1e3),
                     "mrays_per_s": rays_all / (statistics.median(ms_b) / 1e3) / 1e6,
                     "ms": statistics.median(ms_b), "crossings": int(cb_all)},
            "rays_hit": int(hit_all), "lost": int(lost_all), "stuck": int(stuck_all),
            "exact_fallbacks_per_step": int(exact_all),
            "kernel_ms_per_step": {k: v[0] / args.steps for k, v in kt.items()},
            "mesh_create_s": t_create,
            "roofline": rl,
            "e2e": {"value": e2e_value, "unit": "tet-crossings/s",
                    "h2d_bytes_per_step": int(w.mu.nbytes + y_np.nbytes),
                    "d2h_bytes_per_step": int(proj.numel() * 4 + x.numel() * 4)},
            "gpu_launches": int(round(n_launch_step * args.steps)),
            "clocks": clk,
        }
        if ws > 1:
            line["collective"] = {"backend": backend, "op": "all_reduce(SUM) f32 [n_tets]",
                                  "bytes": int(x.numel() * 4)}
            if backend == "nccl":
                line["collective"]["nccl"] = nccl_report(rank, nccl_log)
        if not args.no_cpu_baseline and ws == 1:
            line["cpu_baseline"] = cpu_baseline(w, geom, y_np)
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
