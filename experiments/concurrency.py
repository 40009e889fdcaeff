#!/usr/bin/env python
"""Do the forward and backward walks gain from running side by side?  One
c3 step (plan: entry map built once) timed with CUDA events: forward then
backward on one stream, versus forward on one stream and backward on a
second one (joined before the end event), so the block scheduler can mix
the two kernels' blocks on the SMs."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1908_06909_b200 import tetproj as T  # noqa: E402
from workloads import configs as CF  # noqa: E402


def main(cfg="c3", reps=5):
    w = CF.workload(cfg)
    tm = T.TetMesh.from_mesh(w.mesh)
    mu = torch.from_numpy(w.mu).cuda()
    y = torch.from_numpy(CF.uniform_y(w.geom, 1000)).cuda()
    proj = torch.empty(w.geom.n_rays, device="cuda")
    x = torch.empty(w.mesh.n_tets, device="cuda")
    s1 = torch.cuda.current_stream()
    s2 = torch.cuda.Stream()
    pl = tm.plan(w.geom)
    torch.cuda.synchronize()

    def seq():
        T.tet_plan_project(pl.handle, mu, proj, stream=s1.cuda_stream)
        T.tet_plan_backproject(pl.handle, y, x, stream=s1.cuda_stream)

    def conc():
        s2.wait_stream(s1)
        T.tet_plan_project(pl.handle, mu, proj, stream=s1.cuda_stream)
        T.tet_plan_backproject(pl.handle, y, x, stream=s2.cuda_stream)
        s1.wait_stream(s2)

    out = {"config": cfg}
    for name, fn in (("sequential", seq), ("concurrent", conc), ("sequential2", seq),
                     ("concurrent2", conc)):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s1)
            fn()
            b.record(s1)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        out[name + "_ms"] = statistics.median(ts)
    pl.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["c3"]))
