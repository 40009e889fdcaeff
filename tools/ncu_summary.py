#!/usr/bin/env python
"""Summarise an `ncu --set full` report of walk kernels into JSON (the
metrics profiles/ and bench.py's roofline use).

  python tools/ncu_summary.py REPORT.ncu-rep "capture description;..." > out.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_red.sum",
        "smsp__inst_executed_op_global_red.sum",
        "smsp__sass_inst_executed_op_global_ld.sum",
        "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"]
STALLS = ["wait", "long_scoreboard", "not_selected", "math_pipe_throttle", "dispatch_stall",
          "selected", "short_scoreboard", "branch_resolving", "lg_throttle", "mio_throttle",
          "barrier", "no_instruction", "drain"]


def main():
    rep = sys.argv[1]
    captions = sys.argv[2].split(";") if len(sys.argv) > 2 else []
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    units = rows[1]
    ci = {k: i for i, k in enumerate(hdr)}
    out = []
    for n, r in enumerate(rows[2:]):
        d = {"capture": captions[n] if n < len(captions) else f"kernel {n}"}
        for k in KEYS:
            if k in ci:
                d[k] = (r[ci[k]] + " " + units[ci[k]]).strip()
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in ci:
                d[k] = r[ci[k]]
        out.append(d)
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main()
