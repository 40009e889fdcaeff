#!/usr/bin/env python
"""profiles/ncu_issue.json and profiles/ncu_traffic.json from the ncu
summaries of one capture run (tools/gpu_r02_head_ncu.sh) and the crossings of
the captured launches (tools/launch_crossings.py):

  python tools/ncu_to_profiles.py PREFIX crossings.json "source note"

PREFIX_c3_summary.json holds [c3 forward launch 0, c3 forward launch 1,
c3 backward launch 0]; PREFIX_{c5,c2,c4b,c4a}_{fwd,back}_summary.json one
launch each (c4a, when present: the exact-heavy shape its timed steps run,
tools/gpu_r02_c4a_ncu.sh)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def num(s):
    return float(str(s).split()[0])


def scaled(s):
    v, unit = str(s).split()[:2]
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[unit]


def ms(s):
    v, unit = str(s).split()[:2]
    return float(v) * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
                       "msecond": 1.0, "s": 1e3, "second": 1e3}[unit]


def entry(k, crossings):
    return {
        "warp_inst_per_crossing": round(num(k["smsp__inst_executed.sum"]) / crossings, 4),
        "issue_active_pct": round(num(k["smsp__issue_active.avg.pct_of_peak_sustained_active"]), 2),
        "warps_active_pct": round(num(k["sm__warps_active.avg.pct_of_peak_sustained_active"]), 2),
        "l1_lsu_wavefronts_pct": round(num(k["l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"]), 2),
        "lts_throughput_pct": round(num(k["lts__throughput.avg.pct_of_peak_sustained_elapsed"]), 2),
        "red_l2_sectors_per_crossing": round(num(k["lts__t_sectors_srcunit_tex_op_red.sum"]) / crossings, 4),
        "local_loads_per_crossing": round(num(k["smsp__sass_inst_executed_op_local_ld.sum"]) / crossings, 4),
        "registers": int(num(k["launch__registers_per_thread"])),
        "kernel_ms_ncu": ms(k["gpu__time_duration.sum"]),
        "crossings": crossings,
    }


def main(prefix, cross_path, note):
    cross = json.load(open(cross_path))
    issue = {"_source": note, "kernels": "FT16 walks at HEAD"}
    traffic = {"_source": "dram__bytes_read.sum + dram__bytes_write.sum of the captured walk "
                          "launch / its crossings (ncu flushes caches before each captured "
                          "kernel, so the cold read of the tag table is included), same "
                          "captures as profiles/ncu_issue.json"}
    for cfg in ("c3", "c5", "c2", "c4b", "c4a"):
        if cfg not in cross or (cfg != "c3" and not os.path.exists(f"{prefix}_{cfg}_fwd_summary.json")):
            continue
        c = cross[cfg]["crossings"]
        if cfg == "c3":
            ks = json.load(open(f"{prefix}_c3_summary.json"))
            fwd, back = ks[0], ks[2]
        else:
            fwd = json.load(open(f"{prefix}_{cfg}_fwd_summary.json"))[0]
            back = json.load(open(f"{prefix}_{cfg}_back_summary.json"))[0]
        issue[cfg] = {"forward": entry(fwd, c), "backward": entry(back, c)}
        traffic[cfg] = {d: {"dram_bytes_per_crossing":
                            (scaled(k["dram__bytes_read.sum"]) + scaled(k["dram__bytes_write.sum"])) / c}
                        for d, k in (("forward", fwd), ("backward", back))}
    for name, obj in (("ncu_issue.json", issue), ("ncu_traffic.json", traffic)):
        with open(os.path.join(ROOT, "profiles", name), "w") as f:
            json.dump(obj, f, indent=1)
            f.write("\n")


if __name__ == "__main__":
    main(*sys.argv[1:4])
