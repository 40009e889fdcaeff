"""Sum an ncu launch list (`--metrics gpu__time_duration.sum --csv`) per kernel.

usage: python tools/launch_shares.py launches.csv "header comment" > shares.csv
"""
import csv
import re
import sys
from collections import defaultdict


def main(path, comment):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.DictReader(lines))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0,
                 "msecond": 1.0}[r["Metric Unit"]]
        name = re.sub(r"\(.*", "", r["Kernel Name"]).strip()
        name = re.sub(r"\(bool\)|\(int\)", "", name)
        tot[name] += float(r["Metric Value"].replace(",", "")) * scale
        cnt[name] += 1
    all_ms = sum(tot.values())
    for c in comment.split("\n"):
        print("# " + c)
    print("kernel,launches,total_ms,share")
    for k in sorted(tot, key=tot.get, reverse=True):
        print(f"{k},{cnt[k]},{tot[k]:.3f},{tot[k] / all_ms:.4f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
