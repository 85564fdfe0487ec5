"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`): per kernel name the
launch count, total and mean device time and its share of all SM-kernel time. (ncu's per-launch
times are serialised and cold-cache; shares, not absolutes, compare with the live bench.)

usage: python tools/ncu_summary.py launches.csv"""
import collections
import csv
import json
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = None
    for i, r in enumerate(rows):
        if "Kernel Name" in r and "Metric Name" in r:
            hdr, rows = r, rows[i + 1:]
            break
    if hdr is None:
        raise SystemExit("no ncu table header")
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("(anonymous namespace)::", "")
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        tot[name][0] += 1
        tot[name][1] += v * scale
    all_us = sum(t for _, t in tot.values())
    out = [{"kernel": k, "launches": n, "total_us": round(t, 1), "mean_us": round(t / n, 2), "share": round(t / all_us, 4)}
           for k, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1])]
    for o in out:
        print(json.dumps(o))
    print(json.dumps({"kernels": sum(n for n, _ in tot.values()), "total_us": round(all_us, 1)}))


if __name__ == "__main__":
    main()
