"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
count, total and average device time, share of the listed total.  Usage:
  python tools/launch_summary.py gpurun_out/launches.csv > profiles/r01_launches.txt"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= vi or r[ki] == "":
            continue
        name = r[ki].replace("void ", "").split("(")[0]
        us = float(r[vi].replace(",", "")) * scale[r[ui]]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    print(f"# {path}: {sum(a[0] for a in agg.values())} launches, {tot:.1f} us total (cold-cache, serialised)")
    print(f"{'kernel':40s} {'n':>5s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} {n:5d} {us:10.1f} {us / n:9.2f} {us / tot:6.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
