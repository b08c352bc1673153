"""Aggregate an ncu `--metrics gpu__time_duration.sum --csv` launch list per kernel.
Usage: launch_summary.py launches.csv [first_kernel_regex_of_timed_region]"""
import csv
import re
import sys
from collections import OrderedDict


def main(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.reader(lines)
    hdr = next(rd)
    ci = {h: i for i, h in enumerate(hdr)}
    for r in rd:
        if r[ci["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ci["Kernel Name"]]).replace("void ", "")
        unit = r[ci["Metric Unit"]]
        v = float(r[ci["Metric Value"]].replace(",", ""))
        v_us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[unit] * v
        rows.append((name, v_us))
    agg = OrderedDict()
    for n, v in rows:
        c, t = agg.get(n, (0, 0.0))
        agg[n] = (c + 1, t + v)
    tot = sum(t for _, t in agg.values())
    print(f"{len(rows)} launches, {tot/1e3:.2f} ms total (cold-cache, serialised)")
    print(f"{'kernel':60s} {'count':>7s} {'total ms':>10s} {'mean us':>9s} {'share':>7s}")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n[:60]:60s} {c:7d} {t/1e3:10.3f} {t/c:9.2f} {t/tot:7.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
