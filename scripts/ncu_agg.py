"""Aggregates an ncu --csv launch list (gpu__time_duration.sum [+ dram__bytes_read.sum]) per kernel name."""
import collections
import csv
import sys

rows = [r for r in csv.DictReader(line for line in open(sys.argv[1]) if line.startswith('"'))]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for r in rows:
    k = r["Kernel Name"][:60]
    v = float(r["Metric Value"].replace(",", ""))
    if r["Metric Name"] == "gpu__time_duration.sum":
        agg[k][0] += 1
        agg[k][1] += v
    else:
        agg[k][2] += v
for k, (n, tot, by) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print("%-60s %5d %10.1f us avg %9.1f us  dram read %.3g B/launch" % (k, n, tot / 1e3, tot / max(n, 1) / 1e3,
                                                                          by / max(n, 1)))
