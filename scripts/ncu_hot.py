"""Summarise an ncu report: key metrics per kernel and the hottest SASS lines (stall samples)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "launch__occupancy_limit_shared_mem", "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active"]
for r in rows[2:]:
    print({n: r[h.index(n)] for n in want if n in h})
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
blocks = src.split('"Kernel Name"')
for b in blocks[1:]:
    lines = list(csv.reader(io.StringIO('"Kernel Name"' + b)))
    name = lines[0][1]
    hh = lines[1]
    data = lines[2:]
    si = hh.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[si]) for r in data if len(r) > si and r[si].isdigit())
    print("\n==", name[:80], "samples", tot)
    idx = sorted(range(len(data)), key=lambda i: -(int(data[i][si]) if len(data[i]) > si and data[i][si].isdigit() else 0))[:top]
    for i in sorted(idx):
        print(f"{i:5d} {data[i][si]:>5s}  {data[i][1][:100]}")
