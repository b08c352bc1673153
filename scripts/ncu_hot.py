"""Top SASS lines by stall samples for one kernel of an ncu report (needs -lineinfo / --import-source)."""
import csv
import subprocess
import sys


def main(path, kregex, n=30, ctx=0):
    out = subprocess.check_output(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name", "regex:" + kregex,
                                   "--print-source", "sass"], text=True)
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    data, seen = [], set()
    for r in rows[2:]:
        if len(r) < 3 or r[0] in seen:
            continue
        seen.add(r[0])
        data.append(r)
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[i_s]) for r in data if r[i_s].isdigit())
    order = sorted(range(len(data)), key=lambda i: -int(data[i][i_s]) if data[i][i_s].isdigit() else 0)
    print("total samples", tot)
    for i in order[:n]:
        if ctx:
            for j in range(max(0, i - ctx), i):
                print("      ", data[j][0][-5:], data[j][1][:100])
        print(data[i][i_s].rjust(6), data[i][0][-5:], data[i][1][:100])
        if ctx:
            print()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30,
         int(sys.argv[4]) if len(sys.argv) > 4 else 0)
