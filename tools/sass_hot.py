"""SASS listing with executed-instruction counts of one ncu --set full launch,
split into barrier-delimited segments (run here on a .ncu-rep).

    python tools/sass_hot.py report.ncu-rep [launch_skip] [out.txt]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
skip = sys.argv[2] if len(sys.argv) > 2 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", skip, "--launch-count", "1",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) > 10]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
iW = hdr.index("Warp Stall Sampling (All Samples)")
num = lambda x: int(x) if x.isdigit() else 0  # noqa: E731
seen, d2 = set(), []
for r in data:
    if r[0] not in seen:
        seen.add(r[0])
        d2.append(r)
data = d2
tot = sum(num(r[iE]) for r in data)
print("warp instructions", tot)
op = collections.Counter()
for r in data:
    t = r[iS].split()
    if t:
        op[(t[1] if t[0].startswith("@") else t[0]).split(".")[0]] += num(r[iE])
print(", ".join(f"{k} {v / tot:.3f}" for k, v in op.most_common(14)))
acc, start = 0, 0
for i, r in enumerate(data):
    acc += num(r[iE])
    if "BAR.SYNC" in r[iS] or "EXIT" in r[iS] or i == len(data) - 1:
        print(f"  lines {start}-{i}: {acc} ({acc / tot:.3f})")
        acc, start = 0, i + 1
if len(sys.argv) > 3:
    with open(sys.argv[3], "w") as fh:
        for r in data:
            fh.write(f"{num(r[iE]):9d} {num(r[iW]):6d}  {r[iS]}\n")
