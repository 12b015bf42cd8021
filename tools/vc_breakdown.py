"""Aggregate an ncu launch list (gpu__time_duration.sum, --csv) per kernel and
grid: total, count and mean device time.

    python tools/vc_breakdown.py gpurun_out/vc2d.csv [--per N]   (N = applies)
"""
import collections
import csv
import gzip
import re
import sys


def load(path):
    op = gzip.open if path.endswith(".gz") else open
    rows = list(csv.reader(op(path, "rt")))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
    out = []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        out.append((re.sub(r"\(.*", "", r[ki]).replace("void ", ""), r[gi], v))
    return out


def main():
    path = sys.argv[1]
    per = float(sys.argv[sys.argv.index("--per") + 1]) if "--per" in sys.argv else 1.0
    d = collections.defaultdict(list)
    for name, grid, v in load(path):
        d[(name, grid)].append(v)
    tot = sum(sum(v) for v in d.values())
    for (name, grid), v in sorted(d.items(), key=lambda x: -sum(x[1])):
        s = sum(v)
        print(f"{s / per / 1e3:9.1f} us/apply {100 * s / tot:5.1f}%  n/apply={len(v) / per:6.1f} "
              f"mean={s / len(v) / 1e3:7.2f} us  {name[:44]:44s} {grid}")
    print(f"total {tot / per / 1e3:.1f} us per apply")


if __name__ == "__main__":
    main()
