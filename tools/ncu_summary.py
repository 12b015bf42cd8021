"""Summarise ncu outputs for profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py launches <launches.csv>        # per-kernel share table
    python tools/ncu_summary.py report <prof.ncu-rep> [regex]  # key metrics per launch
"""

import collections
import csv
import io
import re
import subprocess
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def launches(path):
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rows = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows:
        name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "").replace("uc::", "")
        us = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1.0)
        tot[name] += us
        cnt[name] += 1
    T = sum(tot.values())
    out = [f"launches: {len(rows)}, summed device time {T / 1e3:.3f} ms (ncu: serialised, cold cache)",
           "", "| kernel | launches | total ms | share | avg us |", "|---|---|---|---|---|"]
    for k in sorted(tot, key=lambda k: -tot[k]):
        out.append(f"| `{k}` | {cnt[k]} | {tot[k] / 1e3:.3f} | {tot[k] / T:.3f} | {tot[k] / cnt[k]:.2f} |")
    return "\n".join(out)


KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe % active"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 inst % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("sass__inst_executed_register_spilling", "spill insts"),
    ("smsp__inst_executed.sum", "warp insts"),
]


def report(path, pattern=None):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    hdr, units = r[0], r[1]
    idx = {k: hdr.index(k) for k, _ in KEYS if k in hdr}
    ki = hdr.index("Kernel Name")
    out = ["| kernel | " + " | ".join(lbl for k, lbl in KEYS if k in idx) + " |",
           "|---" * (1 + len(idx)) + "|"]
    for row in r[2:]:
        if pattern and not re.search(pattern, row[ki]):
            continue
        cells = []
        for k, _ in KEYS:
            if k in idx:
                cells.append(f"{row[idx[k]]} {units[idx[k]]}".strip())
        out.append(f"| `{re.sub(r'[(].*', '', row[ki])}` | " + " | ".join(cells) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]))
    else:
        print(report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None))
