"""Registers / spills of the kernels matching the given substrings, from a
-Xptxas -v compile of one source file:
    python tools/ptxas_regs.py paper_2006_16764_b200/csrc/precond.cu k_run coarse"""
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16764_b200 import build as B  # noqa: E402

src, pats = sys.argv[1], sys.argv[2:]
r = subprocess.run([B.NVCC, *B.ARCH, *B.FLAGS, "-Xptxas", "-v", "-c", src, "-o", "/tmp/_ptxas.o"],
                   capture_output=True, text=True)
if r.returncode:
    print(r.stderr[-4000:])
    sys.exit(1)
cur = None
info = {}
for line in r.stderr.split("\n"):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
    if cur and any(p in cur for p in pats):
        m1 = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        m2 = re.search(r"Used (\d+) registers", line)
        d = info.setdefault(cur, {})
        if m1:
            d["spill"] = (int(m1.group(1)), int(m1.group(2)))
        if m2:
            d["regs"] = int(m2.group(1))
for k, d in info.items():
    dn = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
    print(f"{dn[:60]:60s} regs={d.get('regs')} spill={d.get('spill')}")
