"""Time the reference package itself (undercool from baseline/_ref, the
unmodified install of tools/install_reference.sh) on ONE core: residual
F(u) = TimestepResidual.__call__ plus the FD Jacobian-vector product
jfnk_matvec (undercool/assembly.py:261-268, newton.py:84-94) on the same
synthetic states as bench.py.  Prints one JSON object.  Run pinned to one
core with single-threaded BLAS/numba (bench.py does this).

    python tools/ref_python_time.py fg2d_2048 [min_seconds]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
sys.path.insert(0, REF)
sys.path.insert(1, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")

import numpy as np  # noqa: E402
import undercool as U  # noqa: E402

from bench import WORKLOADS, synthetic_states  # noqa: E402

name = sys.argv[1]
min_s = float(sys.argv[2]) if len(sys.argv) > 2 else 10.0
w = dict(WORKLOADS[name])
counts, extents = list(w["counts"]), list(w["extents"])
sample = "full workload"
if w["dim"] == 3 or np.prod(counts) > 2048 * 2048:
    # bounded sample: a slab of element layers of the same mesh (same h)
    rows = 16 if w["dim"] == 3 else 512
    extents[-1] *= rows / counts[-1]
    counts[-1] = rows
    sample = f"slab of {rows} of {w['counts'][-1]} element layers (same h), scaled per DoF"
wl = dict(w, counts=tuple(counts), extents=tuple(extents))
N, u, old, prev, v = synthetic_states(wl)
mesh = U.build_mesh(w["dim"], tuple(extents), tuple(counts))
k = U.FreeGrowthKernel() if w["model"] == "free_growth" else U.AlloyKernel()
sc = U.ThetaScheme(w["theta"], w["dt"], w["step"])
res = U.TimestepResidual(mesh, k, old, prev, sc)
f = res(u)
U.jfnk_matvec(res, u, f, v)  # numba JIT warm-up
times = []
while sum(times) < min_s or len(times) < 1:
    t0 = time.perf_counter()
    f = res(u)
    U.jfnk_matvec(res, u, f, v)
    times.append(time.perf_counter() - t0)
sec = float(np.mean(times))
print(json.dumps({"value": round(2 * 2 * N / sec / 1e6, 4), "unit": "MDoF/s", "cores": 1, "kind": "reference",
                  "sample": f"{sample}, {len(times)} timed steps ({sum(times):.1f} s); undercool "
                            "TimestepResidual.__call__ + jfnk_matvec from baseline/_ref, one core "
                            "(taskset, 1 BLAS/numba thread)"}))
