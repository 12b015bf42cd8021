"""Time BlockPrecond.apply (warm, CUDA events) and its build/capture at a given size.

    python tools/vcycle_time.py [--counts 2048 2048] [--reps 20]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2006_16764_b200 as uc  # noqa: E402
from paper_2006_16764_b200.models import seed_initial_condition  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--counts", type=int, nargs="+", default=[2048, 2048])
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--ordering", default="multicolor")
ap.add_argument("--builds", type=int, default=3)
a = ap.parse_args()
mesh = uc.build_mesh(len(a.counts), [0.03 * c for c in a.counts], a.counts)
k = uc.FreeGrowthKernel()
u0 = torch.tensor(seed_initial_condition(mesh, k.params), device="cuda")
sc = uc.ThetaScheme(1.0, 2.25e-4, 0)
pc = None
for rep in range(a.builds):
    pc = None  # recycle the previous hierarchy (buffers + captured graph)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pc = uc.build_precond(mesh, k, u0, sc, uc.PrecondConfig(ordering=a.ordering))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    v = torch.randn_like(u0)
    pc.apply(v)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    for _ in range(3):
        pc.device_apply(v, check=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        pc.device_apply(v, check=False)
    e1.record()
    torch.cuda.synchronize()
    print(f"rep {rep}: build {1e3 * (t1 - t0):.2f} ms  first apply (graph capture) {1e3 * (t2 - t1):.2f} ms  "
          f"warm apply {e0.elapsed_time(e1) / a.reps:.3f} ms", flush=True)
