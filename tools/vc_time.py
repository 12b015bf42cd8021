"""V-cycle application time (CUDA events) and a preconditioned Newton solve of
the seeded dendrite; env UC_SGS_PERCOLOR=1 selects the colour-by-colour passes.

    python tools/vc_time.py --counts 2048 2048 [--model free_growth] [--reps 20]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_16764_b200 as uc  # noqa: E402
from paper_2006_16764_b200.models import seed_initial_condition_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--counts", type=int, nargs="+", default=[2048, 2048])
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--newton", action="store_true")
a = ap.parse_args()
dim = len(a.counts)
mesh = uc.build_mesh(dim, [0.03 * c for c in a.counts], a.counts)
k = uc.FreeGrowthKernel()
u0 = seed_initial_condition_device(mesh, k.params)
sc = uc.ThetaScheme(1.0, 2.25e-4, 0)
pc = uc.build_precond(mesh, k, u0, sc, uc.PrecondConfig(ordering="multicolor"))
v = torch.randn_like(u0)
s = torch.cuda.current_stream()
for _ in range(3):
    out = pc.device_apply(v, check=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(a.reps):
    out = pc.device_apply(v, check=False)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
print(f"counts={a.counts} percolor={bool(os.environ.get('UC_SGS_PERCOLOR'))} apply_ms={ms:.4f} "
      f"|out|={float(out.norm()):.17g}", flush=True)
if a.newton:
    walls = []
    for r in range(3):
        pc = uc.build_precond(mesh, k, u0, sc, uc.PrecondConfig(ordering="multicolor"))
        res = uc.TimestepResidual(mesh, k, u0, u0, sc)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        u, rep = uc.newton_solve(res, u0, uc.NewtonConfig(), precond_apply=pc.apply)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t0)
    print(f"newton: {rep.iterations} its gmres={rep.gmres_iterations} "
          f"sec/it={np.median(walls[1:]) / rep.iterations:.5f} walls={[round(w, 4) for w in walls]}", flush=True)
if a.newton:
    # where the Newton wall time goes: time every preconditioner application
    # and residual/Jv call with synchronising host timers
    import paper_2006_16764_b200.precond as P
    pc = uc.build_precond(mesh, k, u0, sc, uc.PrecondConfig(ordering="multicolor"))
    res = uc.TimestepResidual(mesh, k, u0, u0, sc)
    tap = []
    orig = pc.apply

    def timed_apply(v):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = orig(v)
        torch.cuda.synchronize()
        tap.append(time.perf_counter() - t0)
        return out

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    u, rep = uc.newton_solve(res, u0, uc.NewtonConfig(), precond_apply=timed_apply)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    print(f"breakdown: wall={wall:.4f} applies={len(tap)} sum={sum(tap):.4f} first={tap[0]:.4f} "
          f"median={np.median(tap):.5f} max={max(tap):.4f}", flush=True)
