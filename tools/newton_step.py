"""One warm preconditioned Newton solve of the seeded 2D/3D dendrite (for ncu
launch lists / profiling; not a benchmark number).

    python tools/newton_step.py [--counts 2048 2048] [--reps 2]
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
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
dim = len(a.counts)
mesh = uc.build_mesh(dim, [0.03 * c for c in a.counts], a.counts)
k = uc.FreeGrowthKernel()
u0 = torch.tensor(seed_initial_condition(mesh, k.params), device="cuda")
sc = uc.ThetaScheme(1.0, 2.25e-4, 0)
for r in range(a.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pc = uc.build_precond(mesh, k, u0, sc, uc.PrecondConfig(ordering="multicolor"))
    res = uc.TimestepResidual(mesh, k, u0, u0, sc)
    u, rep = uc.newton_solve(res, u0, uc.NewtonConfig(), precond_apply=pc.apply)
    torch.cuda.synchronize()
    print(f"rep {r}: {time.perf_counter() - t0:.4f} s newton={rep.iterations} gmres={rep.gmres_iterations}",
          flush=True)
