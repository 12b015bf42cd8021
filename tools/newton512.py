"""3D 512^3 on one B200 (BASELINE configs[4] at N=1): V-cycle application and
one warm backward-Euler Newton solve of the seeded dendrite (multicolor
smoother), one preconditioner alive at a time.

    python tools/newton512.py [--counts 512 512 512]
"""
import argparse
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2006_16764_b200 as uc  # noqa: E402
from paper_2006_16764_b200.models import seed_initial_condition_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--counts", type=int, nargs="+", default=[512, 512, 512])
a = ap.parse_args()
mesh = uc.build_mesh(len(a.counts), [0.03 * c for c in a.counts], a.counts)
k = uc.FreeGrowthKernel()
u0 = seed_initial_condition_device(mesh, k.params)
sc = uc.ThetaScheme(1.0, 2.25e-4, 0)
pc = uc.build_precond(mesh, k, u0, sc, uc.PrecondConfig(ordering="multicolor"))
v = torch.randn_like(u0)
for _ in range(2):
    out = pc.device_apply(v, check=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    out = pc.device_apply(v, check=False)
e1.record()
torch.cuda.synchronize()
print(f"counts={a.counts} vcycle_apply_ms={e0.elapsed_time(e1) / 3:.2f}", flush=True)
del out, v
gc.collect()
torch.cuda.empty_cache()
walls = []
for rep in range(2):
    res = uc.TimestepResidual(mesh, k, u0, u0, sc)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    u, r = uc.newton_solve(res, u0, uc.NewtonConfig(), precond_apply=pc.apply)
    torch.cuda.synchronize()
    walls.append(time.perf_counter() - t0)
    del u, res
    gc.collect()
print(f"newton: {r.iterations} its gmres={r.gmres_iterations} converged={r.converged} "
      f"sec/it={walls[-1] / max(r.iterations, 1):.4f} walls={[round(w, 3) for w in walls]} "
      f"mem_GB={torch.cuda.max_memory_allocated() / 1e9:.1f}", flush=True)
