import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2006_16764_b200.driver as drv
from paper_2006_16764_b200.config import RunConfig, MeshConfig, TimeConfig
orig = drv.newton_solve
def wrapped(res, u0, cfg=None, precond_apply=None):
    u, rep = orig(res, u0, cfg, precond_apply=precond_apply)
    print("newton", rep.converged, rep.iterations, rep.gmres_iterations, rep.residual_norms[:6], rep.final_norm, rep.failure_reason, rep.step_lengths, float(u.abs().max()), flush=True)
    return u, rep
drv.newton_solve = wrapped
for order in ("lexicographic", "multicolor"):
    cfg = RunConfig()
    cfg.mesh = MeshConfig(dimension=2, extents=(0.96, 0.96), counts=(32, 32))
    cfg.time = TimeConfig(theta=0.0, dt=5.625e-4, t_final=5.625e-4 * 50)
    cfg.precond.ordering = order
    r = drv.simulate(cfg)
    print(order, r.status, r.failure_detail, r.steps_completed)
