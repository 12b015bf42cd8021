"""Fraction of uniform stencil tiles per level/block of a built preconditioner
(debug aid): the apply kernels skip the stencil loads of those tiles."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_16764_b200 as uc  # noqa: E402
from paper_2006_16764_b200.stepper import run_steps  # noqa: E402

counts = [int(c) for c in sys.argv[1:]] or [2048, 2048]
mesh = uc.build_mesh(len(counts), [0.03 * c for c in counts], counts)
k = uc.FreeGrowthKernel()
st = uc.models.seed_initial_condition_device(mesh, k.params)
for label, state in [("step0 (seed IC)", st), ("after 2 steps", run_steps(mesh, k, st, 2, 0.5, 2.25e-4)[0])]:
    pc = uc.build_precond(mesh, k, state, uc.ThetaScheme(0.5, 2.25e-4, 2), uc.PrecondConfig(ordering="multicolor"))
    v = torch.randn_like(state)
    pc.apply(v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        pc.device_apply(v, check=False)
    e1.record()
    torch.cuda.synchronize()
    print(label, f"V-cycle {e0.elapsed_time(e1) / 10:.3f} ms", flush=True)
    pc = None
