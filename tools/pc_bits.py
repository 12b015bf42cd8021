"""Preconditioner-application bits before/after a kernel change: `save` writes
V-cycle applications (2D/3D, both models, multicolor; unsplit and two local
slabs), `compare` checks the current build / environment against them.

    UC_RESID_GATHER=1 python tools/pc_bits.py save /tmp/pc.npz ; python tools/pc_bits.py compare /tmp/pc.npz
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_16764_b200 as uc  # noqa: E402
from paper_2006_16764_b200.parallel import SlabGroup, SlabPrecond, slab_bounds  # noqa: E402

out = {}
for model, dim, counts in [("free_growth", 2, (200, 130)), ("alloy", 2, (96, 64)), ("free_growth", 3, (40, 36, 48)),
                           ("alloy", 3, (33, 20, 40)), ("free_growth", 3, (70, 17, 64))]:
    mesh = uc.build_mesh(dim, [0.03 * c for c in counts], counts)
    k = uc.FreeGrowthKernel() if model == "free_growth" else uc.AlloyKernel()
    n = mesh.n_nodes
    rng = np.random.default_rng(3)
    if model == "free_growth":
        st = np.concatenate([0.5 + 0.3 * rng.standard_normal(n), 1 + 0.2 * rng.standard_normal(n)])
    else:
        st = np.concatenate([np.tanh(rng.standard_normal(n)), -0.5 + 0.4 * rng.standard_normal(n)])
    st = torch.tensor(st, device="cuda")
    v = torch.tensor(rng.standard_normal(2 * n), device="cuda")
    sc = uc.ThetaScheme(0.5, 2.25e-4, 1)
    pc = uc.build_precond(mesh, k, st, sc, uc.PrecondConfig(ordering="multicolor"))
    out[f"{model}{dim}_{counts}"] = pc.apply(v).cpu().numpy()
    pc = None
    grp = SlabGroup(mesh, k, slab_bounds(mesh, 2, 4))
    spc = SlabPrecond(grp, grp.space.vec(st), sc, uc.PrecondConfig(ordering="multicolor"))
    out[f"{model}{dim}_{counts}_slabs"] = grp.join(spc.apply(grp.space.vec(v))).cpu().numpy()
if sys.argv[1] == "save":
    np.savez(sys.argv[2], **out)
else:
    ref = np.load(sys.argv[2])
    bad = [key for key in out if not np.array_equal(out[key].view(np.int64), ref[key].view(np.int64))]
    print("preconditioner bits identical" if not bad else f"MISMATCH {bad}")
    sys.exit(1 if bad else 0)
