"""V-cycle applications with the marching residual kernel vs the gather kernel
(UC_RESID_GATHER=1): bitwise comparison, 2D/3D, unsplit and 2 slabs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_16764_b200 as uc  # noqa: E402
from paper_2006_16764_b200.parallel import SlabGroup, SlabPrecond, slab_bounds  # noqa: E402

bad = 0
for counts in [(200, 130), (2048, 2048), (40, 36, 48), (33, 20, 40), (128, 128, 128)]:
    dim = len(counts)
    mesh = uc.build_mesh(dim, [0.03 * c for c in counts], counts)
    k = uc.FreeGrowthKernel()
    n = mesh.n_nodes
    rng = np.random.default_rng(3)
    st = torch.tensor(np.concatenate([0.5 + 0.3 * rng.standard_normal(n), 1 + 0.2 * rng.standard_normal(n)]), device="cuda")
    v = torch.tensor(rng.standard_normal(2 * n), device="cuda")
    sc = uc.ThetaScheme(0.5, 2.25e-4, 1)
    outs = []
    for env in ("0", "1"):
        os.environ["UC_RESID_GATHER"] = env
        pc = uc.build_precond(mesh, k, st, sc, uc.PrecondConfig(ordering="multicolor"))
        a = pc.apply(v).cpu().numpy()
        pc = None
        grp = SlabGroup(mesh, k, slab_bounds(mesh, 2, 4))
        spc = SlabPrecond(grp, grp.space.vec(st), sc, uc.PrecondConfig(ordering="multicolor"))
        b = grp.join(spc.apply(grp.space.vec(v))).cpu().numpy()
        outs.append((a, b))
    same = all(np.array_equal(x.view(np.int64), y.view(np.int64)) for x, y in zip(outs[0], outs[1]))
    slab = np.array_equal(outs[0][0].view(np.int64), outs[0][1].view(np.int64))
    print(counts, "march==gather", same, "slabs==unsplit", slab, flush=True)
    bad += (not same) + (not slab)
sys.exit(1 if bad else 0)
