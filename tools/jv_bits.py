"""Jv bits for the division check: `save` writes Jv of random states at a few
sizes (2D/3D, both models), `compare` checks the current build against it.

    python tools/jv_bits.py save /tmp/jv.npz ; (rebuild) ; python tools/jv_bits.py compare /tmp/jv.npz
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_16764_b200 as uc  # noqa: E402

out = {}
for model, dim, counts in [("free_growth", 2, (300, 200)), ("alloy", 2, (256, 130)), ("free_growth", 3, (40, 36, 30)),
                           ("alloy", 3, (33, 20, 17))]:
    h = 0.03 if model == "free_growth" else 0.8
    mesh = uc.build_mesh(dim, [h * c for c in counts], counts)
    k = uc.FreeGrowthKernel() if model == "free_growth" else uc.AlloyKernel()
    n = mesh.n_nodes
    rng = np.random.default_rng(5)
    if model == "free_growth":
        mk = lambda: np.concatenate([0.5 + 0.3 * rng.standard_normal(n), 1 + 0.2 * rng.standard_normal(n)])  # noqa: E731
    else:
        mk = lambda: np.concatenate([np.tanh(rng.standard_normal(n)), -0.5 + 0.4 * rng.standard_normal(n)])  # noqa: E731
    dev = lambda x: torch.tensor(x, device="cuda")  # noqa: E731
    res = uc.TimestepResidual(mesh, k, dev(mk()), dev(mk()), uc.ThetaScheme(0.5, 2e-3, 2))
    for t in range(3):
        u = dev(mk())
        f = res(u)
        v = dev(rng.standard_normal(2 * n))
        out[f"{model}{dim}_{t}"] = uc.jfnk_matvec(res, u, f, v).cpu().numpy()
if sys.argv[1] == "save":
    np.savez(sys.argv[2], **out)
else:
    ref = np.load(sys.argv[2])
    bad = [key for key in out if not np.array_equal(out[key].view(np.int64), ref[key].view(np.int64))]
    print("jv bits identical" if not bad else f"MISMATCH {bad}")
    sys.exit(1 if bad else 0)
