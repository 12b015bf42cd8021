"""Launch each residual/Jv tile variant once (for ncu instruction-mix capture).

    ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,... python tools/kernel_mix.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_16764_b200 as uc  # noqa: E402

CASES = [("free_growth", 2, (2048, 2048)), ("alloy", 2, (2048, 2048)),
         ("free_growth", 3, (256, 256, 256)), ("alloy", 3, (128, 128, 128))]
for model, dim, counts in CASES:
    h = 0.03 if model == "free_growth" else 0.8
    mesh = uc.build_mesh(dim, [h * c for c in counts], counts)
    k = uc.FreeGrowthKernel() if model == "free_growth" else uc.AlloyKernel()
    n = mesh.n_nodes
    rng = np.random.default_rng(11)
    if model == "free_growth":
        mk = lambda: np.concatenate([0.5 + 0.3 * rng.standard_normal(n), 1.0 + 0.2 * rng.standard_normal(n)])  # noqa: E731
    else:
        mk = lambda: np.concatenate([np.tanh(rng.standard_normal(n)), -0.5 + 0.4 * rng.standard_normal(n)])  # noqa: E731
    dev = lambda a: torch.tensor(a, device="cuda")  # noqa: E731
    res = uc.TimestepResidual(mesh, k, dev(mk()), dev(mk()), uc.ThetaScheme(0.5, 2e-3, 2))
    u = dev(mk())
    f = res.device_call(u, check=False)
    res.jv_device(u, f, dev(np.random.default_rng(2).standard_normal(2 * n)), 1.0)
    torch.cuda.synchronize()
    print(model, dim, counts, "elements", int(np.prod(counts)), flush=True)
