"""Pipelined lexicographic SGS vs the grid-barrier wavefront kernel: bitwise
equality of BlockPrecond.apply, plus warm apply times.

    python tools/lex_check.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_16764_b200 as uc  # noqa: E402


def apply(mesh, k, st, v, wave, kind="vcycle", reps=0):
    os.environ["UC_LEX_WAVEFRONT"] = "1" if wave else "0"
    pc = uc.build_precond(mesh, k, st, uc.ThetaScheme(0.5, 2.25e-4, 1),
                          uc.PrecondConfig(kind=kind, ordering="lexicographic"))
    out = pc.apply(v).clone()
    ms = None
    if reps:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            pc.device_apply(v, check=False)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
    return out, ms


cases = [(2, (16, 12)), (2, (64, 40)), (2, (100, 70)), (2, (33, 95)), (2, (512, 512)),
         (3, (8, 6, 5)), (3, (16, 16, 16)), (3, (40, 36, 10)), (3, (64, 64, 64))]
rng = np.random.default_rng(3)
bad = 0
for dim, counts in cases:
    mesh = uc.build_mesh(dim, [0.03 * c for c in counts], counts)
    for model in ("free_growth", "alloy"):
        k = uc.FreeGrowthKernel() if model == "free_growth" else uc.AlloyKernel()
        n = mesh.n_nodes
        if model == "free_growth":
            st = np.concatenate([0.5 + 0.3 * rng.standard_normal(n), 1 + 0.2 * rng.standard_normal(n)])
        else:
            st = np.concatenate([np.tanh(rng.standard_normal(n)), -0.5 + 0.4 * rng.standard_normal(n)])
        st = torch.tensor(st, device="cuda")
        v = torch.tensor(rng.standard_normal(2 * n), device="cuda")
        for kind in ("sgs", "vcycle"):
            a, _ = apply(mesh, k, st, v, False, kind)
            b, _ = apply(mesh, k, st, v, True, kind)
            same = torch.equal(a, b)
            bad += not same
            print(dim, counts, model, kind, "bitwise" if same else f"DIFF {float((a - b).abs().max()):.3e}", flush=True)
for counts in ([512, 512], [2048, 2048], [128, 128, 128]):
    mesh = uc.build_mesh(len(counts), [0.03 * c for c in counts], counts)
    k = uc.FreeGrowthKernel()
    st = uc.models.seed_initial_condition_device(mesh, k.params)
    v = torch.randn_like(st)
    _, t_new = apply(mesh, k, st, v, False, reps=5)
    _, t_old = apply(mesh, k, st, v, True, reps=2)
    print("timing", counts, f"pipelined {t_new:.3f} ms  wavefront {t_old:.3f} ms", flush=True)
print("bad", bad)
