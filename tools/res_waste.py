import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2006_16764_b200 as uc
for counts in [(2048, 2048), (2031, 2048), (2032, 2048), (1905, 2048), (2540, 2048)]:
    mesh = uc.build_mesh(2, [0.03 * c for c in counts], counts)
    k = uc.FreeGrowthKernel()
    n = mesh.n_nodes
    rng = np.random.default_rng(11)
    mk = lambda: torch.tensor(np.concatenate([0.5 + 0.3 * rng.standard_normal(n), 1.0 + 0.2 * rng.standard_normal(n)]), device="cuda")
    u, old, prev = mk(), mk(), mk()
    res = uc.TimestepResidual(mesh, k, old, prev, uc.ThetaScheme(0.5, 2.25e-4, 2))
    for _ in range(3): res.device_call(u, check=False) if hasattr(res, "device_call") else res(u)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): res(u)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(counts, f"{ms:.4f} ms", f"{2*n/ms/1e3:.0f} MDoF/s", f"{counts[0]*counts[1]/ms/1e6:.3f} Gelem/s", "tiles", -(-(counts[0]+1)//127))
