import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2006_16764_b200 as uc

def seq_sgs(st, shape, b, sweeps, dim):
    n = int(np.prod(shape)); x = np.zeros(n)
    nx = shape[0]; ny = shape[1]; nz = shape[2] if dim == 3 else 1
    K = 3 ** dim
    def row(i):
        i0 = i % nx; r = i // nx; i1 = r % ny; i2 = r // ny
        s = b[i]
        for k in range(K):
            if k == K // 2: continue
            dx, dy, dz = k % 3 - 1, (k // 3) % 3 - 1, (k // 9 - 1) if dim == 3 else 0
            j0, j1, j2 = i0 + dx, i1 + dy, i2 + dz
            if not (0 <= j0 < nx and 0 <= j1 < ny and 0 <= j2 < nz): continue
            s = s - st[i, k] * x[j0 + nx * (j1 + ny * j2)]
        x[i] = s / st[i, K // 2]
    for _ in range(sweeps):
        for i in range(n): row(i)
        for i in range(n - 1, -1, -1): row(i)
    return x

for dim, counts in [(2, (6, 4)), (2, (6, 40)), (3, (4, 3, 2))]:
    mesh = uc.build_mesh(dim, [0.03 * c for c in counts], counts)
    k = uc.FreeGrowthKernel()
    rng = np.random.default_rng(0)
    n = mesh.n_nodes
    st = torch.tensor(np.concatenate([0.5 + 0.3 * rng.standard_normal(n), 1 + 0.2 * rng.standard_normal(n)]), device="cuda")
    v = rng.standard_normal(2 * n)
    for wave in ("0", "1"):
        os.environ["UC_LEX_WAVEFRONT"] = wave
        pc = uc.build_precond(mesh, k, st, uc.ThetaScheme(0.5, 2.25e-4, 1), uc.PrecondConfig(kind="sgs", sweeps=1, ordering="lexicographic"))
        out = pc.apply(torch.tensor(v, device="cuda")).cpu().numpy()
        for blk in range(2):
            S = pc.level_stencil(0, blk)
            ref = seq_sgs(S, mesh.node_shape, v[blk * n:(blk + 1) * n], 1, dim)
            d = np.abs(out[blk * n:(blk + 1) * n] - ref)
            bad = np.nonzero(d > 0)[0]
            print(dim, counts, "wave" if wave == "1" else "pipe", blk, "maxdiff", d.max(), "first bad nodes", bad[:10])
