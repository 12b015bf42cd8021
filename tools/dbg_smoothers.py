import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2006_16764_b200 as uc
counts=(200,130)
mesh = uc.build_mesh(2, [0.03*c for c in counts], counts)
k = uc.FreeGrowthKernel(); n = mesh.n_nodes
rng = np.random.default_rng(3)
st = torch.tensor(np.concatenate([0.5+0.3*rng.standard_normal(n), 1+0.2*rng.standard_normal(n)]), device='cuda')
v = torch.tensor(rng.standard_normal(2*n), device='cuda')
sc = uc.ThetaScheme(0.5, 2.25e-4, 1)
for kind, sweeps in (("sgs",1),("sgs",2),("vcycle",2)):
    outs=[]
    for env in ("0","1"):
        os.environ["UC_SGS_SMOOTH2"]="1" if env=="0" else "0"

        pc = uc.build_precond(mesh, k, st, sc, uc.PrecondConfig(kind=kind, sweeps=sweeps, ordering="multicolor"))
        outs.append(pc.apply(v).cpu().numpy()); pc=None
    d = np.abs(outs[0]-outs[1]).reshape(2,131,201)
    bad = np.argwhere(d>0)
    print(kind, sweeps, "maxdiff", d.max(), "nbad", len(bad), "rows", sorted(set(bad[:,1].tolist()))[:20], "cols", sorted(set(bad[:,2].tolist()))[:10])
