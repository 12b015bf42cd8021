import os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_2006_16764_b200 as uc
counts = (2048, 30)
mesh = uc.build_mesh(2, [0.03 * c for c in counts], counts)
k = uc.FreeGrowthKernel()
st = uc.models.seed_initial_condition_device(mesh, k.params)
v = torch.randn_like(st)
pc = uc.build_precond(mesh, k, st, uc.ThetaScheme(1.0, 2.25e-4, 0), uc.PrecondConfig(kind="sgs", sweeps=1, ordering="lexicographic"))
for _ in range(3): pc.apply(v)
torch.cuda.synchronize()
