"""Timing of the one-level lexicographic SGS apply on a 2D mesh: python tools/lex_two.py NX NY"""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_2006_16764_b200 as uc
counts = tuple(int(c) for c in sys.argv[1:3])
mesh = uc.build_mesh(2, [0.03 * c for c in counts], counts)
k = uc.FreeGrowthKernel()
st = uc.models.seed_initial_condition_device(mesh, k.params)
v = torch.randn_like(st)
pc = uc.build_precond(mesh, k, st, uc.ThetaScheme(1.0, 2.25e-4, 0), uc.PrecondConfig(kind="sgs", sweeps=1, ordering="lexicographic"))
for _ in range(2): pc.apply(v)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): pc.device_apply(v, check=False)
e1.record(); torch.cuda.synchronize()
print(counts, f"{e0.elapsed_time(e1) / 5:.3f} ms per sgs apply (2 cycles x 1 sweep)")
