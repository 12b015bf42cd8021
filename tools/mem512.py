import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_16764_b200 as uc
from paper_2006_16764_b200.models import seed_initial_condition_device
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
mesh = uc.build_mesh(3, (0.03 * n,) * 3, (n,) * 3)
k = uc.FreeGrowthKernel()
print("free", torch.cuda.mem_get_info()[0] / 2**30, flush=True)
u0 = seed_initial_condition_device(mesh, k.params)
torch.cuda.synchronize()
print("ic ok free", torch.cuda.mem_get_info()[0] / 2**30, flush=True)
for lv in (1, 2, 4):
    try:
        pc = uc.build_precond(mesh, k, u0, uc.ThetaScheme(1.0, 2.25e-4, 0), uc.PrecondConfig(ordering="multicolor", levels=lv))
        torch.cuda.synchronize()
        print("levels", lv, "ok", pc.level_shapes, "free", torch.cuda.mem_get_info()[0] / 2**30, flush=True)
        pc = None
    except Exception as e:
        print("levels", lv, "FAIL", e, flush=True)
