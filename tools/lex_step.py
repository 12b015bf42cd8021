"""Per-step time of the pipelined lexicographic sweep: one unit (<= 32 rows)
and a many-unit mesh, kind='sgs' (one level), warm apply timing."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2006_16764_b200 as uc  # noqa: E402

for counts, sweeps in [((2048, 30), 1), ((2048, 30), 4), ((2048, 62), 1), ((2048, 2048), 1), ((512, 512), 1)]:
    mesh = uc.build_mesh(2, [0.03 * c for c in counts], counts)
    k = uc.FreeGrowthKernel()
    st = uc.models.seed_initial_condition_device(mesh, k.params)
    v = torch.randn_like(st)
    pc = uc.build_precond(mesh, k, st, uc.ThetaScheme(1.0, 2.25e-4, 0),
                          uc.PrecondConfig(kind="sgs", sweeps=sweeps, ordering="lexicographic"))
    pc.apply(v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        pc.device_apply(v, check=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    n0, n1 = counts[0] + 1, counts[1] + 1
    steps = n0 + 2 * n1
    print(counts, "sweeps", sweeps, f"apply {ms:.3f} ms  per half-sweep {ms / (2 * sweeps):.3f} ms  "
          f"~{1e6 * ms / (2 * sweeps) / steps:.1f} ns per front", flush=True)
