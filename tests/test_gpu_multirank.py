"""The REMOTE branches of the slab transport (csrc/comm.cu: rank neighbours,
send/recv of ghost planes, all-reduced partial sums, rank-OR'ed status flags,
the eager (uncaptured) preconditioner body) run by two processes, one slab
each.  A gpurun lease has one GPU and NCCL refuses two ranks on one device,
so the ranks use the library's host-staged transport (uc_comm_init_host: the
same call sites, planes staged through pinned host buffers and moved by
torch.distributed over gloo).  Results must be bitwise those of the same two
slabs emulated in one process (tests/test_gpu_slabs.py), and the alloy run
must reproduce the reference's Newton/GMRES counts.  The lexicographic V-cycle
(the ranks sweeping in turn) equals the emulated slabs bitwise as well."""

import os
import socket

import numpy as np
import pytest
import torch

from conftest import golden_meta

pytestmark = pytest.mark.gpu
META = golden_meta()
CASE = "run_al2d_256x64_10"
STEPS = 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(grp, uc, models, k, mesh, m, ortho="mgs"):
    """residual, Jv, V-cycle application and STEPS implicit steps on a slab group;
    returns the slab parts of every result (this process's slabs)."""
    from paper_2006_16764_b200.parallel import SlabPrecond, SlabResidual

    sp = grp.space
    u0 = models.directional_initial_condition(mesh, k.params, amplitude=0.5, seed=0, smooth=True)
    state = grp.split(torch.tensor(u0, device="cuda"))
    n = mesh.n_nodes
    rng = np.random.default_rng(5)
    v = grp.split(torch.tensor(rng.standard_normal(2 * n), device="cuda"))
    sc = uc.ThetaScheme(0.5, m["dt"], 3)
    res = SlabResidual(grp, state, sp.clone(state), sc)
    f = res.device_call(state)
    jv = res.jv_device(state, f, v, sp.norm(state))
    pc = SlabPrecond(grp, state, sc, uc.PrecondConfig(ordering="multicolor"))
    mv = pc.apply(v)
    # the reference's default ordering: the ranks sweep in turn
    mv_lex = SlabPrecond(grp, state, sc, uc.PrecondConfig(ordering="lexicographic")).apply(v)
    out = {"f": f, "jv": jv, "mv": mv, "mv_lex": mv_lex}
    prev = sp.clone(state)
    counts = []
    for step in range(STEPS):
        th = 1.0 if step < m["startup_steps"] else m["theta"]
        sc = uc.ThetaScheme(th, m["dt"], step)
        pc = SlabPrecond(grp, state, sc, uc.PrecondConfig(ordering="multicolor"))
        cfg = uc.NewtonConfig(gmres=uc.GmresConfig(orthogonalization=ortho))
        u, rep = uc.newton_solve(SlabResidual(grp, state, prev, sc), state, cfg, precond_apply=pc.apply)
        assert rep.converged
        counts.append((rep.iterations, rep.total_gmres))
        prev, state = state, u
    out["state"] = state
    return {key: [p.cpu().numpy() for p in val.parts] for key, val in out.items()}, counts


def _worker(rank, world, port, tmp):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import paper_2006_16764_b200 as uc
    from paper_2006_16764_b200 import _lib as L
    from paper_2006_16764_b200 import models
    from paper_2006_16764_b200.parallel import SlabGroup

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = META[CASE]
        mesh = uc.build_mesh(m["dim"], m["extents"], m["counts"])
        k = uc.AlloyKernel()
        grp = SlabGroup.from_torch_dist(mesh, k, transport="host")
        for ortho in ("mgs", "cgs2"):
            parts, counts = _run(grp, uc, models, k, mesh, m, ortho)
            np.savez(os.path.join(tmp, f"rank{rank}_{ortho}.npz"), counts=np.array(counts),
                     **{key: val[0] for key, val in parts.items()})
    finally:
        L.load().uc_comm_finalize()
        dist.destroy_process_group()


def test_two_rank_host_transport_equals_emulated_slabs(tmp_path):
    """MGS (the reference's) and CGS2 Arnoldi, both through the rank branches."""
    import torch.multiprocessing as mp

    import paper_2006_16764_b200 as uc
    from paper_2006_16764_b200 import models
    from paper_2006_16764_b200.parallel import SlabGroup, slab_bounds

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn",
                       join=True)
    m = META[CASE]
    mesh = uc.build_mesh(m["dim"], m["extents"], m["counts"])
    k = uc.AlloyKernel()
    grp = SlabGroup(mesh, k, slab_bounds(mesh, world, 4))
    for ortho in ("mgs", "cgs2"):
        ranks = [dict(np.load(tmp_path / f"rank{r}_{ortho}.npz")) for r in range(world)]
        local, counts = _run(grp, uc, models, k, mesh, m, ortho)
        for key, parts in local.items():
            for r in range(world):
                assert np.array_equal(ranks[r][key].view(np.int64), parts[r].view(np.int64)), (ortho, key, r)
        for r in range(world):
            assert [tuple(c) for c in ranks[r]["counts"]] == counts
        assert [c[0] for c in counts] == m["newton"][:STEPS]
        assert [c[1] for c in counts] == m["gmres"][:STEPS]
