"""Slab-decomposed hot path emulated on ONE GPU: k slabs in one
process exchange ghost planes with stream copies through the same kernels and
exchange points as the NCCL transport.  Checked against the unsplit device
path and the reference goldens."""

import os

import numpy as np
import pytest
import torch

from conftest import golden, golden_meta, rel

pytestmark = pytest.mark.gpu
META = golden_meta()


@pytest.fixture(scope="module")
def uc():
    import paper_2006_16764_b200 as uc
    return uc


def _setup(uc, case):
    m = META["residual_" + case]
    g = golden("residual_" + case)
    mesh = uc.build_mesh(m["dim"], m["extents"], m["counts"])
    k = uc.FreeGrowthKernel() if m["model"] == "free_growth" else uc.AlloyKernel(
        uc.AlloyParams(antitrapping_normalized=m["normalized"]))
    return m, g, mesh, k, uc.ThetaScheme(m["theta"], m["dt"], m["step"])


@pytest.mark.parametrize("case", ["fg2d", "fg3d", "al2d", "al3d"])
@pytest.mark.parametrize("world", [2, 3])
def test_slab_residual_and_jv_equal_unsplit(uc, case, world):
    from paper_2006_16764_b200.parallel import SlabGroup, SlabResidual, partition_planes

    m, g, mesh, k, sc = _setup(uc, case)
    nslow = m["counts"][-1] + 1
    slabs = partition_planes(nslow, world, 1)
    grp = SlabGroup(mesh, k, slabs)
    dev = lambda a: torch.tensor(a, device="cuda")  # noqa: E731
    single = uc.TimestepResidual(mesh, k, dev(g["old"]), dev(g["prev"]), sc)
    res = SlabResidual(grp, dev(g["old"]), dev(g["prev"]), sc)
    # same per-element arithmetic and element-id summation order: bitwise equal
    assert torch.equal(grp.join(res.fixed_part), single.fixed_part)
    u = grp.space.vec(dev(g["new"]))
    f = res(u)
    assert torch.equal(grp.join(f), single(dev(g["new"])))
    assert rel(grp.join(f).cpu().numpy(), g["f_call"]) <= 1e-12
    jv = uc.jfnk_matvec(res, u, f, grp.space.vec(dev(g["v"])))
    assert rel(grp.join(jv).cpu().numpy(), g["jv"]) <= 1e-6


@pytest.mark.parametrize("case", ["fg2d", "fg3d", "al2d", "al3d"])
@pytest.mark.parametrize("kind,ordering", [("jacobi", "multicolor"), ("sgs", "multicolor"), ("vcycle", "multicolor"),
                                           ("sgs", "lexicographic"), ("vcycle", "lexicographic")])
def test_slab_preconditioner_equals_unsplit(uc, case, kind, ordering):
    """Lexicographic (the reference's default): the slabs sweep in turn, each
    handing its boundary plane on -- bitwise the unsplit sequential sweep."""
    from paper_2006_16764_b200.parallel import SlabGroup, SlabPrecond, slab_bounds

    m = META["precond_" + case]
    g = golden("precond_" + case)
    mesh = uc.build_mesh(m["dim"], m["extents"], m["counts"])
    k = uc.FreeGrowthKernel() if m["model"] == "free_growth" else uc.AlloyKernel()
    sc = uc.ThetaScheme(m["theta"], m["dt"], m["step"])
    cfg = uc.PrecondConfig(kind=kind, ordering=ordering)
    single = uc.build_precond(mesh, k, g["state"], sc, cfg)
    v = torch.tensor(g["v"], device="cuda")
    ref = single.apply(v)
    nslow = m["counts"][-1] + 1
    nl = max(single.n_levels, 1)
    worlds = [w for w in (2, 3, 4) if (nslow - 1) // 2 ** (nl - 1) >= w]
    assert worlds
    for world in worlds:
        grp = SlabGroup(mesh, k, slab_bounds(mesh, world, nl))
        pc = SlabPrecond(grp, torch.tensor(g["state"], device="cuda"), sc, cfg)
        out = grp.join(pc.apply(grp.space.vec(v)))
        # identical stencils and update order per row; the smoother's halos
        # deliver exactly the values the unsplit sweep reads: bitwise equal
        assert torch.equal(out, ref), (world, float((out - ref).abs().max()))
        key = f"apply_{kind}" + ("_lex" if ordering == "lexicographic" else "")
        assert rel(out.cpu().numpy(), g[key]) <= 1e-12


@pytest.mark.parametrize("world", [2, 4])
def test_slab_newton_steps_match_reference_counts(uc, world):
    from paper_2006_16764_b200 import models
    from paper_2006_16764_b200.parallel import SlabGroup, SlabPrecond, SlabResidual, slab_bounds

    m = META["run_al2d_256x64_10"]
    mesh = uc.build_mesh(m["dim"], m["extents"], m["counts"])
    k = uc.AlloyKernel()
    grp = SlabGroup(mesh, k, slab_bounds(mesh, world, 4))
    u0 = models.directional_initial_condition(mesh, k.params, amplitude=0.5, seed=0, smooth=True)
    state = grp.space.vec(torch.tensor(u0, device="cuda"))
    prev = grp.space.clone(state)
    newton, gm = [], []
    for n in range(m["steps"]):
        th = 1.0 if n < m["startup_steps"] else m["theta"]
        sc = uc.ThetaScheme(th, m["dt"], n)
        pc = SlabPrecond(grp, state, sc, uc.PrecondConfig(ordering="multicolor"))
        res = SlabResidual(grp, state, prev, sc)
        u, rep = uc.newton_solve(res, state, uc.NewtonConfig(), precond_apply=pc.apply)
        assert rep.converged
        newton.append(rep.iterations)
        gm.append(rep.total_gmres)
        prev, state = state, u
    assert newton == m["newton"] and gm == m["gmres"]
    assert rel(grp.join(state).cpu().numpy(), golden("run_al2d_256x64_10")["state"]) <= 1e-8


def test_slab_3d_newton_matches_reference(uc):
    from paper_2006_16764_b200 import models
    from paper_2006_16764_b200.parallel import SlabGroup, SlabPrecond, SlabResidual, slab_bounds

    m = META["run_fg3d_16_3"]
    mesh = uc.build_mesh(m["dim"], m["extents"], m["counts"])
    k = uc.FreeGrowthKernel()
    grp = SlabGroup(mesh, k, slab_bounds(mesh, 2, 4))
    state = grp.space.vec(torch.tensor(models.seed_initial_condition(mesh, k.params), device="cuda"))
    prev = grp.space.clone(state)
    newton, gm = [], []
    for n in range(m["steps"]):
        th = 1.0 if n < m["startup_steps"] else m["theta"]
        sc = uc.ThetaScheme(th, m["dt"], n)
        pc = SlabPrecond(grp, state, sc, uc.PrecondConfig(ordering="multicolor"))
        u, rep = uc.newton_solve(SlabResidual(grp, state, prev, sc), state, precond_apply=pc.apply)
        newton.append(rep.iterations)
        gm.append(rep.total_gmres)
        prev, state = state, u
    assert newton == m["newton"] and gm == m["gmres"]
    assert rel(grp.join(state).cpu().numpy(), golden("run_fg3d_16_3")["state"]) <= 1e-8


def test_nccl_transport_loads_and_initialises():
    """The library's NCCL transport (csrc/comm.cu: dlopen of torch's libnccl,
    unique id, communicator init/finalize) on the GPU box, one rank (a second
    rank on the same GPU is refused by NCCL).  In a subprocess: the
    communicator is process-global."""
    import subprocess
    import sys

    code = (
        "import ctypes as C\n"
        "from paper_2006_16764_b200 import _lib as L\n"
        "from paper_2006_16764_b200.parallel import nccl_library_path\n"
        "lib = L.load(); path = nccl_library_path().encode()\n"
        "idb = (C.c_char * 128)()\n"
        "L.check(lib.uc_nccl_unique_id(path, idb), 'uc_nccl_unique_id')\n"
        "L.check(lib.uc_comm_init_nccl(path, idb, 0, 1), 'uc_comm_init_nccl')\n"
        "assert lib.uc_comm_init_nccl(path, idb, 0, 1) != 0  # second init refused\n"
        "L.check(lib.uc_comm_finalize(), 'uc_comm_finalize')\n"
        "print('nccl ok')\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "nccl ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("counts,world", [((600, 512), 2), ((96, 80, 64), 2), ((70, 40, 96), 3)])
def test_slab_vcycle_equals_unsplit_multi_segment(uc, counts, world):
    """Meshes whose node lines span several 64-node segments of the line-run
    kernels, on 2-3 slabs: the slab V-cycle (multicolor and lexicographic) is
    bitwise the unsplit one."""
    from paper_2006_16764_b200 import models
    from paper_2006_16764_b200.parallel import SlabGroup, SlabPrecond, slab_bounds

    mesh = uc.build_mesh(len(counts), [0.03 * c for c in counts], counts)
    k = uc.FreeGrowthKernel()
    st = models.seed_initial_condition_device(mesh, k.params)
    v = torch.randn(st.numel(), dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(4))
    sc = uc.ThetaScheme(1.0, 2.25e-4, 0)
    for ordering in ("multicolor", "lexicographic"):
        cfg = uc.PrecondConfig(ordering=ordering)
        ref = uc.build_precond(mesh, k, st, sc, cfg).apply(v)
        grp = SlabGroup(mesh, k, slab_bounds(mesh, world, 4))
        out = grp.join(SlabPrecond(grp, grp.split(st), sc, cfg).apply(grp.split(v)))
        assert torch.equal(out, ref), (ordering, float((out - ref).abs().max()))
