"""Parity at the BASELINE.json sizes: the device path against the
golden-pinned CPU oracle (oracle/uc_oracle.c, OpenMP on the box's cores) on
identical inputs at the benchmarked meshes, where tile counts, chunk clamps,
edge buffers and 32-bit row indexing differ from the small golden meshes.

  configs[1]  free growth 2D 2048^2
  configs[2]  alloy 2D 4096^2
  configs[3]  free growth 3D 256^3
  configs[4]  a 512 x 512 x 64-element slab of the 512^3 mesh (one rank's
              share of the 8-GPU run; 513 x 513 node planes)

Per mesh: fixed part and F(u) (<= 1e-12), the fused FD Jv (<= 1e-6), and one
multicolor V-cycle application M^-1 v built from the reference's initial
condition (<= 1e-12).  First implicit Newton iteration (backward-Euler startup
step, gmres.restart = 60 as SURVEY 8(c) prescribes at these sizes): GMRES
count exact, state <= 1e-8, at 2048^2 and alloy 4096^2."""

import os
import sys

import numpy as np
import pytest
import torch

from conftest import ROOT, rel

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.join(ROOT, "oracle"))

MESHES = {
    "fg2d_2048": dict(model="free_growth", dim=2, extents=(61.44, 61.44), counts=(2048, 2048), dt=2.25e-4),
    "al2d_4096": dict(model="alloy", dim=2, extents=(3276.8, 3276.8), counts=(4096, 4096), dt=0.002),
    "fg3d_256": dict(model="free_growth", dim=3, extents=(7.68,) * 3, counts=(256,) * 3, dt=2.25e-4),
    "fg3d_512x512x64": dict(model="free_growth", dim=3, extents=(15.36, 15.36, 1.92), counts=(512, 512, 64),
                            dt=2.25e-4),
}


@pytest.fixture(scope="module")
def O():
    import oracle

    oracle.build()
    oracle.set_threads(os.cpu_count() or 1)
    return oracle


def _setup(name):
    import paper_2006_16764_b200 as uc

    w = MESHES[name]
    mesh = uc.build_mesh(w["dim"], w["extents"], w["counts"])
    k = uc.FreeGrowthKernel() if w["model"] == "free_growth" else uc.AlloyKernel()
    return uc, w, mesh, k


def _ic(uc, w, mesh, k):
    from paper_2006_16764_b200 import models

    if w["model"] == "free_growth":
        return models.seed_initial_condition_device(mesh, k.params)
    return models.directional_initial_condition_device(mesh, k.params, amplitude=0.5, seed=0, smooth=True)


@pytest.mark.parametrize("name", list(MESHES))
def test_residual_jv_vcycle_at_scale(O, name):
    from bench import synthetic_states

    uc, w, mesh, k = _setup(name)
    wl = dict(model=w["model"], counts=w["counts"])
    N, u, old, prev, v = synthetic_states(wl)
    sc = uc.ThetaScheme(0.5, w["dt"], 2)
    dev = torch.device("cuda", 0)
    res = uc.TimestepResidual(mesh, k, torch.tensor(old, device=dev), torch.tensor(prev, device=dev), sc)
    ud, vd = torch.tensor(u, device=dev), torch.tensor(v, device=dev)
    f = res(ud)
    jv = uc.jfnk_matvec(res, ud, f, vd)
    p = O.Problem(w["dim"], w["extents"], w["counts"], w["model"], k.params, 0.5, w["dt"], 2)
    fixed_ref = p.begin(old, prev)
    f_ref = p.residual(u)
    assert rel(res.fixed_part.cpu().numpy(), fixed_ref) <= 1e-12
    assert rel(f.cpu().numpy(), f_ref) <= 1e-12
    jv_ref, _ = p.jv(u, f_ref, v)
    assert rel(jv.cpu().numpy(), jv_ref) <= 1e-6
    del res, f, jv, jv_ref, f_ref, fixed_ref
    # preconditioner from the reference's initial condition, startup scheme
    st = _ic(uc, w, mesh, k)
    sc0 = uc.ThetaScheme(1.0, w["dt"], 0)
    pc = uc.build_precond(mesh, k, st, sc0, uc.PrecondConfig(ordering="multicolor"))
    mv = pc.apply(vd).cpu().numpy()
    q = O.Problem(w["dim"], w["extents"], w["counts"], w["model"], k.params, 1.0, w["dt"], 0)
    mv_ref = O.BlockPC(q, st.cpu().numpy())(v)
    assert rel(mv, mv_ref) <= 1e-12


@pytest.mark.parametrize("name", ["fg2d_2048", "al2d_4096"])
def test_first_newton_iteration_at_scale(O, name):
    uc, w, mesh, k = _setup(name)
    st = _ic(uc, w, mesh, k)
    sc0 = uc.ThetaScheme(1.0, w["dt"], 0)
    pc = uc.build_precond(mesh, k, st, sc0, uc.PrecondConfig(ordering="multicolor"))
    res = uc.TimestepResidual(mesh, k, st, st, sc0)
    cfg = uc.NewtonConfig(max_iterations=1, gmres=uc.GmresConfig(restart=60))
    u1, rep = uc.newton_solve(res, st, cfg, precond_apply=pc.apply)
    u0 = st.cpu().numpy()
    q = O.Problem(w["dim"], w["extents"], w["counts"], w["model"], k.params, 1.0, w["dt"], 0)
    q.begin(u0, u0)
    u_ref, rep_ref = O.newton(q, u0, O.BlockPC(q, u0), max_iterations=1, restart=60)
    assert rep.iterations == rep_ref["iterations"] == 1
    assert rep.gmres_iterations == rep_ref["gmres"]
    assert rel(u1.cpu().numpy(), u_ref) <= 1e-8
