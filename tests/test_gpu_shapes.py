"""Device residual, Jv and preconditioner applications on small and ragged
meshes (one element wide, odd counts, partial tiles in every direction,
tile-edge nodes at the mesh boundary) against the CPU oracle (oracle/, the
restatement pinned to the reference's goldens in tests/test_oracle.py)."""

import os
import sys

import numpy as np
import pytest
import torch

from conftest import ROOT, rel

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.join(ROOT, "oracle"))

SHAPES = [(2, (1, 1)), (2, (1, 7)), (2, (9, 1)), (2, (3, 2)), (2, (127, 5)), (2, (128, 3)), (2, (129, 4)),
          (2, (256, 17)), (2, (300, 33)),
          (3, (1, 1, 1)), (3, (2, 3, 1)), (3, (15, 17, 3)), (3, (16, 16, 2)), (3, (17, 33, 4)),
          (3, (32, 5, 6))]


@pytest.mark.parametrize("dim,counts", SHAPES)
@pytest.mark.parametrize("model", ["free_growth", "alloy"])
def test_residual_and_jv_on_ragged_meshes(dim, counts, model):
    import oracle as O

    import paper_2006_16764_b200 as uc
    from paper_2006_16764_b200.newton import _FdOperator

    h = 0.03 if model == "free_growth" else 0.8
    ext = [h * c for c in counts]
    mesh = uc.build_mesh(dim, ext, counts)
    k = uc.FreeGrowthKernel() if model == "free_growth" else uc.AlloyKernel()
    n = mesh.n_nodes
    rng = np.random.default_rng(sum(counts) + dim)
    if model == "free_growth":
        mk = lambda: np.concatenate([0.5 + 0.3 * rng.standard_normal(n), 1.0 + 0.2 * rng.standard_normal(n)])  # noqa: E731
    else:
        mk = lambda: np.concatenate([np.tanh(rng.standard_normal(n)), -0.5 + 0.4 * rng.standard_normal(n)])  # noqa: E731
    new, old, prev = mk(), mk(), mk()
    v = rng.standard_normal(2 * n)
    th, dt, step = 0.5, (2.25e-4 if model == "free_growth" else 2e-3), 3
    p = O.Problem(dim, ext, counts, model, k.params, th, dt, step)
    p.begin(old, prev)
    f_ref = p.residual(new)
    jv_ref, _ = p.jv(new, f_ref, v)
    dev = lambda a: torch.tensor(a, device="cuda")  # noqa: E731
    res = uc.TimestepResidual(mesh, k, dev(old), dev(prev), uc.ThetaScheme(th, dt, step))
    u = dev(new)
    f = res(u)
    jv = _FdOperator(res, u, f)(dev(v))
    assert rel(f.cpu().numpy(), f_ref) <= 1e-12
    assert rel(jv.cpu().numpy(), jv_ref) <= 1e-6


@pytest.mark.parametrize("dim,counts", [(2, (4, 4)), (2, (8, 16)), (2, (130, 66)), (2, (40, 200)),
                                        (3, (4, 4, 4)), (3, (8, 16, 4)), (3, (36, 10, 8))])
def test_precond_on_small_meshes(dim, counts):
    """Multicolor V-cycle vs the oracle (1e-12); lexicographic pipelined vs the
    front-by-front wavefront sweep (bitwise; the oracle has no lexicographic
    smoother, that mode is pinned by the reference's default-ordering runs)."""
    import oracle as O

    import paper_2006_16764_b200 as uc

    mesh = uc.build_mesh(dim, [0.03 * c for c in counts], counts)
    k = uc.FreeGrowthKernel()
    n = mesh.n_nodes
    rng = np.random.default_rng(5)
    st = np.concatenate([0.5 + 0.3 * rng.standard_normal(n), 1.0 + 0.2 * rng.standard_normal(n)])
    v = rng.standard_normal(2 * n)
    sc = uc.ThetaScheme(0.5, 2.25e-4, 1)
    std, vd = torch.tensor(st, device="cuda"), torch.tensor(v, device="cuda")
    pc = uc.build_precond(mesh, k, std, sc, uc.PrecondConfig(ordering="multicolor"))
    out = pc.apply(vd).cpu().numpy()
    pc = None
    p = O.Problem(dim, [0.03 * c for c in counts], counts, "free_growth", k.params, 0.5, 2.25e-4, 1)
    assert rel(out, O.BlockPC(p, st, kind="vcycle")(v)) <= 1e-12
    outs = []
    for wave in ("0", "1"):
        os.environ["UC_LEX_WAVEFRONT"] = wave
        try:
            pc = uc.build_precond(mesh, k, std, sc, uc.PrecondConfig(ordering="lexicographic"))
            outs.append(pc.apply(vd).clone())
            pc = None
        finally:
            os.environ.pop("UC_LEX_WAVEFRONT", None)
    assert torch.equal(outs[0], outs[1])
