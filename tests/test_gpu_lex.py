"""Pipelined lexicographic Gauss-Seidel (csrc/precond.cu k_lex2d in 2D,
k_lex_pipe3 with shared class rows and k_lex_pipe in 3D) against
the grid-barrier wavefront kernel that executes the reference's sequential
sweep front by front (k_sgs_lex, precond.py:32-51): applications must be
BITWISE identical -- same subtraction order, correctly rounded division --
across unit boundaries (> 32 rows), ragged row counts, both sweep directions,
2D and 3D, both models, one-level SGS and the V-cycle."""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

CASES = [(2, (16, 12)), (2, (64, 40)), (2, (33, 95)), (2, (100, 70)),
         (3, (8, 6, 5)), (3, (16, 16, 16)), (3, (40, 36, 10)), (3, (24, 70, 20))]


def _apply(uc, mesh, k, st, v, wavefront, kind):
    old = os.environ.get("UC_LEX_WAVEFRONT")
    os.environ["UC_LEX_WAVEFRONT"] = "1" if wavefront else "0"
    try:
        pc = uc.build_precond(mesh, k, st, uc.ThetaScheme(0.5, 2.25e-4, 1),
                              uc.PrecondConfig(kind=kind, ordering="lexicographic"))
        return pc.apply(v).clone()
    finally:
        if old is None:
            del os.environ["UC_LEX_WAVEFRONT"]
        else:
            os.environ["UC_LEX_WAVEFRONT"] = old


@pytest.mark.parametrize("dim,counts", CASES)
@pytest.mark.parametrize("model", ["free_growth", "alloy"])
def test_pipelined_lexicographic_is_bitwise_the_sequential_sweep(dim, counts, model):
    import paper_2006_16764_b200 as uc

    mesh = uc.build_mesh(dim, [0.03 * c for c in counts], counts)
    rng = np.random.default_rng(7)
    n = mesh.n_nodes
    if model == "free_growth":
        k = uc.FreeGrowthKernel()
        st = np.concatenate([0.5 + 0.3 * rng.standard_normal(n), 1 + 0.2 * rng.standard_normal(n)])
    else:
        k = uc.AlloyKernel()
        st = np.concatenate([np.tanh(rng.standard_normal(n)), -0.5 + 0.4 * rng.standard_normal(n)])
    st = torch.tensor(st, device="cuda")
    v = torch.tensor(rng.standard_normal(2 * n), device="cuda")
    for kind in ("sgs", "vcycle"):
        a = _apply(uc, mesh, k, st, v, False, kind)
        b = _apply(uc, mesh, k, st, v, True, kind)
        assert torch.equal(a, b), (kind, float((a - b).abs().max()))
        if dim == 3:
            os.environ["UC_LEX3_ROWS"] = "1"
            try:
                c = _apply(uc, mesh, k, st, v, False, kind)
            finally:
                del os.environ["UC_LEX3_ROWS"]
            assert torch.equal(a, c), (kind, float((a - c).abs().max()))


@pytest.mark.parametrize("dim,counts,model", [(2, (64, 40), "free_growth"), (2, (33, 95), "alloy"),
                                              (3, (16, 16, 16), "free_growth"), (3, (12, 10, 8), "alloy")])
def test_uniform_tiles_are_bitwise_the_explicit_stencils(dim, counts, model):
    """Apply kernels read one shared row for stencil rows bitwise equal to it
    (csrc/precond.cu k_tile_uniform, per-row masks); the result must be
    identical to reading every row (UC_PC_NO_UNIFORM=1)."""
    import paper_2006_16764_b200 as uc

    mesh = uc.build_mesh(dim, [0.03 * c for c in counts], counts)
    k = uc.FreeGrowthKernel() if model == "free_growth" else uc.AlloyKernel()
    st = uc.models.seed_initial_condition_device(mesh, uc.FreeGrowthParams()) if model == "free_growth" \
        else uc.models.directional_initial_condition_device(mesh, uc.AlloyParams(), amplitude=0.5, smooth=True)
    v = torch.randn_like(st)
    outs = []
    for flag in ("0", "1"):
        if flag == "1":
            os.environ["UC_PC_NO_UNIFORM"] = "1"
        try:
            for ordering in ("multicolor", "lexicographic"):
                pc = uc.build_precond(mesh, k, st, uc.ThetaScheme(0.5, 2.25e-4, 1),
                                      uc.PrecondConfig(ordering=ordering))
                if flag == "0" and ordering == "multicolor" and model == "free_growth":
                    assert pc.uniform_fraction(0, 1) > 0.5  # constant-coefficient heat block: all interior rows
                outs.append(pc.apply(v).clone())
                pc = None
        finally:
            os.environ.pop("UC_PC_NO_UNIFORM", None)
    assert torch.equal(outs[0], outs[2]) and torch.equal(outs[1], outs[3])
