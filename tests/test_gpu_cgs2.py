"""CGS2 Arnoldi (GmresConfig.orthogonalization="cgs2", csrc/blas.cu
cgs2_group): the same two orthogonalisation passes as the reference's MGS
(krylov.py:48-70), computed pass-wise so a slab run needs two vector global
sums per step.  It must reproduce the reference's Newton/GMRES counts and
states on the run goldens, unsplit and on emulated slabs (hard
part 6)."""

import numpy as np
import pytest
import torch

from conftest import golden, golden_meta, rel

pytestmark = pytest.mark.gpu
META = golden_meta()


def _steps(uc, grp, mesh, k, m, state, cfg):
    from paper_2006_16764_b200.parallel import SlabPrecond, SlabResidual

    sp = grp.space if grp is not None else None
    prev = sp.clone(state) if sp else state.clone()
    counts = []
    for n in range(m["steps"]):
        th = 1.0 if n < m["startup_steps"] else m["theta"]
        sc = uc.ThetaScheme(th, m["dt"], n)
        if grp is None:
            pc = uc.build_precond(mesh, k, state, sc, uc.PrecondConfig(ordering="multicolor"))
            res = uc.TimestepResidual(mesh, k, state, prev, sc)
        else:
            pc = SlabPrecond(grp, state, sc, uc.PrecondConfig(ordering="multicolor"))
            res = SlabResidual(grp, state, prev, sc)
        u, rep = uc.newton_solve(res, state, cfg, precond_apply=pc.apply)
        assert rep.converged
        counts.append((rep.iterations, rep.total_gmres))
        prev, state = state, u
    return counts, state


@pytest.mark.parametrize("run", ["al2d_256x64_10", "fg3d_16_3", "fg2d_128_10"])
@pytest.mark.parametrize("slabs", [0, 2])
def test_cgs2_reproduces_reference_counts(run, slabs):
    import paper_2006_16764_b200 as uc
    from paper_2006_16764_b200 import models
    from paper_2006_16764_b200.parallel import SlabGroup, slab_bounds

    m = META["run_" + run]
    mesh = uc.build_mesh(m["dim"], m["extents"], m["counts"])
    if m["model"] == "free_growth":
        k = uc.FreeGrowthKernel()
        u0 = models.seed_initial_condition(mesh, k.params)
    else:
        k = uc.AlloyKernel()
        u0 = models.directional_initial_condition(mesh, k.params, amplitude=0.5, seed=0, smooth=True)
    cfg = uc.NewtonConfig(gmres=uc.GmresConfig(orthogonalization="cgs2"))
    grp = SlabGroup(mesh, k, slab_bounds(mesh, slabs, 4)) if slabs else None
    state = grp.split(torch.tensor(u0, device="cuda")) if grp else torch.tensor(u0, device="cuda")
    counts, state = _steps(uc, grp, mesh, k, m, state, cfg)
    assert [c[0] for c in counts] == m["newton"]
    assert [c[1] for c in counts] == m["gmres"]
    final = grp.join(state) if grp else state
    try:
        ref = golden("run_" + run)["state"]
    except FileNotFoundError:
        return
    assert rel(final.cpu().numpy(), ref) <= 1e-8


def test_cgs2_config_validation():
    import paper_2006_16764_b200 as uc

    with pytest.raises(ValueError):
        uc.GmresConfig(orthogonalization="householder")


@pytest.mark.parametrize("n", [3_000_000, 8_400_000])
def test_cgs2_long_vectors(n):
    """Vectors long enough that the reduction grid is at its cap (k_mdot keeps
    UC_MDOT_B x grid partials) and k >= 8 (several k_mdot launches per pass):
    h and the new basis vector agree with a torch fp64 CGS2 and with MGS."""
    from paper_2006_16764_b200 import device as D

    g = torch.Generator(device="cuda").manual_seed(3)
    k = 11
    A = torch.randn(n, k + 1, device="cuda", dtype=torch.float64, generator=g)
    Q, _ = torch.linalg.qr(A)
    basis = [Q[:, j].contiguous() for j in range(k + 1)]
    w0 = torch.randn(n, device="cuda", dtype=torch.float64, generator=g)
    ref_w = w0.clone()
    h_ref = torch.zeros(k + 1, device="cuda", dtype=torch.float64)
    for _ in range(2):
        hp = torch.stack([b @ ref_w for b in basis])
        ref_w = ref_w - torch.stack(basis, 1) @ hp
        h_ref += hp
    nrm = float(ref_w.norm())
    for cgs2 in (True, False):
        h, v, broke = D.arnoldi(lambda x: w0.clone(), basis, k, 1.0, cgs2=cgs2)
        assert not broke and np.isfinite(h).all()
        assert np.allclose(h[: k + 1], h_ref.cpu().numpy(), rtol=0, atol=1e-9)
        assert abs(h[k + 1] - nrm) <= 1e-9 * nrm
        assert float((v - ref_w / nrm).abs().max()) <= 1e-9
