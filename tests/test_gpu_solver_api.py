"""Drop-in behaviour of the solver API on the device, mirroring the properties
the reference's own suite pins (pkg/tests/test_gmres.py, test_newton.py,
test_precond.py).  User operators here are plain numpy callables; the Krylov
vectors live on the GPU and every length-n operation runs in libuc_b200.so."""

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def uc():
    import paper_2006_16764_b200 as uc
    return uc


def laplace2d(n):
    t = sp.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(n, n))
    i = sp.identity(n)
    return (sp.kron(i, t) + sp.kron(t, i)).tocsr()


# ---- GMRES (krylov.py:81-208) -------------------------------------------
def test_gmres_identity_and_perfect_preconditioner(uc):
    rhs = np.arange(1.0, 6.0)
    r = uc.gmres_solve(lambda v: v, rhs, tol=1e-12)
    assert r.converged and r.iterations == 1 and np.allclose(r.x, rhs)
    d = np.arange(1.0, 11.0)
    r = uc.gmres_solve(lambda v: d * v, np.ones(10), tol=1e-12, apply_minv=lambda v: v / d)
    assert r.converged and r.iterations == 1 and np.allclose(d * r.x, 1.0, atol=1e-10)


def test_gmres_zero_rhs(uc):
    r = uc.gmres_solve(lambda v: 2 * v, np.zeros(7), tol=1e-10)
    assert r.converged and r.iterations == 0 and np.all(r.x == 0.0)


def test_gmres_laplacian_vs_direct(uc):
    a = laplace2d(100)
    rhs = np.random.default_rng(17).standard_normal(a.shape[0])
    r = uc.gmres_solve(lambda v: a @ v, rhs, tol=1e-8)
    assert r.converged
    direct = spla.spsolve(a.tocsc(), rhs)
    assert np.linalg.norm(r.x - direct) / np.linalg.norm(direct) < 1e-6


def test_gmres_right_preconditioning_true_residual(uc):
    a = laplace2d(20)
    diag = a.diagonal()
    rhs = np.random.default_rng(18).standard_normal(a.shape[0])
    r = uc.gmres_solve(lambda v: a @ v, rhs, tol=1e-7, apply_minv=lambda v: v / diag)
    assert r.converged
    assert np.linalg.norm(a @ r.x - rhs) <= 1e-7 * np.linalg.norm(rhs) * (1 + 1e-9)


def test_gmres_matches_scipy(uc):
    rng = np.random.default_rng(19)
    for _ in range(3):
        a = np.eye(50) + 0.2 * rng.standard_normal((50, 50))
        rhs = rng.standard_normal(50)
        mine = uc.gmres_solve(lambda v: a @ v, rhs, tol=1e-10)
        ref, info = spla.gmres(a, rhs, rtol=1e-10, restart=200, maxiter=2000)
        assert info == 0 and mine.converged
        assert np.linalg.norm(mine.x - ref) / np.linalg.norm(ref) < 1e-8


def test_gmres_restart_maxiter_and_apply_count(uc):
    a = laplace2d(12)
    rhs = np.random.default_rng(20).standard_normal(a.shape[0])
    r = uc.gmres_solve(lambda v: a @ v, rhs, tol=1e-8, config=uc.GmresConfig(restart=10, max_iterations=5000))
    assert r.converged and r.cycles > 1
    r = uc.gmres_solve(lambda v: a @ v, rhs, tol=1e-14, config=uc.GmresConfig(restart=5, max_iterations=10))
    assert not r.converged and r.iterations == 10 and np.isfinite(r.residual_norm)
    a = laplace2d(10)
    rhs = np.random.default_rng(22).standard_normal(a.shape[0])
    calls = {"n": 0}

    def minv(v):
        calls["n"] += 1
        return v / a.diagonal()

    r = uc.gmres_solve(lambda v: a @ v, rhs, tol=1e-9, apply_minv=minv)
    assert r.converged and calls["n"] == r.precond_applies == r.iterations + r.cycles


def test_arnoldi_orthonormal_and_hessenberg(uc):
    rng = np.random.default_rng(23)
    n, m = 40, 20
    a = rng.standard_normal((n, n))
    basis = np.zeros((m + 1, n))
    r0 = rng.standard_normal(n)
    beta = np.linalg.norm(r0)
    basis[0] = r0 / beta
    hess = np.zeros((m + 1, m))
    for k in range(m):
        h, vnew, broke = uc.arnoldi_step(lambda v: a @ v, basis, k, beta)
        assert not broke
        hess[: k + 2, k] = h
        basis[k + 1] = vnew
    assert np.abs(basis @ basis.T - np.eye(m + 1)).max() < 1e-10
    assert np.linalg.norm(a @ basis[:m].T - basis.T @ hess) <= 1e-10 * np.linalg.norm(a)


def test_arnoldi_breakdown_and_exact_solve(uc):
    d = np.array([3.0, 1.0, 2.0])
    basis = np.zeros((2, 3))
    basis[0] = [1.0, 0.0, 0.0]
    h, vnew, broke = uc.arnoldi_step(lambda v: d * v, basis, 0, 1.0)
    assert broke and vnew is None and h[0] == pytest.approx(3.0)
    r = uc.gmres_solve(lambda v: d * v, np.array([2.0, 0.0, 0.0]), tol=1e-12)
    assert r.converged and np.allclose(r.x, [2.0 / 3.0, 0.0, 0.0])


def test_linear_operator_wrapper(uc):
    r = uc.gmres_solve(uc.LinearOperator(n=4, apply=lambda v: 3.0 * v), np.ones(4), tol=1e-12)
    assert r.converged and np.allclose(r.x, 1.0 / 3.0)


# ---- Newton / JFNK (newton.py:73-198) -----------------------------------
def test_matvec_identity_linear_zero(uc):
    f = lambda u: u.copy()  # noqa: E731
    u, v = np.array([1.0, -2.0, 3.0]), np.array([0.5, 0.25, -1.0])
    assert np.linalg.norm(uc.jfnk_matvec(f, u, f(u), v) - v) / np.linalg.norm(v) < 1e-8
    rng = np.random.default_rng(13)
    A = rng.standard_normal((12, 12))
    u, v = rng.standard_normal(12), rng.standard_normal(12)
    jv = uc.jfnk_matvec(lambda w: A @ w, u, A @ u, v)
    assert np.linalg.norm(jv - A @ v) / np.linalg.norm(A @ v) < 1e-7
    g = lambda w: w ** 2  # noqa: E731
    assert np.all(uc.jfnk_matvec(g, np.ones(4), g(np.ones(4)), np.zeros(4)) == 0.0)


def test_matvec_against_dense_fd_jacobian(uc):
    mesh = uc.build_mesh(2, [0.12, 0.12], [4, 4])
    k = uc.FreeGrowthKernel()
    rng = np.random.default_rng(14)
    n2 = 2 * mesh.n_nodes
    u0 = uc.join_fields(0.5 + 0.25 * rng.standard_normal(mesh.n_nodes),
                        1.0 + 0.2 * rng.standard_normal(mesh.n_nodes))
    res = uc.TimestepResidual(mesh, k, u0.copy(), u0.copy(), uc.ThetaScheme(0.5, 2.25e-4, 0))
    f0 = res(u0)
    jac = np.zeros((n2, n2))
    for j in range(n2):
        d = np.zeros(n2)
        d[j] = 1.0
        eps = np.sqrt(np.finfo(float).eps) * (1.0 + abs(u0[j]))
        jac[:, j] = (res(u0 + eps * d) - f0) / eps
    for _ in range(10):
        v = rng.standard_normal(n2)
        ref = jac @ v
        assert np.linalg.norm(uc.jfnk_matvec(res, u0, f0, v) - ref) / np.linalg.norm(ref) <= 1e-5


def test_newton_scalar_quadratic_and_spd(uc):
    u, rep = uc.newton_solve(lambda w: w * w - 4.0, np.full(5, 3.0))
    assert rep.converged and rep.iterations <= 8 and np.allclose(u, 2.0, atol=1e-5)
    norms = rep.residual_norms
    assert max(norms[i + 1] / norms[i] ** 2 for i in range(1, len(norms) - 1)) < 1.0
    rng = np.random.default_rng(15)
    m = rng.standard_normal((20, 20))
    a = m @ m.T + 20 * np.eye(20)
    b = rng.standard_normal(20)
    cfg = uc.NewtonConfig(eta0=1e-12, eta_min=1e-13, eta_max=1e-12)
    u, rep = uc.newton_solve(lambda w: a @ w - b, np.zeros(20), cfg)
    assert rep.converged and rep.iterations == 1 and np.linalg.norm(a @ u - b) < 1e-6 * np.linalg.norm(b)


def test_forcing_and_config(uc):
    cfg = uc.NewtonConfig()
    assert uc.forcing_update(0.01, 1.0, 1.0, cfg) == pytest.approx(0.01)
    assert uc.forcing_update(0.1, 0.01, 1.0, cfg) == pytest.approx(0.01)
    assert uc.forcing_update(0.01, 1e-12, 1.0, cfg) == pytest.approx(max(0.9 * 0.01 ** 1.5, 1e-6))
    for bad in (dict(forcing_gamma=0.0), dict(forcing_power=2.5), dict(eta_min=0.5, eta0=0.1)):
        with pytest.raises(ValueError):
            uc.NewtonConfig(**bad)


def test_newton_backtracking_failure_and_edges(uc):
    u, rep = uc.newton_solve(lambda w: np.arctan(4.0 * w), np.full(3, 2.0), uc.NewtonConfig(rel_tol=1e-10))
    assert rep.converged and min(rep.step_lengths) < 1.0
    assert all(b <= a + 1e-15 for a, b in zip(rep.residual_norms, rep.residual_norms[1:]))
    u, rep = uc.newton_solve(lambda w: np.sign(w) * (1.0 + np.abs(w)), np.array([2.0]),
                             uc.NewtonConfig(max_iterations=5))
    assert not rep.converged and rep.failure_reason
    u, rep = uc.newton_solve(lambda w: w - 1.0, np.ones(4))
    assert rep.converged and rep.iterations == 0
    u, rep = uc.newton_solve(lambda w: w, np.array([1.0, np.nan]))
    assert not rep.converged and "non-finite" in rep.failure_reason


def test_newton_determinism_bitwise(uc):
    from paper_2006_16764_b200.models import seed_initial_condition

    mesh = uc.build_mesh(2, [0.96, 0.96], [16, 16])
    k = uc.FreeGrowthKernel()
    u0 = seed_initial_condition(mesh, k.params)
    outs = []
    for _ in range(2):
        res = uc.TimestepResidual(mesh, k, u0.copy(), u0.copy(), uc.ThetaScheme(0.5, 2.25e-4, 0))
        u, rep = uc.newton_solve(res, u0.copy())
        outs.append((u, rep.gmres_iterations, rep.residual_norms))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1] and outs[0][2] == outs[1][2]


def test_newton_count_baseline_150(uc):
    """Reference regression baseline (test_newton.py:176-193): <= 6 Newton."""
    from paper_2006_16764_b200.models import seed_initial_condition

    mesh = uc.build_mesh(2, [4.5, 4.5], [150, 150])
    k = uc.FreeGrowthKernel()
    u0 = seed_initial_condition(mesh, k.params)
    sc = uc.ThetaScheme(0.5, 2.25e-4, 0)
    pc = uc.build_precond(mesh, k, u0, sc, uc.PrecondConfig(ordering="multicolor"))
    u, rep = uc.newton_solve(uc.TimestepResidual(mesh, k, u0, u0.copy(), sc), u0, uc.NewtonConfig(),
                             precond_apply=pc.apply)
    assert rep.converged and rep.iterations <= 6


# ---- block preconditioner (precond.py:225-299) --------------------------
def _seed_pc(uc, nx, kind, theta=0.5, dt=2.25e-4, radius=0.1, **kw):
    from paper_2006_16764_b200.models import seed_initial_condition

    mesh = uc.build_mesh(2, [0.03 * nx, 0.03 * nx], [nx, nx])
    k = uc.FreeGrowthKernel()
    u = seed_initial_condition(mesh, k.params, radius=radius)
    return mesh, k, u, uc.build_precond(mesh, k, u, uc.ThetaScheme(theta, dt, 0),
                                        uc.PrecondConfig(kind=kind, ordering="multicolor", **kw))


@pytest.mark.parametrize("kind", ["identity", "jacobi", "sgs", "vcycle"])
def test_precond_linear_and_zero_preserving(uc, kind):
    mesh, k, u, pc = _seed_pc(uc, 16, kind)
    rng = np.random.default_rng(28)
    v, w = rng.standard_normal(2 * mesh.n_nodes), rng.standard_normal(2 * mesh.n_nodes)
    rhs = 2.5 * pc.apply(v) - 1.5 * pc.apply(w)
    assert np.allclose(pc.apply(2.5 * v - 1.5 * w), rhs, atol=1e-11 * np.abs(rhs).max())
    assert np.all(pc.apply(np.zeros(2 * mesh.n_nodes)) == 0.0)
    assert uc.apply_precond(pc, v).shape == v.shape


def test_precond_fixed_between_rebuilds(uc):
    mesh, k, u, pc = _seed_pc(uc, 8, "vcycle", dt=1e-4)
    v = np.random.default_rng(29).standard_normal(2 * mesh.n_nodes)
    first = pc.apply(v)
    u += 100.0  # mutate the state the blocks were built from
    assert np.array_equal(first, pc.apply(v))


def test_vcycle_contraction_and_levels(uc):
    """Heat block (constant coefficients) of a free-growth build: the V-cycle
    error propagator I - B A contracts (rho < 0.5) and the hierarchy has the
    reference's level sizes [289, 81, 25, 9] at nx = 16."""
    mesh, k, u, pc = _seed_pc(uc, 16, "vcycle", levels=3)
    n = mesh.n_nodes
    a = pc.level_matrix(0, 1)
    rng = np.random.default_rng(30)
    e = rng.standard_normal(n)
    e /= np.linalg.norm(e)
    rho = 1.0
    for _ in range(12):
        e = e - pc.apply(np.concatenate([np.zeros(n), a @ e]))[n:]
        rho = np.linalg.norm(e)
        if rho < 1e-14:
            break
        e /= rho
    assert rho < 0.5
    _, _, _, pc4 = _seed_pc(uc, 16, "vcycle")
    assert [int(np.prod(s)) for s in pc4.level_shapes] == [17 ** 2, 9 ** 2, 5 ** 2, 3 ** 2]
    _, _, _, pc6 = _seed_pc(uc, 6, "vcycle")
    assert len(pc6.level_shapes) == 2


def test_precond_rejects_nonpositive_diagonal(uc):
    mesh = uc.build_mesh(2, [6.4, 6.4], [8, 8])
    k = uc.AlloyKernel()
    n = mesh.n_nodes
    # solute below -1/(1-k): the phase-block mass (1+(1-k)u) g^2/dt is negative
    u = uc.join_fields(np.zeros(n), np.full(n, -2.0))
    with pytest.raises(ValueError):
        uc.build_precond(mesh, k, u, uc.ThetaScheme(0.5, 1e-3, 0), uc.PrecondConfig(ordering="multicolor"))


def test_precond_config_validation(uc):
    for bad in (dict(kind="amg"), dict(ordering="diagonal"), dict(rebuild="never")):
        with pytest.raises(ValueError):
            uc.PrecondConfig(**bad)
    mesh = uc.build_mesh(2, [0.24, 0.24], [8, 8])
    with pytest.raises(NotImplementedError):
        uc.build_precond(mesh, uc.FreeGrowthKernel(), np.zeros(2 * mesh.n_nodes),
                         uc.ThetaScheme(0.5, 1e-4, 0), uc.PrecondConfig(kind="direct"))
