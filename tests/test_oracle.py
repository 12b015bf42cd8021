"""The CPU oracle (oracle/) pinned against the reference's golden vectors.

Runs on CPU only; this is what makes the oracle trustworthy as the checker
for the device tests at sizes the goldens do not cover.
"""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT, golden, golden_meta, rel

sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

META = golden_meta()
RES_CASES = sorted(k[len("residual_"):] for k in META if k.startswith("residual_"))
PC_CASES = sorted(k[len("precond_"):] for k in META if k.startswith("precond_"))


def _params(model, normalized=True):
    from paper_2006_16764_b200 import AlloyParams, FreeGrowthParams

    return FreeGrowthParams() if model == "free_growth" else AlloyParams(antitrapping_normalized=normalized)


def _problem(m):
    return O.Problem(m["dim"], m["extents"], m["counts"], m["model"],
                     _params(m["model"], m.get("normalized", True)), m["theta"], m["dt"], m["step"])


@pytest.mark.parametrize("case", RES_CASES)
def test_oracle_residual_and_jv(case):
    m = META["residual_" + case]
    g = golden("residual_" + case)
    p = _problem(m)
    fixed = p.begin(g["old"], g["prev"])
    assert rel(fixed, g["fixed"]) <= 1e-12
    f = p.residual(g["new"])
    assert rel(f, g["f_call"]) <= 1e-12
    assert rel(p.assemble("new", g["new"], g["old"], g["prev"]), g["f_new"]) <= 1e-12
    jv, eps = p.jv(g["new"], g["f_call"], g["v"])
    assert eps == pytest.approx(float(g["eps"][0]), rel=1e-14)
    assert rel(jv, g["jv"]) <= 1e-6


@pytest.mark.parametrize("case", PC_CASES)
def test_oracle_preconditioner(case):
    import scipy.sparse as sp

    m = META["precond_" + case]
    g = golden("precond_" + case)
    p = _problem(m)
    n = p.N
    for kind in ("identity", "jacobi", "sgs", "vcycle"):
        pc = O.BlockPC(p, g["state"], kind=kind)
        assert rel(pc(g["v"]), g[f"apply_{kind}"]) <= 1e-12, kind
    pc = O.BlockPC(p, g["state"])
    for b in range(2):
        for lvl, h in enumerate(pc.blocks[b].mats):
            key = f"A{b}" if lvl == 0 else f"L{lvl}_A{b}"
            nl = m["levels"][lvl]
            ref = sp.csr_matrix((g[key + "_data"], g[key + "_indices"], g[key + "_indptr"]),
                                shape=(nl, nl)).toarray()
            # dense form of the stencil
            mine = np.zeros_like(ref)
            shape = pc.blocks[b].shapes[lvl]
            d = len(shape)
            for row in range(nl):
                c = [(row // int(np.prod(shape[:a]))) % shape[a] for a in range(d)]
                for k in range(3 ** d):
                    o = [k % 3 - 1, (k // 3) % 3 - 1, k // 9 - 1][:d]
                    j = [c[a] + o[a] for a in range(d)]
                    if all(0 <= j[a] < shape[a] for a in range(d)):
                        col = sum(j[a] * int(np.prod(shape[:a])) for a in range(d))
                        mine[row, col] = h[row, k]
            assert np.abs(mine - ref).max() <= 1e-12 * np.abs(ref).max()
    assert [int(np.prod(s)) for s in pc.blocks[0].shapes] == m["levels"]
    small = O.BlockPC(p, g["state"], sweeps=1, cycles=1, levels=2, coarse_sweeps=3)
    assert rel(small(g["v"]), g["apply_vcycle_small"]) <= 1e-12
    assert n == g["v"].size // 2


def test_oracle_newton_counts():
    from paper_2006_16764_b200.models import seed_initial_condition
    from paper_2006_16764_b200 import FreeGrowthParams, build_mesh

    m = META["newton_fg2d_32"]
    g = golden("newton_fg2d_32")
    mesh = build_mesh(2, (0.96, 0.96), (32, 32))
    u0 = seed_initial_condition(mesh, FreeGrowthParams(), radius=0.3)
    p = O.Problem(2, (0.96, 0.96), (32, 32), "free_growth", FreeGrowthParams(), 1.0, 2.25e-4, 0)
    p.begin(u0, u0)
    pc = O.BlockPC(p, u0)
    u, rep = O.newton(p, u0, pc)
    assert rep["iterations"] == m["iterations"]
    assert rep["gmres"] == m["gmres"]
    assert rel(u, g["u"]) <= 1e-8


def test_oracle_time_steps_fg3d():
    """3 steps of 3D free growth: counts [4,3,3] / [18,12,10] as the reference."""
    from paper_2006_16764_b200.models import seed_initial_condition
    from paper_2006_16764_b200 import FreeGrowthParams, build_mesh

    m = META["run_fg3d_16_3"]
    mesh = build_mesh(3, m["extents"], m["counts"])
    state = seed_initial_condition(mesh, FreeGrowthParams())
    prev = state.copy()
    newton, gm = [], []
    for n in range(m["steps"]):
        th = 1.0 if n < m["startup_steps"] else m["theta"]
        p = O.Problem(3, m["extents"], m["counts"], "free_growth", FreeGrowthParams(), th, m["dt"], n)
        pc = O.BlockPC(p, state)
        p.begin(state, prev)
        u, rep = O.newton(p, state, pc)
        newton.append(rep["iterations"])
        gm.append(sum(rep["gmres"]))
        prev, state = state, u
    assert newton == m["newton"] and gm == m["gmres"]
    assert rel(state, golden("run_fg3d_16_3")["state"]) <= 1e-8


DIAG_CASES = sorted(k[len("diag_"):] for k in META if k.startswith("diag_") and k != "diag_tips_150")


@pytest.mark.parametrize("case", DIAG_CASES)
def test_oracle_step_diagnostics(case):
    """Balance integrals, total solute and tip (driver.py:76-98,
    diagnostics.py:69-89) against the reference on the seeded states."""
    m = META["residual_" + case]
    d = META["diag_" + case]
    g = golden("residual_" + case)
    spacing = [e / c for e, c in zip(m["extents"], m["counts"])]
    st, sn, so = O.balance_integrals(m["counts"], spacing, g["new"], g["old"], g["prev"])
    assert st == pytest.approx(d["w_dT"], rel=1e-13, abs=1e-17)
    assert sn == pytest.approx(d["w_dphi_new"], rel=1e-13, abs=1e-17)
    assert so == pytest.approx(d["w_dphi_old"], rel=1e-13, abs=1e-17)
    if "total_solute" in d:
        p = _params(m["model"], m.get("normalized", True))
        assert O.total_solute(m["counts"], spacing, g["new"], p.composition, p.partition) == \
            pytest.approx(d["total_solute"], rel=1e-13)
    if "x_tip" in d:
        n = g["new"].size // 2
        level = 0.5 if m["model"] == "free_growth" else 0.0
        tip, found = O.extract_tip(g["new"][: m["counts"][0] + 1], m["extents"][0], level)
        assert (tip, found) == (d["x_tip"], d["found"])
        assert n > 0


def test_oracle_tip_profiles():
    xs = np.linspace(0.0, 4.5, 151)
    prof = {
        "step": np.where(xs < 1.234, 1.0, 0.0),
        "tanh": 0.5 * (1.0 - np.tanh((xs - 2.71) / 0.1)),
        "none": np.ones_like(xs),
        "exact": np.where(xs < 1.5, 1.0, np.where(np.isclose(xs, 1.5), 0.5, 0.0)),
    }
    for name, want in META["diag_tips_150"].items():
        assert O.extract_tip(prof[name], 4.5, 0.5) == (want["x_tip"], want["found"]), name
