"""assemble_residual(..., elements=subset) on the device (uc_residual_subset)
against the reference run on the same subsets (tests/golden/subset_*.npz,
make_golden.py subset_cases; assembly.py:214-230 with `elements`).

Tolerance: 1e-12 relative, as the full residual (the subset kernel sums each
node's elements in increasing id, the reference in subset order).
"""

import numpy as np
import pytest

from conftest import golden, golden_meta, rel

pytestmark = pytest.mark.gpu

META = golden_meta()
CASES = sorted(k[len("subset_"):] for k in META if k.startswith("subset_"))


@pytest.fixture(scope="module")
def uc():
    import paper_2006_16764_b200 as uc
    return uc


def _kernel(uc, model):
    return uc.FreeGrowthKernel() if model == "free_growth" else uc.AlloyKernel()


@pytest.mark.parametrize("case", CASES)
def test_subset_matches_reference(uc, case):
    m = META["subset_" + case]
    g = golden("subset_" + case)
    mesh = uc.build_mesh(m["dim"], list(m["extents"]), list(m["counts"]))
    k = _kernel(uc, m["model"])
    sc = uc.ThetaScheme(m["theta"], m["dt"], m["step"])
    st = uc.StateHistory(g["new"], g["old"], g["prev"])
    for sub in ("color", "rand"):
        for part in ("old", "new", "full"):
            r = uc.assemble_residual(mesh, k, st, sc, elements=g[sub], part=part)
            assert rel(r, g[f"{sub}_{part}"]) < 1e-12, (sub, part)


@pytest.mark.parametrize("model", ["free_growth", "alloy", "massdiff"])
@pytest.mark.parametrize("dim", [2, 3])
def test_additive_over_colors(uc, model, dim):
    # tests/test_assembly.py:123-137, for every device model
    counts = [6, 5] if dim == 2 else [4, 3, 3]
    mesh = uc.build_mesh(dim, [0.3 * c for c in counts], counts)
    k = uc.MassDiffKernel() if model == "massdiff" else _kernel(uc, model)
    nf = 1 if model == "massdiff" else 2
    rng = np.random.default_rng(1)
    st = uc.StateHistory(*(0.5 + 0.2 * rng.standard_normal(nf * mesh.n_nodes) for _ in range(3)))
    sc = uc.ThetaScheme(0.5, 0.05, 3)
    full = uc.assemble_residual(mesh, k, st, sc)
    parts = sum(uc.assemble_residual(mesh, k, st, sc, elements=cls) for cls in mesh.colors)
    assert np.linalg.norm(full - parts) <= 1e-12 * max(np.linalg.norm(full), 1.0)
    # boolean masks select the same elements
    ne = int(np.prod(counts))
    msk = np.zeros(ne, dtype=bool)
    msk[mesh.colors[0]] = True
    a = uc.assemble_residual(mesh, k, st, sc, elements=msk)
    b = uc.assemble_residual(mesh, k, st, sc, elements=mesh.colors[0])
    assert np.array_equal(a, b)


def test_subset_nonfinite_names_position_in_subset(uc):
    mesh = uc.build_mesh(2, [1.0, 1.0], [4, 4])
    k = uc.FreeGrowthKernel()
    n = mesh.n_nodes
    u = np.concatenate([np.full(n, 0.5), np.ones(n)])
    bad = u.copy()
    bad[12] = np.nan  # node (2, 2): elements 5, 6, 9, 10
    sub = np.array([0, 3, 10, 9])
    with pytest.raises(uc.NonFiniteResidualError) as err:
        uc.assemble_residual(mesh, k, uc.StateHistory(bad, u, u), uc.ThetaScheme(0.5, 1e-3, 3), elements=sub)
    # the reference reports argwhere over the subset's integrands, i.e. the
    # first POSITION holding the node: position 2 (element 10), not element 9
    assert "element 2 " in str(err.value) and "quadrature point 0" in str(err.value)
    with pytest.raises(NotImplementedError):
        uc.assemble_residual(mesh, k, uc.StateHistory(u, u, u), uc.ThetaScheme(0.5, 1e-3, 3),
                             elements=np.array([1, 1]))
