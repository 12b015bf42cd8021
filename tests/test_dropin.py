"""The rest of the reference's assembly/mesh surface:
eval_basis (mesh.py:259-265), frozen_quad_state (assembly.py:193-211) and
assemble_field_matrix (assembly.py:271-303), against outputs of the reference
itself (tests/golden/make_golden.py dropin_cases)."""

import numpy as np
import pytest

from conftest import golden, golden_meta, rel

META = golden_meta()
CASES = ["fg2d", "al3d"]


def _mesh(uc, name):
    m = META["dropin_" + name]
    k = uc.FreeGrowthKernel() if m["model"] == "free_growth" else uc.AlloyKernel()
    return m, uc.build_mesh(m["dim"], m["extents"], m["counts"]), k


@pytest.mark.parametrize("name", CASES)
def test_eval_basis_tables(name):
    import paper_2006_16764_b200 as uc

    m, mesh, _ = _mesh(uc, name)
    g = golden("dropin_" + name)
    for ppa in (2, 3, 4):
        b = uc.eval_basis(mesh, 0, uc.gauss_rule(m["dim"], ppa))
        assert np.array_equal(b.values, g[f"basis{ppa}_values"])
        assert np.array_equal(b.gradients, g[f"basis{ppa}_gradients"])
        assert np.array_equal(b.jxw, g[f"basis{ppa}_jxw"])
    with pytest.raises(IndexError):
        uc.eval_basis(mesh, mesh.n_elements)
    pts, wts = uc.gauss_rule(m["dim"])  # still unpacks as (points, weights)
    assert pts.shape == (3 ** m["dim"], m["dim"]) and wts.shape == (3 ** m["dim"],)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_frozen_quad_state(name):
    import torch

    import paper_2006_16764_b200 as uc

    m, mesh, k = _mesh(uc, name)
    g = golden("dropin_" + name)
    sc = uc.ThetaScheme(m["theta"], m["dt"], m["step"])
    qs = uc.frozen_quad_state(mesh, k, g["state"], sc)
    assert isinstance(qs.val_new[0], np.ndarray)
    assert rel(qs.coords, g["coords"]) <= 1e-15
    for f in range(2):
        assert rel(qs.val_new[f], g[f"val{f}"]) <= 1e-13
        for d in range(m["dim"]):
            assert rel(qs.grad_new[f][d], g[f"grad{f}_{d}"]) <= 1e-13
    # device in -> device out
    qd = uc.frozen_quad_state(mesh, k, torch.tensor(g["state"], device="cuda"), sc)
    assert qd.val_new[1].is_cuda and rel(qd.val_new[1].cpu().numpy(), g["val1"]) <= 1e-13
    assert qs.t_new == sc.t_new and qs.part == "new"


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("tag", ["qp", "scalar", "rule2"])
def test_assemble_field_matrix(name, tag):
    import torch

    import paper_2006_16764_b200 as uc

    m, mesh, _ = _mesh(uc, name)
    g = golden("dropin_" + name)
    dim = m["dim"]
    args = {"qp": (g["cm"], g["cd"], None), "scalar": (2.5, 0.75, None),
            "rule2": (g["cm"][:, : 2 ** dim] * 1.0, 0.75, uc.gauss_rule(dim, 2))}[tag]
    mat = uc.assemble_field_matrix(mesh, *args)
    assert np.array_equal(mat.indptr, g[f"M{tag}_indptr"])
    assert np.array_equal(mat.indices, g[f"M{tag}_indices"])
    assert rel(mat.data, g[f"M{tag}_data"]) <= 1e-12
    if tag == "qp":
        dm = uc.assemble_field_matrix(mesh, torch.tensor(g["cm"], device="cuda"), torch.tensor(g["cd"], device="cuda"))
        assert dm.is_cuda and dm.layout == torch.sparse_csr
        assert rel(dm.values().cpu().numpy(), g["Mqp_data"]) <= 1e-12
        with pytest.raises(ValueError):
            uc.assemble_field_matrix(mesh, g["cm"][:, :2], 1.0)
