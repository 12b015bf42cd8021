"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
host-side setup (mesh, parameters, ICs) matches the reference's goldens."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden, golden_meta


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "uc_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(uc_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2006_16764_b200 import _lib as L

    lib = L.load()
    declared = _declared_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
        assert name in L.SIGNATURES, name
    assert lib.uc_abi_version() == 1


def test_library_is_sm100a():
    import subprocess

    from paper_2006_16764_b200 import _lib as L

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", L.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_mesh_matches_reference_layout():
    from paper_2006_16764_b200 import build_mesh

    m = build_mesh(2, (0.48, 0.36), (16, 12))
    assert m.node_shape == (17, 13) and m.n_nodes == 221 and m.n_elements == 192
    assert m.spacing == (0.48 / 16, 0.36 / 12)
    # lexicographic, x fastest; tensor-ordered local nodes (mesh.py:209-228)
    assert list(m.conn[0]) == [0, 1, 17, 18]
    assert list(m.conn[16]) == [17, 18, 34, 35]
    assert np.array_equal(m.coords[17], [0.0, 0.03])
    m3 = build_mesh(3, (1, 1, 1), (2, 3, 4))
    assert list(m3.conn[0]) == [0, 1, 3, 4, 12, 13, 15, 16]
    with pytest.raises(ValueError):
        build_mesh(4, (1,), (1,))


def test_initial_conditions_match_reference():
    from paper_2006_16764_b200 import AlloyParams, FreeGrowthParams, build_mesh
    from paper_2006_16764_b200.models import directional_initial_condition, seed_initial_condition

    g = golden("ic")
    meta = golden_meta()["ic"]
    m = build_mesh(2, meta["alloy"]["extents"], meta["alloy"]["counts"])
    ic = directional_initial_condition(m, AlloyParams(), amplitude=0.5, seed=0, smooth=True)
    assert np.array_equal(ic, g["alloy_256x64"])
    m2 = build_mesh(2, meta["seed"]["extents"], meta["seed"]["counts"])
    assert np.array_equal(seed_initial_condition(m2, FreeGrowthParams()), g["seed_128"])


def test_device_params_follow_reference_derivations():
    from paper_2006_16764_b200 import AlloyKernel, FreeGrowthKernel
    from paper_2006_16764_b200.models import device_params

    fg = device_params(FreeGrowthKernel())
    assert fg.bg == 191.82 * (1.0 / 191.82)
    assert fg.tmelt == 1.0 + 0.55 * 1.0
    assert fg.reg == 1.0
    al = device_params(AlloyKernel())
    assert al.dcoef == pytest.approx(6.267, rel=1e-12)
    assert al.reg == 0.05 ** 4 and al.at_reg2 == 0.02 ** 2


def test_unknown_kernel_is_rejected():
    from paper_2006_16764_b200.models import device_params

    class MassDiffKernel:
        n_fields = 1

    with pytest.raises(NotImplementedError):
        device_params(MassDiffKernel())


def test_gauss_constants_bitwise_numpy():
    """The CUDA literals in csrc/uc_common.cuh equal numpy's leggauss(3)."""
    text = open(os.path.join(ROOT, "paper_2006_16764_b200", "csrc", "uc_common.cuh")).read()
    lits = dict(re.findall(r"#define (UC_[A-Z0-9]+) (0x[0-9a-fp.+-]+)", text))
    x, w = np.polynomial.legendre.leggauss(3)
    assert float.fromhex(lits["UC_GW0"]) == w[0] == w[2]
    assert float.fromhex(lits["UC_GW1"]) == w[1]
    assert float.fromhex(lits["UC_LA"]) == (1.0 - x[0]) / 2.0
    assert float.fromhex(lits["UC_LB"]) == (1.0 + x[0]) / 2.0
    assert float.fromhex(lits["UC_EPS0"]) == np.sqrt(np.finfo(float).eps)


def test_run_config_validation_mirrors_reference():
    """config.py:74-97 checks run before any device work (tests/test_driver.py:60-72)."""
    from paper_2006_16764_b200.config import MeshConfig, RunConfig, TimeConfig, default_config
    from paper_2006_16764_b200.driver import simulate
    from paper_2006_16764_b200.errors import ConfigError

    for mutate in (lambda c: setattr(c, "model", "plasma"),
                   lambda c: setattr(c.mesh, "counts", (4,)),
                   lambda c: setattr(c.time, "theta", 2.0),
                   lambda c: setattr(c.time, "dt", -1.0),
                   lambda c: setattr(c.precond, "ordering", "random")):
        cfg = RunConfig()
        mutate(cfg)
        with pytest.raises(ConfigError):
            simulate(cfg)
    a = default_config("alloy")
    assert a.mesh == MeshConfig(dimension=2, extents=(204.8, 51.2), counts=(256, 64))
    assert a.time == TimeConfig(theta=0.5, dt=0.002, t_final=10.0, startup_dt=0.002)


def test_timescales_mirror_reference():
    from paper_2006_16764_b200 import AlloyKernel, FreeGrowthKernel
    from paper_2006_16764_b200.stepping import timescales

    fg = timescales(FreeGrowthKernel().scales(), 0.03, 2.25e-4, dim=2).as_dict()
    assert fg["dt_heat"] == 0.03 * 0.03 / (4.0 * 4.0) and fg["dt_solute"] == float("inf")
    al = timescales(AlloyKernel().scales(), 0.8, 0.002, dim=2).as_dict()
    p = AlloyKernel().params
    assert al["kappa"] == 2.0 * 0.002 * p.solute_d0 / (0.8 * 0.8)


def test_element_node_weights_sum_to_element_volume():
    from paper_2006_16764_b200 import build_mesh
    from paper_2006_16764_b200.driver import element_node_weights

    for dim, ext, cnt in [(2, (0.96, 0.96), (32, 32)), (3, (0.48, 0.36, 0.24), (8, 6, 4))]:
        m = build_mesh(dim, ext, cnt)
        w = element_node_weights(m)
        assert w.shape == (2 ** dim,)
        assert abs(w.sum() - np.prod(m.spacing)) <= 1e-15 * np.prod(m.spacing) * 8


def test_run_config_error_exit_code(tmp_path):
    """tests/test_driver.py:156-160: a bad config returns EXIT_CONFIG before any device work."""
    from paper_2006_16764_b200.config import RunConfig
    from paper_2006_16764_b200.driver import EXIT_CONFIG, run

    cfg = RunConfig()
    cfg.time.dt = -1.0
    cfg.output.directory = str(tmp_path / "out")
    code, res = run(cfg)
    assert code == EXIT_CONFIG and res.status == "config_error"


def test_no_cpu_fallback_without_a_gpu():
    """The product path has no CPU implementation: without a CUDA device every
    compute entry point fails loudly instead of computing on the host."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("checks the no-GPU behaviour")
    import paper_2006_16764_b200 as uc
    from paper_2006_16764_b200 import _lib as L

    mesh = uc.build_mesh(2, (0.96, 0.96), (8, 8))
    k = uc.FreeGrowthKernel()
    st = np.concatenate([np.full(mesh.n_nodes, 0.5), np.ones(mesh.n_nodes)])
    sc = uc.ThetaScheme(0.5, 2.25e-4, 1)
    with pytest.raises((L.UcError, RuntimeError)):
        uc.TimestepResidual(mesh, k, st, st, sc)(st)
    with pytest.raises((L.UcError, RuntimeError)):
        uc.build_precond(mesh, k, st, sc)
