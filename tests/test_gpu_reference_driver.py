"""The drop-in as a maintainer would use it: the REFERENCE's own time loop
(undercool.driver.simulate, driver.py:134-242 with _advance :101-105 and the
preconditioner build :176-179) with TimestepResidual, newton_solve and
build_precond replaced by this package's, on the reference's own meshes,
kernels, configs and diagnostics.  The reference package is the unmodified
install in baseline/_ref (tools/install_reference.sh; git-ignored, shipped
with the gpurun snapshot).  Counts must equal the reference's goldens and the
final states must agree to 1e-8."""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT, golden, golden_meta, rel

pytestmark = pytest.mark.gpu
META = golden_meta()
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ucref():
    if not os.path.isdir(os.path.join(REF, "undercool")):
        pytest.skip("baseline/_ref not installed (tools/install_reference.sh)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")
    sys.path.insert(0, REF)
    try:
        import undercool
        import undercool.driver as drv
    finally:
        sys.path.remove(REF)
    return undercool, drv


@pytest.mark.parametrize("run", ["fg2d_128_10", "al2d_256x64_10", "fg3d_16_3"])
def test_reference_simulate_with_dropin(ucref, run, monkeypatch):
    import paper_2006_16764_b200 as b200

    undercool, drv = ucref
    from undercool.config import default_config

    m = META["run_" + run]
    cfg = default_config(m["model"])
    cfg.mesh.dimension = m["dim"]
    cfg.mesh.extents = tuple(m["extents"])
    cfg.mesh.counts = tuple(m["counts"])
    cfg.time.dt = m["dt"]
    cfg.time.t_final = m["dt"] * m["steps"]
    cfg.precond.ordering = "multicolor"
    calls = {"res": 0, "pc": 0}

    class Residual(b200.TimestepResidual):
        def __init__(self, *a, **k):
            calls["res"] += 1
            super().__init__(*a, **k)

    def build(*a, **k):
        calls["pc"] += 1
        return b200.build_precond(*a, **k)

    # the substitution a maintainer makes in undercool/driver.py's namespace
    monkeypatch.setattr(drv, "TimestepResidual", Residual)
    monkeypatch.setattr(drv, "newton_solve", b200.newton_solve)
    monkeypatch.setattr(drv, "build_precond", build)
    res = drv.simulate(cfg)
    assert calls["res"] >= m["steps"] and calls["pc"] >= m["steps"]
    assert res.status == m["status"]
    assert [r["newton_iters"] for r in res.records] == m["newton"]
    assert [r["gmres_iters"] for r in res.records] == m["gmres"]
    assert isinstance(res.state, np.ndarray)
    try:
        ref = golden("run_" + run)["state"]
    except FileNotFoundError:
        return
    assert rel(res.state, ref) <= 1e-8
