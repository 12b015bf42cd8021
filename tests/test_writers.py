"""Native snapshot / mesh / config writers vs the reference's files
(vtkio.py:31-86, config.py:150-174), byte for byte.  Host-only: the
formatter is C++ in the same library and runs without a GPU."""

import gzip
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden, golden_meta

META = golden_meta()
W = META["writers"]
WDIR = os.path.join(GOLDEN, "writers")


def _ref(name):
    with open(os.path.join(WDIR, name + ".gz"), "rb") as fh:
        return gzip.decompress(fh.read())


def test_repr_formatter_matches_python():
    from paper_2006_16764_b200.vtkio import repr_double

    rng = np.random.default_rng(5)
    vals = list(rng.standard_normal(3000)) + list(rng.standard_normal(3000) * 10.0 ** rng.integers(-40, 40, 3000))
    vals += list(rng.integers(0, 2 ** 63, 6000, dtype=np.int64).view(np.float64))
    vals += [0.0, -0.0, 1e16, 1e15, 9999999999999998.0, 1e-4, 1e-5, 5e-324, 1.7976931348623157e308,
             float("inf"), float("-inf"), float("nan"), 0.1, 1.0, 2.5e-5, 0.03 * 7, 123456789012345678.0]
    bad = [(repr(float(v)), repr_double(v)) for v in vals if repr(float(v)) != repr_double(v)]
    assert not bad, bad[:5]


@pytest.mark.parametrize("case", ["fg2d_32_10", "al2d_128x32_10", "fg3d_16_3"])
def test_snapshot_files_byte_identical(case, tmp_path):
    from paper_2006_16764_b200 import build_mesh
    from paper_2006_16764_b200.vtkio import write_snapshot_csv, write_snapshot_vtk

    m = W[case]
    mesh = build_mesh(m["dim"], m["extents"], m["counts"])
    st = golden("driver_" + case)["state"]
    n = mesh.n_nodes
    names = m["fields"]
    fields = {names[0]: st[:n], names[1]: st[n:]}
    if "composition" in names:
        fields["composition"] = np.load(os.path.join(WDIR, f"composition_{case}.npz"))["composition"]
    write_snapshot_csv(mesh, fields, str(tmp_path / "s.csv"))
    write_snapshot_vtk(mesh, fields, str(tmp_path / "s.vtk"), comment=f"t = {m['t']!r}")
    assert (tmp_path / "s.csv").read_bytes() == _ref(f"snapshot_{case}.csv")
    assert (tmp_path / "s.vtk").read_bytes() == _ref(f"snapshot_{case}.vtk")


@pytest.mark.parametrize("case", ["mesh2d_6x4", "mesh3d_4x3x2"])
def test_mesh_vtk_byte_identical(case, tmp_path):
    from paper_2006_16764_b200 import build_mesh
    from paper_2006_16764_b200.vtkio import write_mesh_vtk

    m = W[case]
    write_mesh_vtk(build_mesh(m["dim"], m["extents"], m["counts"]), str(tmp_path / "m.vtk"))
    assert (tmp_path / "m.vtk").read_bytes() == _ref(case + ".vtk")


@pytest.mark.parametrize("model", ["free_growth", "alloy"])
def test_config_used_byte_identical(model):
    from paper_2006_16764_b200.config import default_config, save_config

    assert save_config(default_config(model)).encode() == _ref(f"config_{model}.used")


def test_writer_rejects_bad_arguments(tmp_path):
    from paper_2006_16764_b200 import _lib as L
    from paper_2006_16764_b200 import build_mesh
    from paper_2006_16764_b200.vtkio import write_snapshot_csv

    mesh = build_mesh(2, (1.0, 1.0), (4, 4))
    with pytest.raises(ValueError):
        write_snapshot_csv(mesh, {"phi": np.zeros(3)}, str(tmp_path / "x.csv"))
    with pytest.raises(L.UcError):
        write_snapshot_csv(mesh, {"phi": np.zeros(25)}, str(tmp_path / "nodir" / "x.csv"))
