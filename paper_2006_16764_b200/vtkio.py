"""Legacy-VTK and CSV writers (mirrors undercool/vtkio.py:31-86).

Same signatures and byte-identical files as the reference's writers; the
formatting runs in the native library (csrc/writer.cpp: Python-repr number
formatting on a pool of host threads) instead of one ``repr`` call per value.
Fields may be numpy arrays or CUDA tensors (copied to the host once).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib as L

__all__ = ["write_mesh_vtk", "write_snapshot_vtk", "write_snapshot_csv", "repr_double"]


def _threads() -> int:
    return max(1, min(32, os.cpu_count() or 1))


def _mesh_args(mesh):
    dim = int(mesh.dim)
    if int(getattr(mesh, "order", 1)) != 1:
        raise NotImplementedError("the native writers support Q1 meshes only")
    counts = (C.c_int64 * 3)(*(list(mesh.counts) + [1] * (3 - dim)))
    extents = (C.c_double * 3)(*(list(mesh.extents) + [0.0] * (3 - dim)))
    return dim, counts, extents


def _host(values, n):
    if hasattr(values, "detach"):
        values = values.detach().cpu().numpy()
    a = np.ascontiguousarray(values, dtype=np.float64)
    if a.shape != (n,):
        raise ValueError(f"field has shape {a.shape}, expected ({n},)")
    return a


def _write(mesh, fields: dict, path: str, fmt: int, comment: str = "") -> None:
    lib = L.load()
    dim, counts, extents = _mesh_args(mesh)
    n = int(mesh.n_nodes)
    names = list(fields)
    arrays = [_host(fields[k], n) for k in names]
    cnames = (C.c_char_p * max(1, len(names)))(*[k.encode() for k in names])
    cptrs = (C.c_void_p * max(1, len(names)))(*[a.ctypes.data for a in arrays])
    rc = lib.uc_write_snapshot(os.fsencode(path), fmt, dim, counts, extents, len(names), cnames,
                               cptrs, comment.encode(), _threads())
    L.check(rc, "uc_write_snapshot")


def write_snapshot_csv(mesh, fields: dict, path: str) -> None:
    """vtkio.py:76-86: x,y[,z] and the fields, one node per row."""
    _write(mesh, fields, path, 0)


def write_snapshot_vtk(mesh, fields: dict, path: str, comment: str = "") -> None:
    """vtkio.py:54-73: legacy structured-grid point data."""
    _write(mesh, fields, path, 1, comment)


def write_mesh_vtk(mesh, path: str) -> None:
    """vtkio.py:31-51: unstructured-grid nodes and Q1 cells."""
    lib = L.load()
    dim, counts, extents = _mesh_args(mesh)
    L.check(lib.uc_write_mesh_vtk(os.fsencode(path), dim, counts, extents, _threads()),
            "uc_write_mesh_vtk")


def repr_double(x: float) -> str:
    """The native formatter's repr(float(x)) (for tests)."""
    buf = C.create_string_buffer(40)
    L.check(L.load().uc_repr_double(float(x), buf), "uc_repr_double")
    return buf.value.decode()
