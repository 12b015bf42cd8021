"""Structured Q1 meshes described by counts and spacing only.

The device kernels never read coordinates or connectivity: every index is
recomputed from (counts, spacing), which is what lets a 512^3 mesh exist
without the 12 GB of host arrays the reference's build_mesh materialises
(undercool/mesh.py:179-256).  ``coords``/``conn``/``boundary``/``colors`` are
still available, built lazily on the host with the reference's ordering, for
callers and tests that inspect them on small meshes.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["StructuredMesh", "QuadratureRule", "BasisEval", "build_mesh", "gauss_rule", "eval_basis",
           "mesh_descriptor"]


@dataclass(frozen=True)
class QuadratureRule:
    """Tensor Gauss rule on [-1, 1]^dim (mesh.py:26-36); also unpacks as
    (points, weights)."""

    points: np.ndarray   # (nq, dim)
    weights: np.ndarray  # (nq,)

    @property
    def n_points(self) -> int:
        return self.weights.size

    def __iter__(self):
        return iter((self.points, self.weights))

    def __getitem__(self, i):
        return (self.points, self.weights)[i]

    def __len__(self):
        return 2


@dataclass
class BasisEval:
    """Shape functions at the quadrature points of one (every) element
    (mesh.py:39-50): physical gradients, jxw = weight x Jacobian."""

    values: np.ndarray     # (nq, nloc)
    gradients: np.ndarray  # (nq, nloc, dim)
    jxw: np.ndarray        # (nq,)


def _lagrange_1d(order: int, x):
    """1D Lagrange basis on [-1, 1] (mesh.py:63-79), same arithmetic."""
    x = np.asarray(x, dtype=float)
    if order == 1:
        vals = np.stack([(1.0 - x) / 2.0, (1.0 + x) / 2.0], axis=-1)
        ders = np.stack([-0.5 * np.ones_like(x), 0.5 * np.ones_like(x)], axis=-1)
    elif order == 2:
        vals = np.stack([x * (x - 1.0) / 2.0, 1.0 - x * x, x * (x + 1.0) / 2.0], axis=-1)
        ders = np.stack([x - 0.5, -2.0 * x, x + 0.5], axis=-1)
    else:
        raise ValueError(f"unsupported element order {order}")
    return vals, ders


class StructuredMesh:
    def __init__(self, dim, extents, counts, order=1):
        self.dim = dim
        self.extents = tuple(float(e) for e in extents)
        self.counts = tuple(int(c) for c in counts)
        self.order = order
        # spacing exactly as the reference computes it (mesh.py:205)
        self.spacing = tuple(e / c for e, c in zip(self.extents, self.counts))
        self.node_shape = tuple(order * c + 1 for c in self.counts)
        self._lazy = {}

    # -- sizes ------------------------------------------------------------
    @property
    def n_nodes(self) -> int:
        return int(np.prod(self.node_shape))

    @property
    def n_elements(self) -> int:
        return int(np.prod(self.counts))

    @property
    def nodes_per_element(self) -> int:
        return (self.order + 1) ** self.dim

    # -- lazily materialised host views (small meshes / tests) ------------
    @property
    def coords(self) -> np.ndarray:
        if "coords" not in self._lazy:
            axes = [np.linspace(0.0, self.extents[a], self.node_shape[a]) for a in range(self.dim)]
            grids = np.meshgrid(*axes[::-1], indexing="ij")
            self._lazy["coords"] = np.stack([g.reshape(-1) for g in grids[::-1]], axis=1)
        return self._lazy["coords"]

    @property
    def conn(self) -> np.ndarray:
        if "conn" not in self._lazy:
            n1 = self.order + 1
            idx = np.indices(self.counts[::-1]).reshape(self.dim, -1)[::-1]  # per-axis element idx
            strides = [1, self.node_shape[0], self.node_shape[0] * self.node_shape[1]]
            conn = np.empty((self.n_elements, n1 ** self.dim), dtype=np.int64)
            for loc in range(n1 ** self.dim):
                nid = np.zeros(self.n_elements, dtype=np.int64)
                for a in range(self.dim):
                    nid += (self.order * idx[a] + (loc // n1 ** a) % n1) * strides[a]
                conn[:, loc] = nid
            self._lazy["conn"] = conn
        return self._lazy["conn"]

    @property
    def boundary(self) -> np.ndarray:
        x = self.coords
        b = np.zeros(x.shape[0], dtype=bool)
        for a in range(self.dim):
            b |= np.isclose(x[:, a], 0.0) | np.isclose(x[:, a], self.extents[a])
        return b

    @property
    def colors(self):
        idx = np.indices(self.counts[::-1]).reshape(self.dim, -1)[::-1]
        cid = sum((idx[a] % 2) << a for a in range(self.dim))
        return [np.nonzero(cid == c)[0] for c in range(2 ** self.dim) if np.any(cid == c)]

    # -- basis tables (constants of the mesh; mesh.py:104-176) -------------
    def quadrature(self, points_per_axis: int = 3) -> QuadratureRule:
        key = ("rule", points_per_axis)
        if key not in self._lazy:
            self._lazy[key] = gauss_rule(self.dim, points_per_axis)
        return self._lazy[key]

    def basis(self, rule=None) -> BasisEval:
        rule = _as_rule(rule) if rule is not None else self.quadrature()
        key = ("basis", rule.points.tobytes(), rule.weights.tobytes())
        if key not in self._lazy:
            self._lazy[key] = _tabulate_basis(self, rule)
        return self._lazy[key]

    def __repr__(self):
        return f"StructuredMesh(dim={self.dim}, extents={self.extents}, counts={self.counts})"


def _as_rule(rule) -> QuadratureRule:
    if isinstance(rule, QuadratureRule):
        return rule
    pts, wts = (rule.points, rule.weights) if hasattr(rule, "points") else rule
    return QuadratureRule(np.asarray(pts, dtype=float), np.asarray(wts, dtype=float))


def _tabulate_basis(mesh, rule: QuadratureRule) -> BasisEval:
    """Tensor Lagrange tables at the rule's points (mesh.py:151-176)."""
    n1 = mesh.order + 1
    vals1, ders1 = zip(*[_lagrange_1d(mesh.order, rule.points[:, a]) for a in range(mesh.dim)])
    nq = rule.n_points
    nloc = n1 ** mesh.dim
    values = np.ones((nq, nloc))
    gradients = np.zeros((nq, nloc, mesh.dim))
    for loc in range(nloc):
        idx = [(loc // n1 ** a) % n1 for a in range(mesh.dim)]
        v = np.ones(nq)
        for a in range(mesh.dim):
            v = v * vals1[a][:, idx[a]]
        values[:, loc] = v
        for a in range(mesh.dim):
            g = np.ones(nq)
            for b in range(mesh.dim):
                g = g * (ders1[b] if b == a else vals1[b])[:, idx[b]]
            gradients[:, loc, a] = g * (2.0 / mesh.spacing[a])
    detj = np.prod([h / 2.0 for h in mesh.spacing])
    return BasisEval(values=values, gradients=gradients, jxw=rule.weights * detj)


def eval_basis(mesh, element_id: int, rule=None) -> BasisEval:
    """Basis values/gradients/weights of one element, identical for all
    (mesh.py:259-265)."""
    if not 0 <= element_id < mesh.n_elements:
        raise IndexError(f"element id {element_id} out of range")
    return mesh.basis(rule)


def build_mesh(dim: int, extents, counts, order: int = 1) -> StructuredMesh:
    """Validation of undercool/mesh.py:185-201; returns a lazy mesh."""
    if dim not in (2, 3):
        raise ValueError("dimension must be 2 or 3")
    if order not in (1, 2):
        raise ValueError("element order must be 1 (Q1) or 2 (Q2)")
    if dim == 3 and order != 1:
        raise ValueError("3D meshes support order 1 only")
    extents = tuple(float(e) for e in extents)
    counts = tuple(int(c) for c in counts)
    if len(extents) != dim or len(counts) != dim:
        raise ValueError("extents and counts must have one entry per axis")
    if any(e <= 0.0 for e in extents):
        raise ValueError("extents must be positive")
    if any(c < 1 for c in counts):
        raise ValueError("element counts must be at least 1")
    return StructuredMesh(dim, extents, counts, order)


def gauss_rule(dim: int, points_per_axis: int = 3) -> QuadratureRule:
    """Tensor Gauss rule, x fastest (mesh.py:52-61); unpacks as (points, weights)."""
    x, w = np.polynomial.legendre.leggauss(points_per_axis)
    pts = np.stack([g.reshape(-1) for g in np.meshgrid(*([x] * dim), indexing="ij")[::-1]], axis=1)
    wts = np.ones(points_per_axis ** dim)
    for g in np.meshgrid(*([w] * dim), indexing="ij"):
        wts = wts * g.reshape(-1)
    return QuadratureRule(points=pts, weights=wts)


def mesh_descriptor(mesh, slab=None):
    """Duck-typed (dim, counts, spacing, order, slab) of this package's or the
    reference's StructuredMesh."""
    dim = int(mesh.dim)
    counts = tuple(int(c) for c in mesh.counts)
    spacing = tuple(float(h) for h in mesh.spacing)
    order = int(getattr(mesh, "order", 1))
    nslow = counts[dim - 1] + 1
    lo, hi = slab if slab is not None else (0, nslow)
    return dim, counts, spacing, order, (int(lo), int(hi))
