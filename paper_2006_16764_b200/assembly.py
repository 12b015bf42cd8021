"""Residual assembly on the B200 (drop-in for undercool/assembly.py).

``TimestepResidual`` keeps the reference's contract (assembly.py:233-268):
the old-level part is assembled once at construction (``fixed_part``), each
call returns a newly allocated F(u) = A_new(u) + fixed_part, ``evaluations``
counts calls, inputs are never mutated, and a non-finite assembled entry
raises NonFiniteResidualError naming the element and quadrature point.

Vectors may be numpy arrays (copied to the device and back, for
compatibility) or CUDA fp64 tensors (kept on the device).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .device import as_device, context_for, is_device, to_host
from .errors import NonFiniteResidualError
from .models import n_fields_of

__all__ = ["StateHistory", "QuadState", "split_fields", "join_fields", "assemble_residual",
           "TimestepResidual", "NonFiniteResidualError", "scheme_struct", "frozen_quad_state",
           "assemble_field_matrix"]


@dataclass
class StateHistory:
    new: object
    old: object
    prev: object


@dataclass
class QuadState:
    """Fields at quadrature points (assembly.py:57-75): ``val_*[f]`` is
    (n_elem, nq), ``grad_*[f]`` a dim-tuple of (n_elem, nq) components,
    ``coords`` (n_elem, nq, dim).  Device arrays when the state was a CUDA
    tensor, numpy otherwise."""

    part: str
    t_new: float
    t_old: float
    coords: object = None
    val_new: list | None = None
    grad_new: list | None = None
    val_old: list | None = None
    grad_old: list | None = None
    rate0: object = None
    val0_old: object = None


def split_fields(u, n_fields: int):
    return u.reshape(n_fields, -1)


def join_fields(*fields):
    if fields and isinstance(fields[0], torch.Tensor):
        return torch.cat([f.reshape(-1).to(torch.float64) for f in fields])
    return np.concatenate([np.asarray(f, dtype=float).reshape(-1) for f in fields])


def scheme_struct(scheme) -> L.Scheme:
    sc = L.Scheme()
    sc.theta, sc.dt, sc.step = float(scheme.theta), float(scheme.dt), int(scheme.step)
    return sc


def _default_rule(rule) -> None:
    if rule is None:
        return
    pts = rule[0] if isinstance(rule, tuple) else getattr(rule, "points", None)
    if pts is None or len(pts) not in (9, 27):
        raise NotImplementedError("the device path integrates with the 3-point Gauss rule only")


def _raise_nonfinite(ctx, sc, part, u, old, prev):
    f, w, e, q, first = (C.c_int64() for _ in range(5))
    lib = ctx.lib
    L.check(lib.uc_locate_nonfinite(
        ctx.bind(), C.byref(sc), part, L.ptr(u) if u is not None else None, L.ptr(old), L.ptr(prev),
        C.byref(f), C.byref(w), C.byref(e), C.byref(q), C.byref(first)), "uc_locate_nonfinite")
    if f.value < 0:
        raise NonFiniteResidualError("non-finite residual entry after assembly")
    name = "value" if w.value == 0 else f"flux[{w.value - 1}]"
    raise NonFiniteResidualError(
        f"non-finite {name} integrand for field {f.value} at element {e.value} "
        f"(first node {first.value}), quadrature point {q.value}")


class TimestepResidual:
    """Residual of one timestep as a function of the new state only."""

    _uc_device = True

    def __init__(self, mesh, kernel, old, prev, scheme, rule=None):
        _default_rule(rule)
        self.mesh = mesh
        self.kernel = kernel
        self.scheme = scheme
        self.rule = rule
        self.ctx = context_for(mesh, kernel)
        self._host_io = not is_device(old)
        self.old = as_device(old)
        self.prev = as_device(prev)
        self._sc = scheme_struct(scheme)
        n2 = n_fields_of(kernel) * self.ctx.n_local
        if self.old.numel() != n2 or self.prev.numel() != n2:
            raise ValueError(f"state vectors must hold {n2} values")
        fixed = torch.empty_like(self.old)
        L.check(self.ctx.lib.uc_residual(self.ctx.bind(), C.byref(self._sc), L.UC_PART_OLD, None,
                                         L.ptr(self.old), L.ptr(self.prev), None, L.ptr(fixed)),
                "uc_residual(old)")
        self._check(L.UC_PART_OLD, None)
        self._fixed = fixed
        self.evaluations = 0

    @property
    def fixed_part(self):
        return to_host(self._fixed) if self._host_io else self._fixed

    def _check(self, part, u):
        st = self.ctx.status(clear=True)
        if st.residual_nonfinite:
            _raise_nonfinite(self.ctx, self._sc, part, u, self.old, self.prev)

    def device_call(self, u: torch.Tensor, check: bool = True) -> torch.Tensor:
        """F(u) for a device vector, result on the device."""
        self.evaluations += 1
        out = torch.empty_like(u)
        L.check(self.ctx.lib.uc_residual(self.ctx.bind(), C.byref(self._sc), L.UC_PART_NEW, L.ptr(u),
                                         L.ptr(self.old), L.ptr(self.prev), L.ptr(self._fixed),
                                         L.ptr(out)), "uc_residual(new)")
        if check:
            self._check(L.UC_PART_NEW, u)
        return out

    def __call__(self, u_new):
        if is_device(u_new):
            return self.device_call(as_device(u_new))
        return to_host(self.device_call(as_device(u_new)))

    def nonfinite(self) -> bool:
        """Sticky non-finite flag of the last launches (synchronises)."""
        return bool(self.ctx.status(clear=True).residual_nonfinite)

    def jv_device(self, u, fu, v, unorm: float, eps_out=None) -> torch.Tensor:
        """(F(u + eps v) - F(u)) / eps fused on the device (newton.py:107-113).
        Non-finite F(u+eps v) sets the sticky flag checked by the caller."""
        self.evaluations += 1
        out = torch.empty_like(u)
        L.check(self.ctx.lib.uc_jv(self.ctx.bind(), C.byref(self._sc), L.ptr(u), L.ptr(fu), L.ptr(v),
                                   float(unorm), L.ptr(self.old), L.ptr(self.prev), L.ptr(self._fixed),
                                   L.ptr(out), L.ptr(eps_out) if eps_out is not None else None),
                "uc_jv")
        return out


def assemble_residual(mesh, kernel, states, scheme, rule=None, elements=None, part="full"):
    """Global residual of one theta step (assembly.py:214-230) on the device.

    part="old" is the fixed part, part="new" the live part, part="full" their
    sum.  `elements` (element ids, as the reference's mesh.conn[elements])
    restricts the sum to those elements (uc_residual_subset); a non-finite
    report then names the element by its position in `elements`, as the
    reference's _check_finite does (assembly.py:174-190)."""
    if elements is not None:
        return _assemble_subset(mesh, kernel, states, scheme, rule, elements, part)
    _default_rule(rule)
    ctx = context_for(mesh, kernel)
    host = not is_device(states.old)
    old, prev = as_device(states.old), as_device(states.prev)
    sc = scheme_struct(scheme)
    fixed = torch.empty_like(old)
    L.check(ctx.lib.uc_residual(ctx.bind(), C.byref(sc), L.UC_PART_OLD, None, L.ptr(old),
                                L.ptr(prev), None, L.ptr(fixed)), "uc_residual(old)")
    if part == "old":
        out = fixed
        st = ctx.status()
        if st.residual_nonfinite:
            _raise_nonfinite(ctx, sc, L.UC_PART_OLD, None, old, prev)
    else:
        if part not in ("new", "full"):
            raise ValueError(f"unknown part {part!r}")
        if ctx.status().residual_nonfinite and part == "full":
            _raise_nonfinite(ctx, sc, L.UC_PART_OLD, None, old, prev)
        new = as_device(states.new)
        zero = torch.zeros_like(old)
        out = torch.empty_like(old)
        L.check(ctx.lib.uc_residual(ctx.bind(), C.byref(sc), L.UC_PART_NEW, L.ptr(new), L.ptr(old),
                                    L.ptr(prev), L.ptr(zero if part == "new" else fixed),
                                    L.ptr(out)), "uc_residual(new)")
        if ctx.status().residual_nonfinite:
            _raise_nonfinite(ctx, sc, L.UC_PART_NEW, new, old, prev)
    return to_host(out) if host else out


def _assemble_subset(mesh, kernel, states, scheme, rule, elements, part):
    _default_rule(rule)
    if part not in ("old", "new", "full"):
        raise ValueError(f"unknown part {part!r}")
    ctx = context_for(mesh, kernel)
    ids = np.asarray(elements)
    n_el = int(np.prod(mesh.counts))
    if ids.dtype == bool:
        ids = np.nonzero(ids)[0]
    ids = ids.astype(np.int64).reshape(-1)
    if ids.size and (ids.min() < 0 or ids.max() >= n_el):
        raise IndexError("element id out of range")
    if np.unique(ids).size != ids.size:
        raise NotImplementedError("repeated element ids are not assembled on the device")
    mask_h = np.zeros(n_el, dtype=np.uint8)
    mask_h[ids] = 1
    mask = torch.from_numpy(mask_h).to("cuda")
    host = not is_device(states.old)
    old, prev = as_device(states.old), as_device(states.prev)
    sc = scheme_struct(scheme)
    lib = ctx.lib

    def run(pt, u, fixed, out):
        L.check(lib.uc_residual_subset(ctx.bind(), C.byref(sc), pt, L.ptr(u) if u is not None else None,
                                       L.ptr(old), L.ptr(prev), L.ptr(fixed) if fixed is not None else None,
                                       L.ptr(mask), L.ptr(out)), "uc_residual_subset")
        if ctx.status().residual_nonfinite:
            _raise_nonfinite_subset(ctx, sc, pt, u, old, prev, mask, ids, mesh)

    fixed = None
    if part in ("old", "full"):
        fixed = torch.empty_like(old)
        run(L.UC_PART_OLD, None, None, fixed)
        if part == "old":
            return to_host(fixed) if host else fixed
    new = as_device(states.new)
    out = torch.empty_like(old)
    run(L.UC_PART_NEW, new, fixed, out)
    return to_host(out) if host else out


def _raise_nonfinite_subset(ctx, sc, part, u, old, prev, mask, ids, mesh):
    """The reference scans field, then integrand part, then (position in the
    subset, qp) (assembly.py:174-190).  The device locator orders elements by
    id, so the first position holding the offending (field, part) pair is found
    by bisection over prefixes of the subset (an error path: O(log n) calls)."""

    def locate(m):
        r = [C.c_int64() for _ in range(5)]
        L.check(ctx.lib.uc_locate_nonfinite_subset(
            ctx.bind(), C.byref(sc), part, L.ptr(u) if u is not None else None, L.ptr(old),
            L.ptr(prev), L.ptr(m), *[C.byref(x) for x in r]), "uc_locate_nonfinite_subset")
        return [x.value for x in r]

    def prefix_mask(n):
        m = torch.zeros_like(mask)
        m[torch.from_numpy(ids[:n]).to(mask.device)] = 1
        return m

    f, w, e, q, first = locate(mask)
    if f < 0:
        raise NonFiniteResidualError("non-finite residual entry after assembly")
    lo, hi = 1, len(ids)
    while lo < hi:  # smallest prefix holding a non-finite (f, w) integrand
        mid = (lo + hi) // 2
        r = locate(prefix_mask(mid))
        if r[0] == f and r[1] == w:
            hi = mid
        else:
            lo = mid + 1
    f, w, e, q, first = locate(prefix_mask(lo) - prefix_mask(lo - 1))
    pos = lo - 1
    name = "value" if w == 0 else f"flux[{w - 1}]"
    raise NonFiniteResidualError(
        f"non-finite {name} integrand for field {f} at element {pos} "
        f"(first node {first}), quadrature point {q}")


def _basis_tables(mesh, rule):
    """Device copy of the rule's basis tables [V | G | jxw | points] (mesh.py:151-176)."""
    from .mesh import _as_rule

    if int(getattr(mesh, "order", 1)) != 1:
        raise NotImplementedError("only Q1 meshes run on the B200 path")
    r = _as_rule(rule) if rule is not None else None
    b = mesh.basis(r) if hasattr(mesh, "basis") else None
    if b is None or r is None:
        from .mesh import gauss_rule, _tabulate_basis

        r = r or gauss_rule(mesh.dim)
        b = _tabulate_basis(mesh, r)
    flat = np.concatenate([b.values.reshape(-1), b.gradients.reshape(-1), b.jxw.reshape(-1),
                           r.points.reshape(-1)])
    return torch.tensor(flat, dtype=torch.float64, device="cuda"), r.n_points


def frozen_quad_state(mesh, kernel, state, scheme, rule=None) -> QuadState:
    """One state interpolated to the quadrature points (assembly.py:193-211):
    values, physical gradients and point coordinates of every element, on the
    device (k_quad_state, any tensor Gauss rule).  Whole meshes only."""
    nf = n_fields_of(kernel)
    host = not is_device(state)
    u = as_device(state)
    ctx = context_for(mesh, kernel)
    tables, nq = _basis_tables(mesh, rule)
    ne, dim = mesh.n_elements, mesh.dim
    vals = torch.empty((nf, ne, nq), dtype=torch.float64, device=u.device)
    grads = torch.empty((nf, dim, ne, nq), dtype=torch.float64, device=u.device)
    coords = torch.empty((ne, nq, dim), dtype=torch.float64, device=u.device)
    L.check(ctx.lib.uc_quad_state(ctx.bind(), L.ptr(u), nf, L.ptr(tables), nq, L.ptr(coords), L.ptr(vals),
                                  L.ptr(grads)), "uc_quad_state")
    cv = (lambda t: to_host(t)) if host else (lambda t: t)
    qs = QuadState(part="new", t_new=scheme.t_new, t_old=scheme.t_old)
    qs.coords = cv(coords)
    qs.val_new = [cv(vals[f]) for f in range(nf)]
    qs.grad_new = [tuple(cv(grads[f, d]) for d in range(dim)) for f in range(nf)]
    return qs


def assemble_field_matrix(mesh, cmass, cdiff, rule=None):
    """(cmass psi_j, psi_i) + (cdiff grad psi_j, grad psi_i) (assembly.py:271-303)
    on the device, written straight into CSR (k_field_csr).  cmass/cdiff are
    scalars or (n_elements, nq) arrays; numpy/scalar coefficients give a
    scipy.sparse.csr_matrix (as the reference), CUDA tensors a torch sparse CSR
    tensor on the device.  Whole Q1 meshes only."""
    from .models import FreeGrowthKernel

    tables, nq = _basis_tables(mesh, rule)
    ne = mesh.n_elements
    on_device = any(isinstance(c, torch.Tensor) and c.is_cuda for c in (cmass, cdiff))

    def coef(c):
        t = c if isinstance(c, torch.Tensor) else torch.as_tensor(np.asarray(c, dtype=float))
        t = t.to(device="cuda", dtype=torch.float64).contiguous()
        if t.dim() == 0 or t.numel() == 1:
            return t.reshape(1), 0
        if tuple(t.shape) != (ne, nq):
            raise ValueError(f"coefficient shape {tuple(t.shape)} is not (n_elements, nq) = ({ne}, {nq})")
        return t, nq

    cm, cms = coef(cmass)
    cd, cds = coef(cdiff)
    ctx = context_for(mesh, FreeGrowthKernel())
    nnz = int(ctx.lib.uc_field_matrix_nnz(ctx.bind()))
    n = mesh.n_nodes
    indptr = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    indices = torch.empty(nnz, dtype=torch.int32, device="cuda")
    data = torch.empty(nnz, dtype=torch.float64, device="cuda")
    L.check(ctx.lib.uc_field_matrix(ctx.bind(), L.ptr(cm), cms, L.ptr(cd), cds, L.ptr(tables), nq, L.ptr(indptr),
                                    L.ptr(indices), L.ptr(data)), "uc_field_matrix")
    if on_device:
        return torch.sparse_csr_tensor(indptr, indices.to(torch.int64), data, size=(n, n))
    import scipy.sparse as sps

    return sps.csr_matrix((to_host(data), to_host(indices), to_host(indptr)), shape=(n, n))
