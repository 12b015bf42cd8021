"""Device plumbing: contexts, vector conversion and the vector kernels.

Vectors on the hot path are contiguous fp64 CUDA tensors in the reference's
block-by-field layout.  torch provides memory and streams only; every
arithmetic operation below is a kernel of libuc_b200.so.
"""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np
import torch

from . import _lib as L
from .mesh import mesh_descriptor
from .models import device_params

__all__ = ["Context", "context_for", "blas", "as_device", "is_device", "to_host",
           "norm", "dot", "axpy", "sub", "div", "scale", "require_cuda"]


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise L.UcError("no CUDA device: the B200 hot path has no CPU implementation")
    return torch.device("cuda", torch.cuda.current_device())


def is_device(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def as_device(x) -> torch.Tensor:
    dev = require_cuda()
    if isinstance(x, torch.Tensor):
        if x.is_cuda and x.dtype == torch.float64 and x.is_contiguous():
            return x
        return x.to(device=dev, dtype=torch.float64).contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return torch.from_numpy(arr).to(dev, non_blocking=False)


def to_host(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x)


class Context:
    """Owns one uc_ctx (mesh + model constants + scratch) on the current device."""

    def __init__(self, mesh_desc, params: L.ModelParams):
        lib = L.load()
        require_cuda()
        dim, counts, spacing, order, (lo, hi) = mesh_desc
        md = L.MeshDesc()
        md.dim, md.order = dim, order
        for a in range(3):
            md.counts[a] = counts[a] if a < dim else 1
            md.spacing[a] = spacing[a] if a < dim else 1.0
        md.slab_lo, md.slab_hi = lo, hi
        h = C.c_void_p()
        self._stream = torch.cuda.current_stream().cuda_stream
        L.check(lib.uc_ctx_create(C.byref(md), C.byref(params), C.c_void_p(self._stream),
                                  C.byref(h)), "uc_ctx_create")
        self.h = h
        self.lib = lib
        self.desc = mesh_desc
        self.params = params
        self.n_local = int(lib.uc_n_local(h))
        self._fin = weakref.finalize(self, lib.uc_ctx_destroy, h)

    def bind(self):
        """Follow torch's current stream (cheap when unchanged)."""
        s = torch.cuda.current_stream().cuda_stream
        if s != self._stream:
            L.check(self.lib.uc_set_stream(self.h, C.c_void_p(s)), "uc_set_stream")
            self._stream = s
        return self.h

    def status(self, clear: bool = True) -> L.Status:
        st = L.Status()
        L.check(self.lib.uc_status(self.bind(), C.byref(st), 1 if clear else 0), "uc_status")
        return st


_cache: dict = {}


def _params_key(mp: L.ModelParams):
    return tuple(getattr(mp, f) for f, _ in L.ModelParams._fields_)


def context_key(mesh, kernel, slab=None):
    return (mesh_descriptor(mesh, slab), _params_key(device_params(kernel)), torch.cuda.current_device())


def context_for(mesh, kernel, slab=None, fresh: bool = False) -> Context:
    """Shared (cached) context for a mesh/model pair, or a private one."""
    desc = mesh_descriptor(mesh, slab)
    if desc[3] != 1:
        raise NotImplementedError("only Q1 meshes run on the B200 path (order=%d)" % desc[3])
    mp = device_params(kernel)
    if fresh:
        return Context(desc, mp)
    key = (desc, _params_key(mp), torch.cuda.current_device())
    ctx = _cache.get(key)
    if ctx is None:
        ctx = Context(desc, mp)
        _cache[key] = ctx
    return ctx


_blas = {}


def blas() -> Context:
    """Context used for mesh-independent vector kernels."""
    dev = torch.cuda.current_device() if torch.cuda.is_available() else -1
    ctx = _blas.get(dev)
    if ctx is None:
        mp = L.ModelParams()
        mp.model = L.UC_MODEL_FREE_GROWTH
        ctx = Context((2, (1, 1), (1.0, 1.0), 1, (0, 2)), mp)
        _blas[dev] = ctx
    return ctx


def norm(x: torch.Tensor) -> float:
    ctx = blas()
    out = C.c_double()
    L.check(ctx.lib.uc_norm_host(ctx.bind(), x.numel(), L.ptr(x), C.byref(out)), "uc_norm")
    return out.value


def dot(a: torch.Tensor, b: torch.Tensor) -> float:
    ctx = blas()
    out = C.c_double()
    L.check(ctx.lib.uc_dot_host(ctx.bind(), a.numel(), L.ptr(a), L.ptr(b), C.byref(out)), "uc_dot")
    return out.value


def axpy(a: torch.Tensor, s: float, b: torch.Tensor, out=None) -> torch.Tensor:
    """a + s*b with numpy's two roundings."""
    ctx = blas()
    out = torch.empty_like(a) if out is None else out
    L.check(ctx.lib.uc_axpy(ctx.bind(), a.numel(), L.ptr(a), float(s), L.ptr(b), L.ptr(out)), "uc_axpy")
    return out


def sub(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    ctx = blas()
    out = torch.empty_like(a)
    L.check(ctx.lib.uc_sub(ctx.bind(), a.numel(), L.ptr(a), L.ptr(b), L.ptr(out)), "uc_sub")
    return out


def div(a: torch.Tensor, s: float) -> torch.Tensor:
    ctx = blas()
    out = torch.empty_like(a)
    L.check(ctx.lib.uc_scale_div(ctx.bind(), a.numel(), L.ptr(a), float(s), L.ptr(out)), "uc_scale_div")
    return out


def scale(s: float, a: torch.Tensor) -> torch.Tensor:
    ctx = blas()
    out = torch.empty_like(a)
    L.check(ctx.lib.uc_scale(ctx.bind(), a.numel(), float(s), L.ptr(a), L.ptr(out)), "uc_scale")
    return out


def combine(basis, k: int, y: np.ndarray) -> torch.Tensor:
    """sum_j y[j] basis[j] for j < k."""
    ctx = blas()
    out = torch.empty_like(basis[0])
    ptrs = (C.c_void_p * max(k, 1))(*[b.data_ptr() for b in basis[:k]])
    yy = np.ascontiguousarray(y[:k], dtype=np.float64)
    L.check(ctx.lib.uc_combine(ctx.bind(), out.numel(), ptrs, k,
                               yy.ctypes.data_as(C.POINTER(C.c_double)), L.ptr(out)), "uc_combine")
    return out


def _vec_check(x: torch.Tensor):
    ctx = blas()
    bad, nz = C.c_int32(), C.c_int32()
    L.check(ctx.lib.uc_vec_check(ctx.bind(), x.numel(), L.ptr(x), C.byref(bad), C.byref(nz)), "uc_vec_check")
    return bool(bad.value), bool(nz.value)


def all_finite(x: torch.Tensor) -> bool:
    """np.all(np.isfinite(x)) (newton.py:144,175) through k_vec_check."""
    return not _vec_check(x)[0]


def any_nonzero(x: torch.Tensor) -> bool:
    """np.any(x) (newton.py:176) through k_vec_check."""
    return _vec_check(x)[1]


def arnoldi(apply_op, basis: list, k: int, scale: float, cgs2: bool = False):
    """One Arnoldi step (krylov.py:48-70) on device vectors: (h numpy, new
    vector or None, breakdown)."""
    w = as_device(apply_op(basis[k]))
    if any(w.data_ptr() == b.data_ptr() for b in basis[: k + 1]):
        w = w.clone()  # MGS updates w in place; never alias a basis vector
    slot = torch.empty_like(w)
    h = np.zeros(k + 2)
    broke = C.c_int()
    ctx = blas()
    fn = ctx.lib.uc_arnoldi_cgs2 if cgs2 else ctx.lib.uc_arnoldi
    L.check(fn(ctx.bind(), w.numel(), L.ptrs(basis[: k + 1] + [slot]), k, L.ptr(w),
               float(scale), h.ctypes.data_as(C.POINTER(C.c_double)), C.byref(broke)),
            "uc_arnoldi")
    if broke.value:
        return h, None, True
    return h, slot, False


class DeviceSpace:
    """Vector space of single contiguous fp64 CUDA tensors (one GPU)."""

    def vec(self, x):
        return as_device(x)

    norm = staticmethod(norm)
    dot = staticmethod(dot)
    sub = staticmethod(sub)
    div = staticmethod(div)
    scale = staticmethod(scale)
    combine = staticmethod(combine)
    all_finite = staticmethod(all_finite)
    any_nonzero = staticmethod(any_nonzero)
    arnoldi = staticmethod(arnoldi)

    @staticmethod
    def axpy(a, s, b):
        return axpy(a, s, b)

    @staticmethod
    def zeros_like(x):
        return torch.zeros_like(x)

    @staticmethod
    def clone(x):
        return x.clone()

    @staticmethod
    def is_native(x) -> bool:
        return is_device(x)


DEVICE = DeviceSpace()


def space_of(x):
    """The vector space a vector belongs to (slab vectors carry theirs)."""
    sp = getattr(x, "space", None)
    return sp if sp is not None else DEVICE
