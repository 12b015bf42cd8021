"""Slab decomposition of the hot path.

The mesh is cut into slabs of node planes along the slowest axis (y in 2D,
z in 3D).  A slab owns planes [lo, hi); the element layer straddling a slab
boundary is evaluated by both neighbours from one ghost plane of each input,
so residual and Jv need one plane exchange per input and no reverse exchange
(csrc/comm.cu).  Dot products are global sums (one scalar allreduce each).
The preconditioner smoother exchanges one plane per parity half of every
half-sweep (csrc/precond.cu).

Two transports, same kernels:
  * ``SlabGroup.local(...)``   k slabs in ONE process on one device; planes
    are copied on the stream.  This is how the multi-rank data path is tested
    on a single GPU (tests/test_gpu_slabs.py).
  * ``SlabGroup.from_torch_dist(...)`` one slab per process/GPU; NCCL
    send/recv and allreduce issued by the library on the CUDA stream.

Vectors of a group are ``SlabVec`` (one block-ordered tensor per local slab);
newton_solve / gmres_solve accept them directly (their ``space`` does the
global reductions).  Partitioning and the torch.distributed plane exchange
used for host-side checks run on CPU with the gloo backend
(tests/test_parallel_gloo.py).
"""

from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np
import torch

from . import _lib as L
from . import device as D
from .assembly import scheme_struct
from .errors import NonFiniteResidualError
from .mesh import mesh_descriptor
from .models import device_params
from .precond import _KINDS, PrecondConfig

__all__ = ["partition_planes", "SlabVec", "SlabSpace", "SlabGroup", "SlabResidual",
           "SlabPrecond", "exchange_planes_torch", "slab_bounds"]


def partition_planes(nslow: int, world: int, align: int = 1):
    """Split node planes [0, nslow) into `world` contiguous slabs whose inner
    boundaries are multiples of `align` (coarse grids of a V-cycle with L levels
    need align = 2^(L-1)).  Returns [(lo, hi)] with hi of the last = nslow."""
    if world < 1:
        raise ValueError("world must be >= 1")
    units = (nslow - 1) // align  # boundary positions available
    if units < world and world > 1:
        raise ValueError(f"{nslow} planes cannot be split into {world} slabs aligned to {align}")
    bounds = [0]
    for r in range(1, world):
        bounds.append(((units * r) // world) * align)
    bounds.append(nslow)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def slab_bounds(mesh, world: int, levels: int = 4):
    """Slab bounds for `mesh` aligned for a `levels`-level V-cycle."""
    nslow = mesh.counts[mesh.dim - 1] + 1
    return partition_planes(nslow, world, 2 ** max(levels - 1, 0))


class SlabVec:
    """One block-ordered device tensor per local slab."""

    __slots__ = ("parts", "space")

    def __init__(self, parts, space):
        self.parts = list(parts)
        self.space = space

    def __len__(self):
        return len(self.parts)


class SlabSpace:
    """Vector space of a slab group: local kernels per slab, global reductions
    through uc_dot_group / uc_arnoldi_group."""

    def __init__(self, group):
        self.group = group

    def _ctxs(self):
        return self.group.handles

    def wrap(self, parts):
        return SlabVec(parts, self)

    def vec(self, x):
        if isinstance(x, SlabVec):
            return x
        return self.group.split(x)

    def is_native(self, x):
        return isinstance(x, SlabVec)

    def _dot(self, a, b, do_sqrt):
        out = C.c_double()
        n = len(a.parts)
        L.check(L.load().uc_dot_group(self._ctxs(), n, L.ptrs(a.parts),
                                      L.ptrs(b.parts) if b is not None else None, 1 if do_sqrt else 0,
                                      C.byref(out)), "uc_dot_group")
        return out.value

    def norm(self, x):
        return self._dot(x, None, True)

    def dot(self, a, b):
        return self._dot(a, b, False)

    def sub(self, a, b):
        return self.wrap([D.sub(p, q) for p, q in zip(a.parts, b.parts)])

    def div(self, a, s):
        return self.wrap([D.div(p, s) for p in a.parts])

    def scale(self, s, a):
        return self.wrap([D.scale(s, p) for p in a.parts])

    def axpy(self, a, s, b):
        return self.wrap([D.axpy(p, s, q) for p, q in zip(a.parts, b.parts)])

    def combine(self, basis, k, y):
        return self.wrap([D.combine([b.parts[i] for b in basis], k, y) for i in range(len(basis[0].parts))])

    def zeros_like(self, x):
        return self.wrap([torch.zeros_like(p) for p in x.parts])

    def clone(self, x):
        return self.wrap([p.clone() for p in x.parts])

    def all_finite(self, x):
        return bool(np.isfinite(self.norm(x)))

    def any_nonzero(self, x):
        return self.norm(x) != 0.0

    def arnoldi(self, apply_op, basis, k, scale, cgs2: bool = False):
        w = apply_op(basis[k])
        parts = []
        for i, p in enumerate(w.parts):
            if any(p.data_ptr() == b.parts[i].data_ptr() for b in basis[: k + 1]):
                p = p.clone()
            parts.append(p)
        slot = self.wrap([torch.empty_like(p) for p in parts])
        ns = len(parts)
        mat = []
        for i in range(ns):
            mat += [b.parts[i] for b in basis[: k + 1]] + [slot.parts[i]]
        h = np.zeros(k + 2)
        broke = C.c_int()
        fn = L.load().uc_arnoldi_cgs2_group if cgs2 else L.load().uc_arnoldi_group
        L.check(fn(self._ctxs(), ns, L.ptrs(mat), k, L.ptrs(parts), float(scale),
                   h.ctypes.data_as(C.POINTER(C.c_double)), C.byref(broke)), "uc_arnoldi_group")
        if broke.value:
            return h, None, True
        return h, slot, False


class SlabGroup:
    """The slabs of one mesh/model driven by this process."""

    def __init__(self, mesh, kernel, slabs, dist_rank=None, dist_world=None, pg=None):
        self._args = (mesh, kernel, list(slabs), dist_rank, dist_world, pg)
        self._pg = pg  # torch.distributed process group of the ranks (None = WORLD)
        self.mesh = mesh
        self.kernel = kernel
        self.slabs = list(slabs)
        self.dim = mesh.dim
        mp = device_params(kernel)
        self.ctxs = [D.Context(mesh_descriptor(mesh, s), mp) for s in self.slabs]
        lib = L.load()
        for lo_c, hi_c in zip(self.ctxs, self.ctxs[1:]):
            L.check(lib.uc_ctx_link_local(lo_c.h, hi_c.h), "uc_ctx_link_local")
        if dist_rank is not None:
            ctx = self.ctxs[0]
            lo_rank = dist_rank - 1 if self.slabs[0][0] > 0 else -1
            hi_rank = dist_rank + 1 if dist_rank + 1 < dist_world else -1
            L.check(lib.uc_ctx_set_neighbors(ctx.h, lo_rank, hi_rank), "uc_ctx_set_neighbors")
        self.space = SlabSpace(self)
        self.plane = int(np.prod(mesh.node_shape[: mesh.dim - 1]))
        self._dist = dist_rank is not None and (dist_world or 1) > 1

    @classmethod
    def local(cls, mesh, kernel, world: int, levels: int = 4):
        """`world` slabs emulated in this process on the current device."""
        return cls(mesh, kernel, slab_bounds(mesh, world, levels))

    @classmethod
    def from_torch_dist(cls, mesh, kernel, levels: int = 4, group=None, transport: str = "nccl"):
        """One slab per torch.distributed rank; initialises the library's NCCL
        communicator from a unique id broadcast over torch.distributed.
        transport="host": the same remote code path with planes and partial
        sums staged through host memory and moved by torch.distributed (gloo);
        for several ranks sharing one GPU, where NCCL cannot run (tests)."""
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        path = nccl_library_path()
        lib = L.load()
        if world > 1 and transport == "host":
            HostTransportCallbacks.install(group, rank, world)
        elif world > 1:
            idb = (C.c_char * 128)()
            if rank == 0:
                L.check(lib.uc_nccl_unique_id(path.encode(), idb), "uc_nccl_unique_id")
            obj = [bytes(idb)]
            src = 0 if group is None else dist.get_global_rank(group, 0)
            dist.broadcast_object_list(obj, src=src, group=group)
            idb = (C.c_char * 128).from_buffer_copy(obj[0])
            L.check(lib.uc_comm_init_nccl(path.encode(), idb, rank, world), "uc_comm_init_nccl")
        bounds = slab_bounds(mesh, world, levels)
        return cls(mesh, kernel, [bounds[rank]], dist_rank=rank if world > 1 else None, dist_world=world,
                   pg=group)

    def clone(self) -> "SlabGroup":
        """Fresh contexts on the same slabs (a preconditioner owns its own)."""
        return SlabGroup(*self._args)

    @property
    def handles(self):
        return (C.c_void_p * len(self.ctxs))(*[c.bind().value for c in self.ctxs])

    def split(self, x) -> SlabVec:
        """Global block-ordered vector -> this process's slab parts."""
        g = D.as_device(x)
        n = g.numel() // 2
        parts = []
        for lo, hi in self.slabs:
            a, b = lo * self.plane, hi * self.plane
            parts.append(torch.cat([g[a:b], g[n + a:n + b]]).contiguous())
        return SlabVec(parts, self.space)

    def join(self, v: SlabVec) -> torch.Tensor:
        """Slab parts (all slabs local) -> global block-ordered vector."""
        halves = [[], []]
        for p in v.parts:
            m = p.numel() // 2
            halves[0].append(p[:m])
            halves[1].append(p[m:])
        return torch.cat(halves[0] + halves[1])

    def flag(self, field: str) -> bool:
        """Sticky status flag over all slabs (and all ranks)."""
        bad = any(getattr(c.status(clear=True), field) for c in self.ctxs)
        if self._dist:
            import torch.distributed as dist

            dev = "cpu" if dist.get_backend(self._pg) == "gloo" else "cuda"
            t = torch.tensor([1.0 if bad else 0.0], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self._pg)
            bad = bool(t.item() > 0)
        return bad


class HostTransportCallbacks:
    """uc_comm_init_host callbacks over torch.distributed (CPU tensors aliasing
    the library's pinned staging buffers; every call completes before it
    returns)."""

    _live = None  # keeps the ctypes callbacks alive while the library holds them

    def __init__(self, group):
        self.group = group
        self._sr = L.SENDRECV_FN(self._sendrecv)
        self._ar = L.ALLREDUCE_FN(self._allreduce)
        self.struct = L.HostTransport(None, self._sr, self._ar)

    @classmethod
    def install(cls, group, rank, world):
        cb = cls(group)
        L.check(L.load().uc_comm_init_host(C.byref(cb.struct), rank, world), "uc_comm_init_host")
        cls._live = cb
        return cb

    def _peer(self, r):
        import torch.distributed as dist

        return r if self.group is None else dist.get_global_rank(self.group, r)

    def _sendrecv(self, user, nops, ops):
        import torch.distributed as dist

        try:
            reqs = []
            for i in range(nops):
                op = ops[i]
                t = torch.from_numpy(np.ctypeslib.as_array(op.buf, shape=(op.count,)))
                fn = dist.isend if op.kind == 0 else dist.irecv
                reqs.append(fn(t, self._peer(op.peer), group=self.group))
            for r in reqs:
                r.wait()
            return 0
        except Exception as exc:  # reported through the library's error path
            print(f"host transport sendrecv failed: {exc!r}", file=sys.stderr)
            return 1

    def _allreduce(self, user, vals, n):
        import torch.distributed as dist

        try:
            t = torch.from_numpy(np.ctypeslib.as_array(vals, shape=(n,)))
            dist.all_reduce(t, group=self.group)
            return 0
        except Exception as exc:
            print(f"host transport allreduce failed: {exc!r}", file=sys.stderr)
            return 1


def nccl_library_path() -> str:
    try:
        import nvidia.nccl

        base = os.path.dirname(nvidia.nccl.__file__ or list(nvidia.nccl.__path__)[0])
        cand = os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(cand):
            return cand
    except Exception:
        pass
    return "libnccl.so.2"


class SlabResidual:
    """TimestepResidual over a slab group (assembly.py:233-268 contract)."""

    _uc_device = True

    def __init__(self, group: SlabGroup, old, prev, scheme):
        self.group = group
        self.scheme = scheme
        sp = group.space
        self.old = sp.vec(old)
        self.prev = sp.vec(prev)
        self._sc = scheme_struct(scheme)
        self._fixed = sp.wrap([torch.empty_like(p) for p in self.old.parts])
        n = len(group.ctxs)
        L.check(L.load().uc_residual_group(group.handles, n, C.byref(self._sc), L.UC_PART_OLD,
                                           L.ptrs([None] * n), L.ptrs(self.old.parts),
                                           L.ptrs(self.prev.parts), L.ptrs([None] * n),
                                           L.ptrs(self._fixed.parts)), "uc_residual_group(old)")
        if group.flag("residual_nonfinite"):
            raise NonFiniteResidualError("non-finite old-level residual")
        self.evaluations = 0

    @property
    def fixed_part(self):
        return self._fixed

    def device_call(self, u, check: bool = True):
        self.evaluations += 1
        out = self.group.space.wrap([torch.empty_like(p) for p in u.parts])
        n = len(u.parts)
        L.check(L.load().uc_residual_group(self.group.handles, n, C.byref(self._sc), L.UC_PART_NEW,
                                           L.ptrs(u.parts), L.ptrs(self.old.parts),
                                           L.ptrs(self.prev.parts), L.ptrs(self._fixed.parts),
                                           L.ptrs(out.parts)), "uc_residual_group(new)")
        if check and self.group.flag("residual_nonfinite"):
            raise NonFiniteResidualError("non-finite residual entry after assembly")
        return out

    def __call__(self, u):
        return self.device_call(self.group.space.vec(u))

    def jv_device(self, u, fu, v, unorm, eps_out=None):
        self.evaluations += 1
        out = self.group.space.wrap([torch.empty_like(p) for p in v.parts])
        n = len(v.parts)
        L.check(L.load().uc_jv_group(self.group.handles, n, C.byref(self._sc), L.ptrs(u.parts),
                                     L.ptrs(fu.parts), L.ptrs(v.parts), float(unorm),
                                     L.ptrs(self.old.parts), L.ptrs(self.prev.parts),
                                     L.ptrs(self._fixed.parts), L.ptrs(out.parts),
                                     L.ptr(eps_out) if eps_out is not None else None), "uc_jv_group")
        return out

    def nonfinite(self) -> bool:
        return self.group.flag("residual_nonfinite")


class SlabPrecond:
    """BlockPrecond over a slab group (precond.py:225-299 contract)."""

    _uc_device = True

    def __init__(self, group: SlabGroup, state, scheme, config: PrecondConfig | None = None):
        cfg = config or PrecondConfig(ordering="multicolor")
        if cfg.kind == "direct":
            raise NotImplementedError("kind='direct' has no device implementation")
        self.group = group.clone()  # the hierarchy lives in its own contexts
        self.space = group.space
        self.cfg = cfg
        st = group.space.vec(state)
        pc = L.PrecondCfg()
        pc.kind = _KINDS[cfg.kind]
        pc.sweeps, pc.cycles, pc.levels, pc.coarse_sweeps = cfg.sweeps, cfg.cycles, cfg.levels, cfg.coarse_sweeps
        pc.ordering = 1 if cfg.ordering == "lexicographic" else 0
        sc = scheme_struct(scheme)
        rc = L.load().uc_precond_build_group(self.group.handles, len(self.group.ctxs), C.byref(sc),
                                             L.ptrs(st.parts), C.byref(pc))
        if rc == L.UC_ERR_ARG:
            raise ValueError(L.load().uc_last_error().decode())
        L.check(rc, "uc_precond_build_group")
        self.applications = 0

    def _uc_deferred(self, v):
        self.applications += 1
        out = self.space.wrap([torch.empty_like(p) for p in v.parts])
        L.check(L.load().uc_precond_apply_group(self.group.handles, len(v.parts), L.ptrs(v.parts),
                                                L.ptrs(out.parts)), "uc_precond_apply_group")
        return out

    def _uc_check(self):
        if self.group.flag("precond_nonfinite"):
            raise FloatingPointError("preconditioner produced non-finite values")

    def apply(self, v):
        out = self._uc_deferred(self.space.vec(v))
        self._uc_check()
        return out

    __call__ = apply


def exchange_planes_torch(local: torch.Tensor, plane: int, group=None):
    """Host-side reference of the slab halo: returns (ghost_lo, ghost_hi) plane
    pairs [2 fields][plane] for a block-ordered local vector, exchanged with
    torch.distributed send/recv (gloo on CPU, NCCL on GPU).  Used to check the
    partition/halo logic without a GPU."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n = local.numel() // 2
    f = local.view(2, n)
    top = f[:, n - plane:].contiguous()
    bottom = f[:, :plane].contiguous()
    glo = torch.zeros_like(top) if rank > 0 else None
    ghi = torch.zeros_like(top) if rank + 1 < world else None
    ops = []
    if rank + 1 < world:
        ops += [dist.P2POp(dist.isend, top, rank + 1, group), dist.P2POp(dist.irecv, ghi, rank + 1, group)]
    if rank > 0:
        ops += [dist.P2POp(dist.isend, bottom, rank - 1, group), dist.P2POp(dist.irecv, glo, rank - 1, group)]
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return glo, ghi
