"""ctypes binding of the C ABI in include/uc_b200.h.

This is the only place the shared library is loaded.  There is no fallback:
if the library or a CUDA device is missing, every device entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libuc_b200.so")

UC_OK, UC_ERR_NONFINITE, UC_ERR_ARG, UC_ERR_CUDA, UC_ERR_UNSUPPORTED = 0, 1, 2, 3, 4
UC_MODEL_FREE_GROWTH, UC_MODEL_ALLOY, UC_MODEL_MASS_DIFF = 1, 2, 3
UC_PART_NEW, UC_PART_OLD = 0, 1
UC_PC_IDENTITY, UC_PC_JACOBI, UC_PC_SGS, UC_PC_VCYCLE = 0, 1, 2, 3


class MeshDesc(C.Structure):
    _fields_ = [("dim", C.c_int32), ("order", C.c_int32), ("counts", C.c_int64 * 3),
                ("spacing", C.c_double * 3), ("slab_lo", C.c_int64), ("slab_hi", C.c_int64)]


class ModelParams(C.Structure):
    _fields_ = [("model", C.c_int32), ("normalized", C.c_int32), ("eps", C.c_double),
                ("reg", C.c_double), ("aniso_reg_grad", C.c_double), ("bg", C.c_double),
                ("beta", C.c_double), ("alpha", C.c_double), ("latent", C.c_double),
                ("hcell", C.c_double), ("tmelt", C.c_double), ("at_reg2", C.c_double),
                ("kpart", C.c_double), ("coupling", C.c_double), ("dcoef", C.c_double),
                ("g4_coef", C.c_double), ("pull_velocity", C.c_double),
                ("mass_coef", C.c_double)]


class Scheme(C.Structure):
    _fields_ = [("theta", C.c_double), ("dt", C.c_double), ("step", C.c_int64)]


class PrecondCfg(C.Structure):
    _fields_ = [("kind", C.c_int32), ("sweeps", C.c_int32), ("cycles", C.c_int32),
                ("levels", C.c_int32), ("coarse_sweeps", C.c_int32), ("ordering", C.c_int32)]


class HostOp(C.Structure):
    _fields_ = [("kind", C.c_int32), ("peer", C.c_int32), ("count", C.c_int64), ("buf", C.POINTER(C.c_double))]


SENDRECV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.POINTER(HostOp))
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int)


class HostTransport(C.Structure):
    _fields_ = [("user", C.c_void_p), ("sendrecv", SENDRECV_FN), ("allreduce_sum", ALLREDUCE_FN)]


class DiagArgs(C.Structure):
    _fields_ = [("what", C.c_int32), ("pad", C.c_int32), ("elem_node_weight", C.c_double * 8),
                ("composition", C.c_double), ("tip_level", C.c_double), ("extent_x", C.c_double)]


DIAG_BALANCE, DIAG_SOLUTE, DIAG_TIP, DIAG_N = 1, 2, 4, 8


class Status(C.Structure):
    _fields_ = [("residual_nonfinite", C.c_int32), ("precond_nonfinite", C.c_int32),
                ("precond_bad_diag", C.c_int32), ("pad", C.c_int32)]


_P = C.c_void_p
_D = C.c_double
_I64 = C.c_int64
_I = C.c_int

# name -> (restype, argtypes); every symbol declared in include/uc_b200.h
SIGNATURES = {
    "uc_abi_version": (C.c_int, []),
    "uc_last_error": (C.c_char_p, []),
    "uc_ctx_create": (_I, [C.POINTER(MeshDesc), C.POINTER(ModelParams), _P, C.POINTER(_P)]),
    "uc_ctx_destroy": (_I, [_P]),
    "uc_set_stream": (_I, [_P, _P]),
    "uc_n_local": (_I64, [_P]),
    "uc_ghost_ptr": (_P, [_P, _I, _I]),
    "uc_residual": (_I, [_P, C.POINTER(Scheme), _I, _P, _P, _P, _P, _P]),
    "uc_locate_nonfinite": (_I, [_P, C.POINTER(Scheme), _I, _P, _P, _P] + [C.POINTER(_I64)] * 5),
    "uc_residual_subset": (_I, [_P, C.POINTER(Scheme), _I, _P, _P, _P, _P, _P, _P]),
    "uc_locate_nonfinite_subset": (_I, [_P, C.POINTER(Scheme), _I, _P, _P, _P, _P] + [C.POINTER(_I64)] * 5),
    "uc_jv": (_I, [_P, C.POINTER(Scheme), _P, _P, _P, _D, _P, _P, _P, _P, _P]),
    "uc_dot": (_I, [_P, _I64, _P, _P, _P]),
    "uc_norm": (_I, [_P, _I64, _P, _P]),
    "uc_dot_host": (_I, [_P, _I64, _P, _P, C.POINTER(_D)]),
    "uc_norm_host": (_I, [_P, _I64, _P, C.POINTER(_D)]),
    "uc_arnoldi": (_I, [_P, _I64, C.POINTER(_P), _I, _P, _D, C.POINTER(_D), C.POINTER(_I)]),
    "uc_combine": (_I, [_P, _I64, C.POINTER(_P), _I, C.POINTER(_D), _P]),
    "uc_arnoldi_cgs2": (_I, [_P, _I64, C.POINTER(_P), _I, _P, _D, C.POINTER(_D), C.POINTER(_I)]),
    "uc_arnoldi_cgs2_group": (_I, [C.POINTER(_P), _I, C.POINTER(_P), _I, C.POINTER(_P), _D,
                                   C.POINTER(_D), C.POINTER(_I)]),
    "uc_axpy": (_I, [_P, _I64, _P, _D, _P, _P]),
    "uc_sub": (_I, [_P, _I64, _P, _P, _P]),
    "uc_scale_div": (_I, [_P, _I64, _P, _D, _P]),
    "uc_scale": (_I, [_P, _I64, _D, _P, _P]),
    "uc_quad_state": (_I, [_P, _P, _I, _P, _I, _P, _P, _P]),
    "uc_field_matrix_nnz": (_I64, [_P]),
    "uc_field_matrix": (_I, [_P, _P, _I64, _P, _I64, _P, _I, _P, _P, _P]),
    "uc_vec_check": (_I, [_P, _I64, _P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "uc_precond_build": (_I, [_P, C.POINTER(Scheme), _P, C.POINTER(PrecondCfg)]),
    "uc_precond_apply": (_I, [_P, _P, _P]),
    "uc_precond_stencil": (_I, [_P, _I, _I, _P]),
    "uc_precond_levels": (_I, [_P, C.POINTER(_I64)]),
    "uc_precond_uniform": (_I, [_P, _I, _I, C.POINTER(_D)]),
    "uc_status": (_I, [_P, C.POINTER(Status), _I]),
    "uc_fp64_probe": (_I, [_P, _I, C.POINTER(_D), C.POINTER(_D)]),
    "uc_initial_state": (_I, [_P, _I, C.POINTER(_D), C.POINTER(_D), _P]),
    "uc_step_diagnostics": (_I, [_P, _P, _P, _P, C.POINTER(DiagArgs), _P]),
    "uc_map_u_to_c": (_I, [_P, _P, _D, _P]),
    "uc_write_snapshot": (_I, [C.c_char_p, _I, _I, C.POINTER(_I64), C.POINTER(_D), _I,
                               C.POINTER(C.c_char_p), C.POINTER(_P), C.c_char_p, _I]),
    "uc_write_mesh_vtk": (_I, [C.c_char_p, _I, C.POINTER(_I64), C.POINTER(_D), _I]),
    "uc_repr_double": (_I, [_D, C.c_char_p]),
    "uc_nccl_unique_id": (_I, [C.c_char_p, _P]),
    "uc_comm_init_nccl": (_I, [C.c_char_p, _P, _I, _I]),
    "uc_comm_finalize": (_I, []),
    "uc_comm_init_host": (_I, [C.POINTER(HostTransport), _I, _I]),
    "uc_ctx_set_neighbors": (_I, [_P, _I, _I]),
    "uc_ctx_link_local": (_I, [_P, _P]),
    "uc_residual_group": (_I, [C.POINTER(_P), _I, C.POINTER(Scheme), _I] + [C.POINTER(_P)] * 5),
    "uc_jv_group": (_I, [C.POINTER(_P), _I, C.POINTER(Scheme), C.POINTER(_P), C.POINTER(_P),
                         C.POINTER(_P), _D, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P),
                         C.POINTER(_P), _P]),
    "uc_dot_group": (_I, [C.POINTER(_P), _I, C.POINTER(_P), C.POINTER(_P), _I, C.POINTER(_D)]),
    "uc_arnoldi_group": (_I, [C.POINTER(_P), _I, C.POINTER(_P), _I, C.POINTER(_P), _D,
                              C.POINTER(_D), C.POINTER(_I)]),
    "uc_precond_build_group": (_I, [C.POINTER(_P), _I, C.POINTER(Scheme), C.POINTER(_P),
                                    C.POINTER(PrecondCfg)]),
    "uc_precond_apply_group": (_I, [C.POINTER(_P), _I, C.POINTER(_P), C.POINTER(_P)]),
    "uc_step_diagnostics_group": (_I, [C.POINTER(_P), _I] + [C.POINTER(_P)] * 3
                                  + [C.POINTER(DiagArgs), C.POINTER(_P)]),
}

_lock = threading.Lock()
_lib = None


class UcError(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load the library (no CUDA needed for loading itself)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise UcError(
                    f"B200 hot-path library not built: {path} is missing "
                    "(run `python -m paper_2006_16764_b200.build`)")
            lib = C.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc != UC_OK:
        msg = load().uc_last_error().decode(errors="replace")
        raise UcError(f"{what}: {msg} (code {rc})")


def ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def ptrs(ts) -> "C.Array":
    """ctypes void* array of tensor data pointers (None allowed)."""
    return (C.c_void_p * len(ts))(*[None if t is None else t.data_ptr() for t in ts])
