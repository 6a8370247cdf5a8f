"""ctypes binding of libpdst.so (include/pdst.h).

The shared library is built in-tree by ``build_ext.py`` (``__graft_entry__.build``).
There is no fallback: if it is missing, importing the operators raises.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import ConstitutiveDomainError, PdstCudaError, SingularPatchError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PDST_LIB") or os.path.join(HERE, "libpdst.so")  # PDST_LIB: experiment builds

OK, EINVAL, EDOMAIN, ESINGULAR, ECUDA, ESTATE, ENOTSUP, ENCCL = range(8)
HOST, DEVICE, HOST_ASYNC = 0, 1, 2
KIND = {"pic": 0, "exn": 1, "modn": 2}


class Mesh(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("x0", C.c_double), ("y0", C.c_double), ("x1", C.c_double),
                ("y1", C.c_double), ("dirichlet", C.POINTER(C.c_uint8))]


class Time(C.Structure):
    _fields_ = [("k", C.c_int32), ("nodes", C.POINTER(C.c_double)), ("weights", C.POINTER(C.c_double)),
                ("K_t", C.POINTER(C.c_double)), ("m_t", C.POINTER(C.c_double))]


class Disc(C.Structure):
    _fields_ = [("gamma1", C.c_double), ("gamma2", C.c_double), ("gamma_cip", C.c_double),
                ("enable_viscous", C.c_int32), ("enable_convection", C.c_int32), ("enable_pressure", C.c_int32),
                ("pressure_space", C.c_int32)]


class Params(C.Structure):
    _fields_ = [("p", C.c_double), ("delta", C.c_double), ("nu", C.c_double), ("nu_inf", C.c_double)]


_lib = None

P = C.c_void_p
D = C.c_double
I = C.c_int
I64 = C.c_int64

SIGNATURES = {
    "pdst_create": [C.POINTER(Mesh), C.POINTER(Time), C.POINTER(Disc), C.POINTER(Params), D, I, P, C.POINTER(P)],
    "pdst_destroy": [P],
    "pdst_set_stream": [P, P],
    "pdst_sizes": [P, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64), C.POINTER(I64)],
    "pdst_set_lifting": [P, P, I],
    "pdst_linearize": [P, P, I, D, I],
    "pdst_jacobian_apply": [P, P, P, I],
    "pdst_jacobian_defect": [P, P, P, P, I],
    "pdst_residual": [P, P, P, P, P, P, I],
    "pdst_mass_apply": [P, P, P, I],
    "pdst_mass_dot": [P, P, P, P, I],
    "pdst_dot": [P, P, P, I64, P, I],
    "pdst_multidot": [P, P, I64, I, P, I64, P, I],
    "pdst_multi_axpy": [P, P, P, I64, I, P, P, P, I64, I],
    "pdst_cell_maps": [P, P, P],
    "pdst_hierarchy": [P, I, C.POINTER(I)],
    "pdst_hierarchy_depth": [P, I, C.POINTER(I)],
    "pdst_sync": [P],
    "pdst_level_sizes": [P, I, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(I64)],
    "pdst_patches_build": [P, I, D, C.POINTER(I), C.POINTER(I64)],
    "pdst_patch_matrices": [P, I, P],
    "pdst_patch_info": [P, I, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(I64)],
    "pdst_vanka": [P, I, P, P, I, D, I],
    "pdst_vanka_increment": [P, I, P, P, I, I, D, I],
    "pdst_level_apply": [P, I, P, P, I],
    "pdst_restrict": [P, I, P, P, I],
    "pdst_prolong": [P, I, P, P, I],
    "pdst_vcycle": [P, P, P, I, I, D, I],
    "pdst_set_coarse_solver": [P, I, I, D, I, D],
    "pdst_set_coarse_mode": [P, I],
    "pdst_manufactured_forcing": [P, D, P, I],
    "pdst_error_norms": [P, P, D, D, I, I, P, I],
    "pdst_profile": [P, I],
    "pdst_profile_read": [P, I, C.POINTER(D), C.POINTER(I64)],
    "pdst_fp64_peak": [I, C.POINTER(D)],
    "pdst_strip": [P, I, I, I, I, I, I, I, I, I],
    "pdst_strip_comm": [P, P],
    "pdst_strip_halo": [P, P],
    "pdst_strip_step": [P, P, P, P, P, D],
    "pdst_strips_step_local": [P, I, P, P, P, P, D],
    "pdst_last_error": [],
    "pdst_version": [],
    "pdst_launch_count": [],
}


def lib():
    """Load libpdst.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = (C.c_char_p if name in ("pdst_last_error", "pdst_version") else
                          C.c_int64 if name == "pdst_launch_count" else C.c_int)
        _lib = L
    return _lib


def check(rc, what="pdst", level=None, patch=None):
    if rc == OK:
        return
    msg = lib().pdst_last_error().decode(errors="replace")
    if rc == EDOMAIN:
        raise ConstitutiveDomainError(msg)
    if rc == ESINGULAR:
        raise SingularPatchError(level if level is not None else -1, patch if patch is not None else -1)
    if rc in (EINVAL,):
        raise ValueError(f"{what}: {msg}")
    if rc == ENOTSUP:
        raise NotImplementedError(f"{what}: {msg}")
    if rc == ESTATE:
        raise RuntimeError(f"{what}: {msg}")
    raise PdstCudaError(f"{what} failed ({rc}): {msg}")


def dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def vptr(a, n=None, name="array"):
    """void* of a contiguous numpy array or a torch tensor (None -> NULL).

    With ``n``: the buffer must hold exactly n contiguous float64 values (the
    C ABI takes bare pointers, so a short or mistyped buffer would be read or
    written out of bounds); anything else raises ValueError, as the
    reference's numpy reshapes do on a size mismatch."""
    if a is None:
        return None
    if n is not None:
        if isinstance(a, np.ndarray):
            ok = a.dtype == np.float64 and a.flags.c_contiguous
            size = a.size
        else:
            import torch

            ok = a.dtype == torch.float64 and a.is_contiguous()
            size = a.numel()
        if not ok:
            raise ValueError(f"{name}: expected a contiguous float64 buffer")
        if size != n:
            raise ValueError(f"{name}: expected {n} values, got {size}")
    if isinstance(a, np.ndarray):
        return C.c_void_p(a.ctypes.data)
    return C.c_void_p(a.data_ptr())
