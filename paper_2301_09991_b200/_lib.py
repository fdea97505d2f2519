"""ctypes binding of libconvsn_sm100.so (C ABI in include/convsn_sm100.h).

The product has no CPU fallback: every compute entry point goes through this
library on a CUDA device, and a missing library or device raises immediately.
"""

import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libconvsn_sm100.so")

F32, F64 = 0, 1
_c_int, _c_i64, _c_dbl, _vp = ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p


class Geom(ctypes.Structure):
    """Mirror of ``csn_geom``."""

    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nd", ctypes.c_int32),
                ("ng", ctypes.c_int32), ("na", ctypes.c_int32), ("ghost_w", ctypes.c_int32),
                ("ghost_e", ctypes.c_int32), ("pad_", ctypes.c_int32),
                ("dx", ctypes.c_double), ("dy", ctypes.c_double)]


_GP = ctypes.POINTER(Geom)
_DP = ctypes.POINTER(ctypes.c_double)

_SIGNATURES = {
    "csn_version": ([], _c_int),
    "csn_launch_count": ([], ctypes.c_ulonglong),
    "csn_error_string": ([_c_int], ctypes.c_char_p),
    "csn_set_tuning": ([ctypes.c_char_p, _c_int, ctypes.POINTER(ctypes.c_int)], _c_int),
    "csn_partials_size": ([_c_int, _GP, _c_int], _c_i64),
    "csn_apply_boundary": ([_c_int, _GP, _vp, _c_int, _vp, _vp, _vp], _c_int),
    "csn_upwind_residual": ([_c_int, _GP, _vp, _c_int, _vp, _vp, _c_int, _vp, _vp, _vp, _c_int,
                             _vp, _vp, _vp], _c_int),
    "csn_upwind_smooth": ([_c_int, _GP, _vp, _c_int, _c_int, _vp, _c_int, _GP, _vp, _vp, _vp, _vp,
                           _c_int, _c_dbl, _vp, _c_int, _vp], _c_int),
    "csn_upwind_smooth_sub": ([_c_int, _GP, _vp, _c_int, _c_int, _vp, _c_int, _GP, _vp, _vp, _vp,
                               _vp, _c_int, _c_dbl, _vp, _c_int, _vp], _c_int),
    "csn_restrict": ([_c_int, _GP, _GP, _vp, _c_int, _vp, _vp, _c_int, _vp, _c_int, _vp], _c_int),
    "csn_coarse_tail": ([_c_int, _c_int, _GP, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_int, _vp],
                        _c_int),
    "csn_prolong": ([_c_int, _GP, _GP, _vp, _c_int, _vp, _c_int, _vp], _c_int),
    "csn_pg_diffusivities": ([_c_int, _c_int, _GP, _DP, _DP, _vp, _c_int, _vp, _c_int, _vp, _c_int,
                              _c_int, _c_dbl, _vp, _vp, _vp, _vp, _c_int, _vp, _vp], _c_int),
    "csn_pg_workspace_size": ([_c_int, _GP, _c_int], _c_i64),
    "csn_pg_residual": ([_c_int, _c_int, _GP, _DP, _vp, _c_int, _vp, _c_int, _vp, _vp, _c_int,
                         _vp, _vp, _c_int, _vp, _vp, _vp, _vp, _c_int, _vp, _c_int, _c_dbl,
                         _vp, _vp, _vp, _c_int, _c_int, _c_dbl, _vp, _c_int, _vp], _c_int),
    "csn_scalar_flux": ([_c_int, _GP, _vp, _c_int, _vp, _vp, _vp], _c_int),
    "csn_group_source": ([_c_int, _GP, _vp, _vp, _vp, _vp, _c_dbl, _vp, _vp, _vp, _vp], _c_int),
    "csn_fission_source": ([_GP, _vp, _vp, _vp, _c_dbl, _vp, _vp], _c_int),
    "csn_production": ([_GP, _vp, _vp, _vp, _vp, _vp], _c_int),
    "csn_sum_f64": ([_vp, _c_i64, _vp, _vp], _c_int),
    "csn_scale": ([_c_int, _vp, _c_i64, _c_dbl, _c_int, _vp], _c_int),
    "csn_sub_interior": ([_c_int, _GP, _vp, _c_int, _vp, _c_int, _vp], _c_int),
    "csn_ema": ([_c_int, _GP, _vp, _c_int, _vp, _c_int, _c_dbl, _c_int, _vp], _c_int),
    "csn_dir_lincomb": ([_c_int, _c_i64, _c_int, _c_int, _vp, _vp, _c_dbl, _vp, _vp, _c_dbl, _c_dbl,
                         _vp, _vp], _c_int),
    "csn_iso_diffusivity": ([_c_int, _c_i64, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp, _DP, _vp,
                             _vp], _c_int),
    "csn_convolve": ([_c_int, _GP, _vp, _c_int, _DP, _c_int, _c_int, _vp, _vp, _vp], _c_int),
    "csn_pass1d": ([_c_int, _GP, _vp, _c_int, _DP, _c_int, _c_int, _c_int, _vp, _vp], _c_int),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None


def load(path=LIB_PATH):
    """Load the kernel library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build the sm_100a kernels first "
                           "(`make` or `python -c 'import __graft_entry__ as g; g.build()'`)")
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(code, what):
    if code == 0:
        return
    msg = load().csn_error_string(code).decode()
    if code > 0:
        raise ValueError(f"{what}: {msg} (code {code})")
    raise RuntimeError(f"{what}: CUDA error: {msg}")


def call(name, *args):
    check(getattr(load(), name)(*args), name)


def set_tuning(key, value):
    """Switch a kernel variant (csn_set_tuning); returns the previous value."""
    prev = ctypes.c_int(0)
    check(load().csn_set_tuning(key.encode(), int(value), ctypes.byref(prev)),
          f"csn_set_tuning({key!r})")
    return prev.value


def require_cuda(t, what="field"):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise RuntimeError(f"{what} must be a CUDA tensor: this package runs only on the "
                           "sm_100a kernels (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")


def dtype_code(t):
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.float64:
        return F64
    raise ValueError(f"unsupported dtype {t.dtype}; expected float32 or float64")


def ptr(t):
    return None if t is None else _vp(t.data_ptr())


def stream():
    return _vp(torch.cuda.current_stream().cuda_stream)


def host_f64(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a, a.ctypes.data_as(_DP)


def geom(nx, ny, nd, ng, na, dx, dy, ghost_w=0, ghost_e=0):
    return Geom(int(nx), int(ny), int(nd), int(ng), int(na), int(ghost_w), int(ghost_e), 0,
                float(dx), float(dy))
