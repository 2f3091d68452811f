"""ctypes binding of the C ABI in include/kmx.h (libkmx.so, built in-tree).

The product path has no CPU fallback: importing this module on a machine
without the built library, or calling into it without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkmx.so")

KMX_OK = 0
KMX_EINVAL = -1
KMX_ERECON = -2
KMX_EINEXACT = -3
KMX_ECUDA = -4
KMX_ENOMEM = -5

KMX_SIGNED = 1
KMX_NO_VALIDATE = 2
KMX_NO_SPLIT = 4
KMX_NO_TUNE = 8


class ReconstructionError(ArithmeticError):
    """The overlapped digit streams are inconsistent (precondition violated).

    Mirrors kronmul.ksint.ReconstructionError (ksint.py:44-45)."""


class KmxCudaError(RuntimeError):
    """A CUDA error inside libkmx."""


_lock = threading.Lock()
_lib = None

_u32p = ctypes.POINTER(ctypes.c_uint32)
_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t
_i = ctypes.c_int
_u = ctypes.c_uint

_SIGS = {
    "kmx_ks_params": (_i, [_i, _i, _i, _i, _u, _i64p]),
    "kmx_ks_out_words": (_i, [_i, _i, _i, _u]),
    "kmx_ks_workspace_bytes": (_sz, [_i, _i, _i, _i, _i, _u]),
    "kmx_ks_mul": (_i, [_i, _i, _i, _i, _i, _vp, _vp, _i, _vp, _i, _vp, _sz, _u, _vp]),
    "kmx_ws_status": (_i, [_vp, _vp]),
    "kmx_ws_limb_products": (_i, [_vp, _i, _i, _i, _i, _i, _u, _u64p, _vp]),
    "kmx_ks_mul_host": (_i, [_i, _i, _i, _i, _i, _vp, _vp, _i, _vp, _i, _u, _u64p]),
    "kmx_pack_limbs": (_i, [_i, _i, _i]),
    "kmx_pack": (_i, [_i, _i, _i, _i, _i, _vp, _i, _vp, _i, _vp, _vp, _sz, _vp]),
    "kmx_pack_host": (_i, [_i, _i, _i, _i, _i, _vp, _i, _vp, _i, _vp]),
    "kmx_reconstruct": (_i, [_i, _i, _i, _vp, _vp, _i, _vp, _i, _vp, _sz, _vp, _vp]),
    "kmx_reconstruct_workspace_bytes": (_sz, [_i, _i, _i]),
    "kmx_reconstruct_host": (_i, [_i, _i, _i, _vp, _vp, _i, _vp, _i, _vp]),
    "kmx_bks_workspace_bytes": (_sz, [_i, _i, _i, _i]),
    "kmx_bks_workspace_bytes_cb": (_sz, [_i, _i, _i, _i, _i]),
    "kmx_bks_uni_engine": (_i, [_i, _i, _i, _i]),
    "kmx_bks_mul": (_i, [_i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _sz, _vp]),
    "kmx_bks_mul_host": (_i, [_i, _i, _i, _i, _i, _vp, _vp, _vp]),
    "kmx_bks_wide_out_words": (_i, [_i, _i, _i]),
    "kmx_bks_wide_workspace_bytes": (_sz, [_i, _i, _i, _i, _i]),
    "kmx_bks_wide_mul": (_i, [_i, _i, _i, _i, _i, _vp, _vp, _i, _vp, _i, _vp, _sz, _vp]),
    "kmx_bks_wide_mul_host": (_i, [_i, _i, _i, _i, _i, _vp, _vp, _i, _vp, _i]),
    "kmx_mod_workspace_bytes": (_sz, [_i, _i, _i, _i, ctypes.c_uint64]),
    "kmx_mod_mul": (_i, [_i, _i, _i, _i, ctypes.c_uint64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "kmx_mod_mul_host": (_i, [_i, _i, _i, _i, ctypes.c_uint64, _vp, _vp, _vp, _u64p]),
    "kmx_bks_mod_workspace_bytes": (_sz, [_i, _i, _i, _i, ctypes.c_uint64]),
    "kmx_bks_mod_mul": (_i, [_i, _i, _i, _i, ctypes.c_uint64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "kmx_bks_mod_mul_host": (_i, [_i, _i, _i, _i, ctypes.c_uint64, _vp, _vp, _vp]),
    "kmx_imad_peak": (ctypes.c_double, [_i]),
    "kmx_tc_peak": (ctypes.c_double, [_i]),
    "kmx_tc_peak_n": (ctypes.c_double, [_i, _i]),
    "kmx_mul_engine": (_i, [_i, _i, _i, _i, _u]),
    "kmx_mul_karatsuba_levels": (_i, [_i, _i, _i, _i, _i, _u]),
    "kmx_mul_plan": (_i, [_i, _i, _i, _i, _i, _u, _i64p]),
    "kmx_error_string": (ctypes.c_char_p, [_i]),
    "kmx_last_launch_count": (_i, []),
    "kmx_prof_enable": (None, [_i]),
    "kmx_prof_read": (_i, [ctypes.POINTER(ctypes.c_float), _i]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)


def lib():
    """Load libkmx.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(or `make -C paper_0712_4046_b200/csrc`); the product path has no CPU fallback")
            L = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def check(rc: int, what: str = "kmx") -> None:
    """Map a C-ABI return code to the reference's exception types."""
    if rc == KMX_OK:
        return
    msg = f"{what}: {lib().kmx_error_string(rc).decode()}"
    if rc == KMX_ERECON:
        raise ReconstructionError(msg)
    if rc in (KMX_EINVAL, KMX_EINEXACT):
        raise ValueError(msg)
    if rc == KMX_ENOMEM:
        raise MemoryError(msg)
    raise KmxCudaError(msg)


def ptr(a) -> int:
    """Address of a numpy array or torch tensor."""
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data
