"""ctypes binding of libpars3.so (the C ABI declared in include/pars3.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2407_17651_b200/csrc``).  There is no fallback: if it is
missing, every entry point raises.  Device pointers come from torch CUDA
tensors (``data_ptr()``), the stream from ``torch.cuda.current_stream()``.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PARS3_LIB overrides the library path (A/B builds of the same ABI)
LIB_PATH = os.environ.get("PARS3_LIB") or os.path.join(_HERE, "_build", "libpars3.so")

PARS3_OK = 0
PARS3_ERR_ARG = -1
PARS3_ERR_CUDA = -2
PARS3_ERR_STRUCT = -3
PARS3_ERR_NOMEM = -4
PARS3_SLOW_PATH = -5

_c_i32 = ctypes.c_int32
_c_i64 = ctypes.c_int64
_vp = ctypes.c_void_p


class SplitView(ctypes.Structure):
    """Mirror of ``pars3_split_view`` (include/pars3.h): host arrays."""

    _fields_ = [
        ("n", _c_i64), ("beta", _c_i64), ("diag", _vp), ("mid_ptr", _vp), ("mid_col", _vp),
        ("mid_val", _vp), ("outer_count", _c_i64), ("outer_row", _vp), ("outer_col", _vp),
        ("outer_val", _vp),
    ]


class PlanOptions(ctypes.Structure):
    """Mirror of ``pars3_plan_options``."""

    _fields_ = [("tile_rows", _c_i32), ("local_slots", _c_i32), ("seg_max", _c_i32),
                ("gap", _c_i32), ("mode", _c_i32), ("flags", _c_i32), ("max_ctas", _c_i32)]


PLAN_SKIP_EMPTY = 1
PLAN_CUT_BLOCKS = 4
PLAN_LOCALITY = 8      # try the internal locality order on every plan (pars3.h)
PLAN_NO_LOCALITY = 16  # never use it
PLAN_DIRECT = 32       # direct mode (no shared staging) forced (pars3.h)
PLAN_NO_DIRECT = 64    # never direct mode
PLAN_HOST_BUILD = 128  # tile plan by the host builder (never csrc/tileplan_gpu.cu)
PRODUCT_ACC = 1        # pars3_plan_product: y += A x
PRODUCT_STRICT = 2
PRODUCT_XBOUND = 4    # with STRICT: x's bound is already in the plan's slot (pars3_plan_xbound_slot)     # the grid scale from this x (a pure function of x)


# name -> (restype, argtypes)
_SIGS = {
    "pars3_last_error": (ctypes.c_char_p, []),
    "pars3_abi_version": (ctypes.c_int, []),
    "pars3_sss_spmv_atomic": (ctypes.c_int, [_c_i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pars3_plan_create": (ctypes.c_int, [ctypes.POINTER(SplitView), ctypes.POINTER(PlanOptions),
                                         _c_i32, _vp, ctypes.POINTER(_vp), _vp]),
    "pars3_plan_create_resident": (ctypes.c_int, [ctypes.POINTER(SplitView), ctypes.POINTER(SplitView),
                                                  ctypes.POINTER(PlanOptions), _c_i32, _vp,
                                                  ctypes.POINTER(_vp), _vp]),
    "pars3_plan_spmv": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "pars3_plan_spmv_acc": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "pars3_plan_set_peers": (ctypes.c_int, [_vp, _c_i32, _c_i32, _c_i64, _vp, _vp, _vp]),
    "pars3_peer_finish": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp, _vp]),
    "pars3_ipc_alloc": (ctypes.c_int, [_c_i64, ctypes.POINTER(_vp)]),
    "pars3_ipc_free": (ctypes.c_int, [_vp]),
    "pars3_ipc_handle": (ctypes.c_int, [_vp, _vp]),
    "pars3_ipc_open": (ctypes.c_int, [_vp, ctypes.POINTER(_vp)]),
    "pars3_ipc_close": (ctypes.c_int, [_vp]),
    "pars3_plan_spmv_dot": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "pars3_plan_bytes": (ctypes.c_int, [_vp, ctypes.POINTER(_c_i64)]),
    "pars3_dot": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp]),
    "pars3_plan_stats": (ctypes.c_int, [_vp, _vp]),
    "pars3_tile_plan_arrays": (ctypes.c_int, [_vp, _vp, _c_i32, _c_i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pars3_locality_order": (ctypes.c_int, [ctypes.POINTER(SplitView), _vp, ctypes.POINTER(_c_i64)]),
    "pars3_full_csr_host": (ctypes.c_int, [ctypes.POINTER(SplitView), _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pars3_full_csr_device": (ctypes.c_int, [ctypes.POINTER(SplitView), _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pars3_plan_profile": (ctypes.c_int, [_vp, _vp, _vp, _c_i32, _c_i32, _vp, _vp]),
    "pars3_plan_product": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _c_i32, _vp]),
    "pars3_plan_product_axpy": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_i32, _vp]),
    "pars3_plan_xbound_slot": (ctypes.c_int, [_vp, ctypes.POINTER(_vp)]),
    "pars3_plan_status": (ctypes.c_int, [_vp, ctypes.POINTER(_c_i32), _vp]),
    "pars3_plan_kernel_count": (ctypes.c_int, [_vp, _c_i32, ctypes.POINTER(_c_i32)]),
    "pars3_plan_destroy": (ctypes.c_int, [_vp]),
    "pars3_plan_phases": (ctypes.c_int, [_vp, _vp]),
    "pars3_mrs_lanczos": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, ctypes.c_double, ctypes.c_double,
                                         _vp, _vp]),
    "pars3_mrs_state_size": (ctypes.c_int, [_vp, _vp]),
    "pars3_mrs_lanczos_dev": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pars3_mrs_rotate_dev": (ctypes.c_int, [_vp, _vp, _c_i32, _vp]),
    "pars3_mrs_update_dev": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pars3_mrs_update_dev2": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pars3_mrs_update": (ctypes.c_int, [_c_i64, _vp, ctypes.c_double, _vp, _vp, _vp,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_double, _vp, _vp]),
    "pars3_pattern_from_lower": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp]),
    "pars3_rcm_order": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, ctypes.c_int]),
    "pars3_rcm_order_device": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp]),
    "pars3_rcm_order_lower_device": (ctypes.c_int, [_c_i64, _vp, _vp, _c_i64, _vp, _vp]),
    "pars3_permute_lower_device": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                                  _vp, _vp]),
    "pars3_split_device": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _c_i64, _vp, _vp, _vp, _vp, _vp, _vp,
                                          _vp, _vp, _vp]),
    "pars3_bandwidth_device": (ctypes.c_int, [_c_i64, _vp, _vp, ctypes.POINTER(_c_i64), _vp]),
    "pars3_classify_conflicts_device": (ctypes.c_int, [_c_i64, _vp, _vp, _c_i64, _vp, ctypes.POINTER(_c_i64)]
                                        + [_vp] * 9),
    "pars3_permute_lower": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                           ctypes.c_int]),
    "pars3_split_count": (ctypes.c_int, [_c_i64, _vp, _vp, _c_i64, ctypes.POINTER(_c_i64),
                                         ctypes.POINTER(_c_i64)]),
    "pars3_split_fill": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _c_i64, _vp, _vp, _vp, _vp, _vp,
                                        _vp]),
    "pars3_mm_open": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(_vp), ctypes.POINTER(_c_i64),
                                     ctypes.POINTER(_c_i64), ctypes.POINTER(_c_i32)]),
    "pars3_mm_fill": (ctypes.c_int, [_vp, _vp, _vp, _vp, ctypes.c_int]),
    "pars3_mm_close": (ctypes.c_int, [_vp]),
    "pars3_mm_write": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, _c_i64, _c_i64, _vp, _vp,
                                      _vp, ctypes.c_int]),
    "pars3_vector_read": (ctypes.c_int, [ctypes.c_char_p, _vp, ctypes.POINTER(_c_i64), ctypes.c_int]),
    "pars3_vector_write": (ctypes.c_int, [ctypes.c_char_p, _c_i64, _vp, ctypes.c_int]),
    "pars3_permutation_read": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(_c_i64), _vp, _vp,
                                              ctypes.c_int]),
    "pars3_permutation_write": (ctypes.c_int, [ctypes.c_char_p, _c_i64, _vp, ctypes.c_int]),
    "pars3_classify_conflicts": (ctypes.c_int, [_c_i64, _vp, _vp, _c_i64, _vp,
                                                ctypes.POINTER(_c_i64), _vp, _vp, _vp, _vp, _vp,
                                                _vp, _vp, _vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load():
    """Load libpars3.so once; raise if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"libpars3.so not found at {LIB_PATH}: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, what: str = "") -> None:
    """Map a C return code to the reference's exception types."""
    if rc == PARS3_OK:
        return
    msg = load().pars3_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == PARS3_ERR_ARG:
        raise ValueError(msg)
    if rc == PARS3_ERR_STRUCT:
        from .formats import StructuralError
        raise StructuralError(msg)
    if rc == PARS3_ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def ptr(a) -> int | None:
    """Address of a numpy array or torch tensor (None for None/empty)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data if a.size else None
    return a.data_ptr() if a.numel() else None


def stream_ptr(stream=None) -> int | None:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream or None
