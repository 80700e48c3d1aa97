"""Device residency: upload a split once, build the GPU plan once, reuse both.

``Pars3Operator`` is the object the hot loop holds: device copies of the
split's arrays (int32 indices, float64 values) plus the opaque native plan
(libpars3 ``pars3_plan``), with ``matvec`` / ``matvec_dot`` entry points
over device tensors and no host round trip.  The reference has no such
object because its arrays already live where its kernels run; here the
upload is the analogue of the numba first-call cost (bench.py:79-86 keeps
it out of the clock).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

__all__ = ["require_cuda", "Pars3Operator", "operator_for_split", "operator_for_sss"]


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the PARS3 product path runs on a CUDA device only (no CPU fallback); "
                           "no CUDA device is visible")
    _lib.load()
    return torch


def _dev(a, dtype, torch, device):
    t = torch.from_numpy(np.ascontiguousarray(a)).to(dtype)
    return t.to(device, non_blocking=False)


class Pars3Operator:
    """y = A x on one GPU for a (diag, middle, outer) decomposition of A."""

    def __init__(self, n, beta, diag, mid_ptr, mid_col, mid_val, outer_row, outer_col, outer_val,
                 p=1, block_start=None, device=None):
        torch = require_cuda()
        self.torch = torch
        self.device = torch.device(device if device is not None else "cuda")
        self.n = int(n)
        self.beta = int(beta)
        self.p = int(p)
        d = self.device
        self.diag = _dev(diag, torch.float64, torch, d)
        self.mid_ptr = _dev(mid_ptr, torch.int32, torch, d)
        self.mid_col = _dev(mid_col, torch.int32, torch, d)
        self.mid_val = _dev(mid_val, torch.float64, torch, d)
        self.outer_row = _dev(outer_row, torch.int32, torch, d)
        self.outer_col = _dev(outer_col, torch.int32, torch, d)
        self.outer_val = _dev(outer_val, torch.float64, torch, d)
        self.mid_count = int(self.mid_col.numel())
        self.outer_count = int(self.outer_col.numel())
        self.nnz = self.mid_count + self.outer_count
        view = _lib.SplitView(
            self.n, self.beta, _lib.ptr(self.diag), _lib.ptr(self.mid_ptr), _lib.ptr(self.mid_col),
            _lib.ptr(self.mid_val), self.mid_count, _lib.ptr(self.outer_row),
            _lib.ptr(self.outer_col), _lib.ptr(self.outer_val), self.outer_count)
        bs = np.ascontiguousarray(block_start if block_start is not None else [0, self.n],
                                  dtype=np.int64)
        handle = ctypes.c_void_p()
        L = _lib.load()
        with torch.cuda.device(self.device):
            _lib.check(L.pars3_plan_create(ctypes.byref(view), self.p, _lib.ptr(bs),
                                           ctypes.byref(handle), _lib.stream_ptr()),
                       "pars3_plan_create")
        self._handle = handle
        self._L = L

    # -- hot entry points (device tensors in, device tensors out) ---------
    def matvec(self, x, y=None, stream=None):
        """y = A x for a contiguous float64 CUDA tensor x of length n."""
        if y is None:
            y = self.torch.empty(self.n, dtype=self.torch.float64, device=self.device)
        _lib.check(self._L.pars3_plan_spmv(self._handle, _lib.ptr(x), _lib.ptr(y),
                                           _lib.stream_ptr(stream)), "pars3_plan_spmv")
        return y

    def matvec_dot(self, x, w, y=None, dot=None, stream=None):
        """y = A x and dot = <y, w> (device scalar tensor) in one pass."""
        t = self.torch
        if y is None:
            y = t.empty(self.n, dtype=t.float64, device=self.device)
        if dot is None:
            dot = t.empty(1, dtype=t.float64, device=self.device)
        _lib.check(self._L.pars3_plan_spmv_dot(self._handle, _lib.ptr(x), _lib.ptr(y),
                                               _lib.ptr(w), _lib.ptr(dot),
                                               _lib.stream_ptr(stream)), "pars3_plan_spmv_dot")
        return y, dot

    def kernel_count(self, with_dot: bool = False) -> int:
        c = ctypes.c_int32()
        _lib.check(self._L.pars3_plan_kernel_count(self._handle, int(with_dot), ctypes.byref(c)))
        return int(c.value)

    def plan_bytes(self) -> int:
        b = ctypes.c_int64()
        _lib.check(self._L.pars3_plan_bytes(self._handle, ctypes.byref(b)))
        return int(b.value)

    def close(self):
        if getattr(self, "_handle", None) is not None and self._handle.value:
            self._L.pars3_plan_destroy(self._handle)
            self._handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def operator_for_split(s, p=1, block_start=None, device=None) -> Pars3Operator:
    """Operator for a BandSplit, cached on the split object per (p, device)."""
    key = (int(p), str(device))
    cache = getattr(s, "_device", None)
    if cache is None:
        cache = {}
        object.__setattr__(s, "_device", cache)
    op = cache.get(key)
    if op is None:
        op = Pars3Operator(s.n, s.beta, s.diag, s.mid_ptr, s.mid_col, s.mid_val, s.outer_row,
                           s.outer_col, s.outer_val, p=p, block_start=block_start, device=device)
        cache[key] = op
    return op


def operator_for_sss(m, device=None) -> Pars3Operator:
    """Operator for a whole SssMatrix (everything in the band, beta = n)."""
    key = ("sss", str(device))
    cache = getattr(m, "_device", None)
    if cache is None:
        cache = {}
        object.__setattr__(m, "_device", cache)
    op = cache.get(key)
    if op is None:
        e = np.zeros(0, np.int32)
        op = Pars3Operator(m.n, max(1, m.n), m.diags, m.row_ptr, m.col_ind, m.off_diags, e, e,
                           np.zeros(0), device=device)
        cache[key] = op
    return op
