"""Device residency: build the GPU plan once per split, reuse it for every product.

``Pars3Operator`` is the object the hot loop holds: the opaque native plan
(libpars3 ``pars3_plan``: the split re-tiled into row tiles with shared-
memory column windows, uploaded once) with ``matvec`` / ``matvec_dot``
entry points over device tensors and no host round trip.  The reference
has no such object because its arrays already live where its kernels run;
building it is the analogue of the numba first-call cost that
bench.py:79-86 of the reference keeps out of the clock.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

__all__ = ["require_cuda", "Pars3Operator", "SssDevice", "operator_for_split", "operator_for_sss",
           "sss_device", "dot"]


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the PARS3 product path runs on a CUDA device only (no CPU fallback); "
                           "no CUDA device is visible")
    _lib.load()
    return torch


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class Pars3Operator:
    """y = A x on one GPU for a (diag, middle, outer) decomposition of A."""

    def __init__(self, n, beta, diag, mid_ptr, mid_col, mid_val, outer_row, outer_col, outer_val,
                 p=1, block_start=None, device=None, options=None, resident=None):
        """``resident``: optional dict of CUDA tensors holding the same split on
        this device (mid_ptr int64, mid_col int32, mid_val float64, outer_row /
        outer_col int32, outer_val float64; ``prepare_gpu(..., keep_device=True)``):
        the tile plan is then built from them without another upload."""
        torch = require_cuda()
        self.torch = torch
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.n = int(n)
        self.beta = int(beta)
        self.p = int(p)
        host = dict(diag=_c(diag, np.float64), mid_ptr=_c(mid_ptr, np.int64),
                    mid_col=_c(mid_col, np.int32), mid_val=_c(mid_val, np.float64),
                    outer_row=_c(outer_row, np.int32), outer_col=_c(outer_col, np.int32),
                    outer_val=_c(outer_val, np.float64))
        self.nnz = int(host["mid_col"].size + host["outer_col"].size)
        view = _lib.SplitView(self.n, self.beta, _lib.ptr(host["diag"]), _lib.ptr(host["mid_ptr"]),
                              _lib.ptr(host["mid_col"]), _lib.ptr(host["mid_val"]),
                              int(host["outer_col"].size), _lib.ptr(host["outer_row"]),
                              _lib.ptr(host["outer_col"]), _lib.ptr(host["outer_val"]))
        # (tile_rows, local_slots, seg_max, gap, mode, flags, max_ctas); 0 / -1 = default
        opts = _lib.PlanOptions(*(tuple(options or ()) + (0, 0, 0, -1, 0, 0, 0)[len(options or ()):]))
        bs = _c(block_start if block_start is not None else [0, self.n], np.int64)
        handle = ctypes.c_void_p()
        L = _lib.load()
        rview = None
        if resident is not None and all(resident[k].device == self.device for k in resident):
            r = resident
            if (r["mid_ptr"].numel() == self.n + 1 and r["mid_col"].numel() >= host["mid_col"].size
                    and r["outer_col"].numel() >= host["outer_col"].size):
                rview = _lib.SplitView(self.n, self.beta, None, _lib.ptr(r["mid_ptr"]), _lib.ptr(r["mid_col"]),
                                       _lib.ptr(r["mid_val"]), int(host["outer_col"].size),
                                       _lib.ptr(r["outer_row"]), _lib.ptr(r["outer_col"]),
                                       _lib.ptr(r["outer_val"]))
        with torch.cuda.device(self.device):
            _lib.check(L.pars3_plan_create_resident(ctypes.byref(view),
                                                    ctypes.byref(rview) if rview is not None else None,
                                                    ctypes.byref(opts), self.p, _lib.ptr(bs),
                                                    ctypes.byref(handle), None),
                       "pars3_plan_create")
        self._handle = handle
        self._L = L

    # -- hot entry points (device tensors in, device tensors out) ---------
    def matvec(self, x, y=None, stream=None, accumulate=False, strict=False):
        """y = A x for a contiguous float64 CUDA tensor x of length n
        (``accumulate``: y += A x, y not zeroed).  ``strict``: the product's
        fixed-point grid takes its scale from this x (a pure function of x,
        one extra read of x) rather than from the previous product's
        (pars3_plan_product, include/pars3.h)."""
        if y is None:
            y = self.torch.empty(self.n, dtype=self.torch.float64, device=self.device)
            if accumulate:
                y.zero_()
        flags = (_lib.PRODUCT_ACC if accumulate else 0) | (_lib.PRODUCT_STRICT if strict else 0)
        _lib.check(self._L.pars3_plan_product(self._handle, _lib.ptr(x), _lib.ptr(y), None, None, flags,
                                              _lib.stream_ptr(stream)), "pars3_plan_product")
        return y

    def matvec_dot(self, x, w, y=None, dot=None, stream=None, strict=False):
        """y = A x and dot = <y, w> (device scalar tensor); ``w`` may be ``y``."""
        t = self.torch
        if y is None:
            y = t.empty(self.n, dtype=t.float64, device=self.device)
        if w is None:
            w = y
        if dot is None:
            dot = t.empty(1, dtype=t.float64, device=self.device)
        _lib.check(self._L.pars3_plan_product(self._handle, _lib.ptr(x), _lib.ptr(y), _lib.ptr(w),
                                              _lib.ptr(dot), _lib.PRODUCT_STRICT if strict else 0,
                                              _lib.stream_ptr(stream)), "pars3_plan_product")
        return y, dot

    def xbound_slot(self):
        """Device address (int, 0 when the plan has none) of the word a kernel
        may fill with the bound of the next x (pars3_plan_xbound_slot)."""
        slot = ctypes.c_void_p()
        _lib.check(self._L.pars3_plan_xbound_slot(self._handle, ctypes.byref(slot)), "pars3_plan_xbound_slot")
        return int(slot.value or 0)

    def matvec_axpy(self, x, out, p, a, q, b, dot=None, stream=None, strict=False, xbound=False):
        """out = A x + a p + b q and, with ``dot`` (a device scalar tensor),
        dot = <out, out>: the product fused with the vector update that
        follows it in a Krylov step (pars3_plan_product_axpy).  ``a`` and ``b``
        are one-element CUDA tensors (device scalars, e.g. views of a solver's
        state), so the recurrence needs no host round trip.  ``out`` must not
        alias x, p or q.  ``xbound`` (with ``strict``): the kernel that produced
        x left its bound in ``xbound_slot()``, so the product skips its pass over x."""
        _lib.check(self._L.pars3_plan_product_axpy(
            self._handle, _lib.ptr(x), _lib.ptr(out), _lib.ptr(p), _lib.ptr(a), _lib.ptr(q), _lib.ptr(b),
            _lib.ptr(dot) if dot is not None else None,
            (_lib.PRODUCT_STRICT if strict else 0) | (_lib.PRODUCT_XBOUND if strict and xbound else 0),
            _lib.stream_ptr(stream)), "pars3_plan_product_axpy")
        return out

    # -- host-resident vectors: pipelined copies --------------------------
    def matvec_host(self, x, out=None, non_blocking=False, strict=True):
        """y = A x for a HOST float64 tensor x (pinned for overlap), result in
        the host tensor ``out``.  Three streams and double-buffered device
        vectors pipeline consecutive calls: call k+1's host->device copy runs
        on the copy engine while call k's product and device->host copy are
        still in flight (PCIe is full duplex).  With ``non_blocking`` the call
        returns once the work is enqueued: ``out`` (and re-use of ``x``) is
        safe after ``torch.cuda.synchronize()`` or ``self.host_sync()``."""
        torch = self.torch
        pl = getattr(self, "_pipe", None)
        if pl is None:
            dev = self.device
            pl = self._pipe = {
                "k": 0,
                "h2d": torch.cuda.Stream(dev), "comp": torch.cuda.Stream(dev),
                "d2h": torch.cuda.Stream(dev),
                "x": [torch.empty(self.n, dtype=torch.float64, device=dev) for _ in range(2)],
                "y": [torch.empty(self.n, dtype=torch.float64, device=dev) for _ in range(2)],
                "ev_x": [torch.cuda.Event() for _ in range(2)],
                "ev_y": [torch.cuda.Event() for _ in range(2)],
                "ev_out": [torch.cuda.Event() for _ in range(2)],
            }
        if out is None:
            out = torch.empty(self.n, dtype=torch.float64, pin_memory=x.is_pinned())
        b = pl["k"] & 1
        pl["k"] += 1
        h2d, comp, d2h = pl["h2d"], pl["comp"], pl["d2h"]
        # buffer b is free once call k-2's product (reads x[b]) and copy-out
        # (reads y[b]) are done
        h2d.wait_event(pl["ev_y"][b])
        with torch.cuda.stream(h2d):
            pl["x"][b].copy_(x, non_blocking=True)
        pl["ev_x"][b].record(h2d)
        comp.wait_event(pl["ev_x"][b])
        comp.wait_event(pl["ev_out"][b])
        self.matvec(pl["x"][b], pl["y"][b], stream=comp, strict=strict)
        pl["ev_y"][b].record(comp)
        d2h.wait_event(pl["ev_y"][b])
        with torch.cuda.stream(d2h):
            out.copy_(pl["y"][b], non_blocking=True)
        pl["ev_out"][b].record(d2h)
        if not non_blocking:
            pl["ev_out"][b].synchronize()
        return out

    def host_join(self, stream=None):
        """Make ``stream`` (default: the current stream) wait for every
        pipelined host product, without blocking the host."""
        pl = getattr(self, "_pipe", None)
        if pl is not None:
            (stream or self.torch.cuda.current_stream(self.device)).wait_stream(pl["d2h"])

    def host_sync(self):
        """Wait for every pipelined host product (matvec_host)."""
        pl = getattr(self, "_pipe", None)
        if pl is not None:
            pl["d2h"].synchronize()

    def status(self, stream=None) -> int:
        """Flags since the previous call (synchronises the stream).  Every
        product is exact whatever the input; these say
        how it got there: bit 0 -- a product was redone by the fp64 pass
        (non-finite x, x beyond the grid's bound, or a grid too coarse for
        the result), so it is exact but not bitwise repeatable; bit 1 -- some
        tiles accumulated in fp64 (the per-tile guard)."""
        f = ctypes.c_int32()
        _lib.check(self._L.pars3_plan_status(self._handle, ctypes.byref(f), _lib.stream_ptr(stream)),
                   "pars3_plan_status")
        return int(f.value)

    def profile(self, x, y=None, with_dot=True, reps=20, stream=None) -> dict:
        """Per-phase times of ``reps`` products (CUDA events on the stream):
        the main kernel, the finish / fix-up phase, the rest, the total (ms
        per product; pars3_plan_profile)."""
        if y is None:
            y = self.torch.empty(self.n, dtype=self.torch.float64, device=self.device)
        ms = np.zeros(4)
        _lib.check(self._L.pars3_plan_profile(self._handle, _lib.ptr(x), _lib.ptr(y), int(bool(with_dot)),
                                              int(reps), _lib.ptr(ms), _lib.stream_ptr(stream)),
                   "pars3_plan_profile")
        return {"main_ms": float(ms[0]), "finish_ms": float(ms[1]), "rest_ms": float(ms[2]),
                "total_ms": float(ms[3])}

    def kernel_count(self, with_dot: bool = False) -> int:
        c = ctypes.c_int32()
        _lib.check(self._L.pars3_plan_kernel_count(self._handle, int(with_dot), ctypes.byref(c)))
        return int(c.value)

    def plan_bytes(self) -> int:
        b = ctypes.c_int64()
        _lib.check(self._L.pars3_plan_bytes(self._handle, ctypes.byref(b)))
        return int(b.value)

    def stats(self) -> dict:
        a = np.zeros(20, dtype=np.int64)
        _lib.check(self._L.pars3_plan_stats(self._handle, _lib.ptr(a)))
        keys = ("tiles", "slices", "padded_slots", "entries", "windows", "max_local", "grid",
                "device_bytes", "list_tiles", "accum_words", "locality_order", "local_slots",
                "locality_dropped", "direct", "grid_form", "grid_hbits", "grid_cmax", "grid_ev",
                "built_on_device", "far_entries")
        return {k: int(v) for k, v in zip(keys, a)}

    def close(self):
        if getattr(self, "_handle", None) is not None and self._handle.value:
            self._L.pars3_plan_destroy(self._handle)
            self._handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dot(a, b, out=None, stream=None):
    """<a, b> of two float64 CUDA vectors into a device scalar (libpars3 k_dot)."""
    torch = require_cuda()
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=a.device)
    _lib.check(_lib.load().pars3_dot(a.numel(), _lib.ptr(a), _lib.ptr(b), _lib.ptr(out),
                                     _lib.stream_ptr(stream)), "pars3_dot")
    return out


class SssDevice:
    """Device copy of a whole SssMatrix (int32 row_ptr/col_ind) for the
    atomic comparison kernel."""

    def __init__(self, m, device=None):
        torch = require_cuda()
        self.device = torch.device(device if device is not None else "cuda")
        self.n = m.n
        self.row_ptr = torch.from_numpy(_c(m.row_ptr, np.int32)).to(self.device)
        self.col_ind = torch.from_numpy(_c(m.col_ind, np.int32)).to(self.device)
        self.off_diags = torch.from_numpy(_c(m.off_diags, np.float64)).to(self.device)
        self.diags = torch.from_numpy(_c(m.diags, np.float64)).to(self.device)


def _cache(obj):
    cache = getattr(obj, "_device", None)
    if cache is None:
        cache = {}
        object.__setattr__(obj, "_device", cache)
    return cache


def operator_for_split(s, p=1, block_start=None, device=None, options=None) -> Pars3Operator:
    """Operator for a BandSplit, cached on the split object."""
    key = ("split", int(p), str(device), tuple(options) if options else None)
    cache = _cache(s)
    op = cache.get(key)
    if op is None:
        # prepare_gpu(..., keep_device=True) leaves the split on the device: the first
        # plan takes it (no second upload) and releases it
        resident = cache.pop("resident_split", None)
        op = Pars3Operator(s.n, s.beta, s.diag, s.mid_ptr, s.mid_col, s.mid_val, s.outer_row,
                           s.outer_col, s.outer_val, p=p, block_start=block_start, device=device,
                           options=options, resident=resident)
        del resident
        cache[key] = op
    return op


def operator_for_sss(m, device=None, options=None) -> Pars3Operator:
    """Operator for a whole SssMatrix (every entry in the band, beta = n)."""
    key = ("sss", str(device), tuple(options) if options else None)
    cache = _cache(m)
    op = cache.get(key)
    if op is None:
        e = np.zeros(0, np.int32)
        op = Pars3Operator(m.n, max(1, m.n), m.diags, m.row_ptr, m.col_ind, m.off_diags, e, e,
                           np.zeros(0), device=device, options=options)
        cache[key] = op
    return op


def sss_device(m, device=None) -> SssDevice:
    key = ("sssdev", str(device))
    cache = _cache(m)
    d = cache.get(key)
    if d is None:
        d = SssDevice(m, device)
        cache[key] = d
    return d
