"""CPU oracle for the PARS3 path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and
only as the checker or as the timed CPU baseline.  The product package
``paper_2407_17651_b200`` never imports it.

Two halves:

* ``oracle.c`` (compiled to ``oracle/_build/liboracle.so`` by
  ``oracle/Makefile``) restates the reference's numba kernels --
  ``_spmv_sss`` (serial.py:50-61), ``_pars3`` (parallel.py:60-120) and the
  RCM drivers (reorder.py:137-286) -- in C.
* this file restates the reference's numpy preprocessing --
  ``split_bands`` (split.py:116-141), ``partition_rows`` (split.py:173-188),
  ``classify_conflicts`` (split.py:303-361), ``default_beta``
  (split.py:44-50), ``compute_bandwidth`` (reorder.py:120-134) and the
  permute-then-to-SSS chain ``coo_to_sss(apply_permutation(...))``
  (reorder.py:289-297, formats.py:413-475) -- in numpy, on int64 arrays,
  returning plain dicts of arrays.

Parity pinned against the live reference: tests/golden/make_golden.py runs
the unmodified reference package on the same seeded inputs and stores its
outputs; tests/test_oracle_golden.py checks this module against them.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


def build() -> str:
    """Compile oracle.c (idempotent; make decides)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        L.oracle_spmv_sss.argtypes = [ctypes.c_int64, _i64p, _i64p, _f64p, _f64p, _f64p, _f64p]
        L.oracle_pars3.argtypes = [_i64p, _i64p, _f64p, _f64p, ctypes.c_int64, _i64p, _i64p,
                                   _f64p, _i64p, _i64p, _i64p, _i64p, _i64p, _i64p, _f64p,
                                   _f64p, _f64p, ctypes.c_int64, ctypes.c_int]
        L.oracle_pattern_from_sss.argtypes = [ctypes.c_int64, _i64p, _i64p, _i64p, _i64p]
        L.oracle_rcm_order.argtypes = [ctypes.c_int64, _i64p, _i64p, _i64p]
        for f in (L.oracle_spmv_sss, L.oracle_pars3, L.oracle_pattern_from_sss,
                  L.oracle_rcm_order):
            f.restype = None
        _lib = L
    return _lib


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a, t):
    return a.ctypes.data_as(t)


# ----------------------------------------------------------------- kernels

def spmv_serial(row_ptr, col_ind, off_diags, diags, x) -> np.ndarray:
    """serial.py:64-73 via the C restatement of _spmv_sss (bit-identical)."""
    rp, ci, od, dg, xx = _i64(row_ptr), _i64(col_ind), _f64(off_diags), _f64(diags), _f64(x)
    n = dg.size
    y = np.zeros(n)
    lib().oracle_spmv_sss(n, _p(rp, _i64p), _p(ci, _i64p), _p(od, _f64p), _p(dg, _f64p),
                          _p(xx, _f64p), _p(y, _f64p))
    return y


def spmv_pars3(split: dict, plan: dict, x, nthreads: int | None = None) -> np.ndarray:
    """parallel.py:136-183 via the C restatement of _pars3."""
    n = int(split["n"])
    xx = _f64(x)
    y = np.zeros(n)
    k = int(plan["conflict_idx"].size)
    msg = np.empty(max(k, 1))
    a = {name: _i64(split[name]) for name in ("mid_ptr", "mid_col", "outer_row", "outer_col")}
    v = {name: _f64(split[name]) for name in ("mid_val", "diag", "outer_val")}
    q = {name: _i64(plan[name]) for name in ("block_start", "safe_start", "conflict_ptr",
                                             "conflict_idx", "apply_order", "apply_ptr")}
    p = int(q["block_start"].size - 1)
    nt = int(nthreads if nthreads else p)
    lib().oracle_pars3(_p(a["mid_ptr"], _i64p), _p(a["mid_col"], _i64p), _p(v["mid_val"], _f64p),
                       _p(v["diag"], _f64p), int(a["outer_row"].size), _p(a["outer_row"], _i64p),
                       _p(a["outer_col"], _i64p), _p(v["outer_val"], _f64p),
                       _p(q["block_start"], _i64p), _p(q["safe_start"], _i64p),
                       _p(q["conflict_ptr"], _i64p), _p(q["conflict_idx"], _i64p),
                       _p(q["apply_order"], _i64p), _p(q["apply_ptr"], _i64p), _p(xx, _f64p),
                       _p(y, _f64p), _p(msg, _f64p), p, nt)
    return y


# ----------------------------------------------------------- preprocessing

def pattern_from_sss(n, row_ptr, col_ind):
    """Symmetrised adjacency (reorder.py:103-117) of an SSS pattern."""
    rp, ci = _i64(row_ptr), _i64(col_ind)
    indptr = np.empty(n + 1, dtype=np.int64)
    indices = np.empty(2 * ci.size, dtype=np.int64)
    lib().oracle_pattern_from_sss(n, _p(rp, _i64p), _p(ci, _i64p), _p(indptr, _i64p),
                                  _p(indices, _i64p))
    return indptr, indices


def pattern_from_coo(n, row, col):
    """reorder.py:103-117 restated: unique both-direction off-diagonal keys."""
    r, c = _i64(row), _i64(col)
    off = r != c
    r, c = r[off], c[off]
    key = np.unique(np.concatenate((r * n + c, c * n + r)))
    counts = np.bincount(key // n, minlength=n) if n else np.zeros(0, np.int64)
    indptr = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
    return indptr, (key % n if n else key).astype(np.int64)


def rcm_order(n, indptr, indices) -> np.ndarray:
    """reorder.py:251-286 via the C restatement; returns forward[old]=new."""
    ip, ix = _i64(indptr), _i64(indices)
    fw = np.empty(n, dtype=np.int64)
    lib().oracle_rcm_order(n, _p(ip, _i64p), _p(ix, _i64p), _p(fw, _i64p))
    return fw


def permute_sss(n, row_ptr, col_ind, off_diags, diags, forward):
    """coo_to_sss(apply_permutation(sss_to_coo(m), perm)) restated for the
    off-diagonal part (reorder.py:289-297, formats.py:413-490): entry (i,c,v)
    moves to (f[i], f[c]); the lower one of the mirrored pair keeps v if
    f[i] > f[c], else it is the mirror (f[c], f[i]) holding -v.  Rows sorted,
    columns ascending.  The diagonal is permuted alongside."""
    rp, ci, od, fw = _i64(row_ptr), _i64(col_ind), _f64(off_diags), _i64(forward)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    fr, fc = fw[rows], fw[ci]
    swap = fr < fc
    nr = np.where(swap, fc, fr)
    nc = np.where(swap, fr, fc)
    nv = np.where(swap, -od, od)
    order = np.argsort(nr * n + nc, kind="stable")
    nr, nc, nv = nr[order], nc[order], nv[order]
    counts = np.bincount(nr, minlength=n)
    new_rp = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
    new_diag = np.empty(n)
    new_diag[fw] = _f64(diags)
    return new_rp, nc.astype(np.int64), nv, new_diag


def compute_bandwidth(n, row_ptr, col_ind) -> int:
    """reorder.py:120-134 for SSS input."""
    ci = _i64(col_ind)
    if ci.size == 0:
        return 0
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(_i64(row_ptr)))
    return int(np.max(rows - ci))


def default_beta(n: int, bandwidth: int) -> int:
    """split.py:44-50."""
    return max(1, min(max(8, n // 1000), bandwidth))


def split_bands(n, row_ptr, col_ind, off_diags, diags, beta) -> dict:
    """split.py:116-141."""
    rp, ci, od = _i64(row_ptr), _i64(col_ind), _f64(off_diags)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    in_mid = (rows - ci) <= beta
    mid_counts = np.bincount(rows[in_mid], minlength=n)
    return {
        "n": n, "beta": int(beta), "diag": _f64(diags),
        "mid_ptr": np.concatenate(([0], np.cumsum(mid_counts))).astype(np.int64),
        "mid_col": ci[in_mid], "mid_val": od[in_mid],
        "outer_row": rows[~in_mid], "outer_col": ci[~in_mid], "outer_val": od[~in_mid],
    }


def partition_rows(n: int, p: int) -> np.ndarray:
    """split.py:173-188 (front-loaded remainder)."""
    q, r = divmod(n, p)
    sizes = np.full(p, q, dtype=np.int64)
    sizes[:r] += 1
    return np.concatenate(([0], np.cumsum(sizes))).astype(np.int64)


def classify_conflicts(split: dict, block_start) -> dict:
    """split.py:303-361 (the PartitionPlan fields)."""
    n = int(split["n"])
    bs = _i64(block_start)
    p = bs.size - 1
    row_owner = np.searchsorted(bs, np.arange(n, dtype=np.int64), side="right") - 1
    mid_ptr, mid_col = split["mid_ptr"], split["mid_col"]
    mid_rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(mid_ptr))
    owner = row_owner[mid_rows]
    is_conflict = mid_col < bs[owner]
    safe_start = mid_ptr[:-1] + np.bincount(mid_rows[is_conflict], minlength=n)
    conflict_idx = np.flatnonzero(is_conflict).astype(np.int64)
    conflict_ptr = np.concatenate(([0], np.cumsum(np.bincount(owner[conflict_idx], minlength=p))))
    conflict_target = row_owner[mid_col[conflict_idx]]
    apply_order = np.argsort(conflict_target, kind="stable").astype(np.int64)
    apply_ptr = np.concatenate(([0], np.cumsum(np.bincount(conflict_target, minlength=p))))
    halo_lo = bs[:p].copy()
    for w in range(p):
        mine = conflict_idx[conflict_ptr[w]:conflict_ptr[w + 1]]
        if mine.size:
            halo_lo[w] = int(mid_col[mine].min())
    return {
        "n": n, "p": p, "beta": int(split["beta"]), "block_start": bs,
        "row_owner": row_owner.astype(np.int64), "safe_start": safe_start.astype(np.int64),
        "conflict_idx": conflict_idx, "conflict_ptr": conflict_ptr.astype(np.int64),
        "conflict_target": conflict_target.astype(np.int64), "apply_order": apply_order,
        "apply_ptr": apply_ptr.astype(np.int64), "halo_lo": halo_lo.astype(np.int64),
    }


def rel_err(y, y_ref) -> float:
    """cli.py:130-134 / SPEC D14: ||y - y_ref||_inf / max(1, ||y_ref||_inf)."""
    y, y_ref = np.asarray(y, np.float64), np.asarray(y_ref, np.float64)
    if y_ref.size == 0:
        return 0.0
    return float(np.max(np.abs(y - y_ref)) / max(1.0, float(np.max(np.abs(y_ref)))))
