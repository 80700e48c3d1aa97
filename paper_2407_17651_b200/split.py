"""3-way band split, row partition and conflict plan (reference split.py).

``split_bands`` and ``classify_conflicts`` run natively in libpars3.so
(csrc/prep.cpp) and return the same arrays as split.py:116-141 and
split.py:303-361.  Dataclass names and fields follow the reference
(``BandSplit`` split.py:58-113, ``PartitionPlan`` split.py:191-266,
``ConflictReport`` split.py:269-300); column/row index arrays of the bands
are int32, pointers and plan arrays int64.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .formats import SssMatrix, StructuralError

__all__ = ["locality_order", "BandSplit", "PartitionPlan", "ConflictReport", "default_beta", "split_bands",
           "merge_splits", "partition_rows", "classify_conflicts", "conflict_report"]


def default_beta(n: int, bandwidth: int) -> int:
    """Middle half-width: n/1000 clamped to [8, bandwidth], at least 1 (D11)."""
    return max(1, min(max(8, n // 1000), bandwidth))


def _freeze(a):
    a.setflags(write=False)
    return a


@dataclass(frozen=True, eq=False)
class BandSplit:
    """diag + middle band (1 <= i-c <= beta, compressed rows) + outer triplets."""

    n: int
    beta: int
    diag: np.ndarray
    mid_ptr: np.ndarray
    mid_col: np.ndarray
    mid_val: np.ndarray
    outer_row: np.ndarray
    outer_col: np.ndarray
    outer_val: np.ndarray

    def __post_init__(self):
        if self.beta < 1:
            raise ValueError(f"split bandwidth must be at least 1, got {self.beta}")
        conv = {"diag": np.float64, "mid_ptr": np.int64, "mid_col": np.int32,
                "mid_val": np.float64, "outer_row": np.int32, "outer_col": np.int32,
                "outer_val": np.float64}
        arrs = {k: np.ascontiguousarray(getattr(self, k), dtype=t).ravel() for k, t in conv.items()}
        if (arrs["diag"].size != self.n or arrs["mid_ptr"].size != self.n + 1
                or arrs["mid_ptr"][0] != 0):
            raise StructuralError("diag/mid_ptr sizes do not match the dimension")
        if arrs["mid_ptr"][-1] != arrs["mid_col"].size or arrs["mid_col"].size != arrs["mid_val"].size:
            raise StructuralError("middle-band arrays disagree on entry count")
        if not (arrs["outer_row"].size == arrs["outer_col"].size == arrs["outer_val"].size):
            raise StructuralError("outer-band arrays disagree on entry count")
        for k, a in arrs.items():
            object.__setattr__(self, k, _freeze(a))
        object.__setattr__(self, "_device", None)

    @property
    def middle_count(self) -> int:
        return int(self.mid_col.size)

    @property
    def outer_count(self) -> int:
        return int(self.outer_col.size)

    def mid_rows(self) -> np.ndarray:
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.mid_ptr))


def split_bands(m: SssMatrix, beta: int) -> BandSplit:
    """Split at off-diagonal distance beta; storage order kept in each band."""
    if beta < 1:
        raise ValueError(f"split bandwidth must be at least 1, got {beta}")
    L = _lib.load()
    mid = _lib._c_i64()
    out = _lib._c_i64()
    import ctypes
    _lib.check(L.pars3_split_count(m.n, _lib.ptr(m.row_ptr), _lib.ptr(m.col_ind), int(beta),
                                   ctypes.byref(mid), ctypes.byref(out)), "split_bands")
    mp = np.empty(m.n + 1, dtype=np.int64)
    mc = np.empty(mid.value, dtype=np.int32)
    mv = np.empty(mid.value, dtype=np.float64)
    orow = np.empty(out.value, dtype=np.int32)
    ocol = np.empty(out.value, dtype=np.int32)
    oval = np.empty(out.value, dtype=np.float64)
    _lib.check(L.pars3_split_fill(m.n, _lib.ptr(m.row_ptr), _lib.ptr(m.col_ind),
                                  _lib.ptr(m.off_diags), int(beta), _lib.ptr(mp), _lib.ptr(mc),
                                  _lib.ptr(mv), _lib.ptr(orow), _lib.ptr(ocol), _lib.ptr(oval)),
               "split_bands")
    return BandSplit(m.n, int(beta), m.diags, mp, mc, mv, orow, ocol, oval)


def locality_order(s: BandSplit):
    """The internal order a device plan may adopt for locality (no reference
    counterpart; DESIGN.md §3 "locality order"): RCM of the split's graph
    after dropping the entries that no path of length 2 or 3 supports.
    Returns ``(Permutation, dropped)`` with ``forward[split label] =
    internal label`` and the number of directed edges the filter removed.
    Host-native; the plan applies it inside the product, so the caller's
    labels never change."""
    import ctypes

    from .reorder import Permutation
    L = _lib.load()
    view = _lib.SplitView(s.n, s.beta, _lib.ptr(s.diag), _lib.ptr(s.mid_ptr), _lib.ptr(s.mid_col),
                          _lib.ptr(s.mid_val), int(s.outer_col.size), _lib.ptr(s.outer_row),
                          _lib.ptr(s.outer_col), _lib.ptr(s.outer_val))
    fw = np.empty(s.n, dtype=np.int64)
    dropped = ctypes.c_int64()
    _lib.check(L.pars3_locality_order(ctypes.byref(view), _lib.ptr(fw), ctypes.byref(dropped)),
               "locality_order")
    return Permutation(fw), int(dropped.value)


def merge_splits(s: BandSplit) -> SssMatrix:
    """Inverse of split_bands, bit-exact (split.py:144-170): per row the outer
    columns (< i - beta) precede the middle ones."""
    oc = np.bincount(s.outer_row, minlength=s.n) if s.outer_count else np.zeros(s.n, np.int64)
    mc = np.diff(s.mid_ptr)
    rp = np.zeros(s.n + 1, dtype=np.int64)
    np.cumsum(oc + mc, out=rp[1:])
    optr = np.zeros(s.n + 1, dtype=np.int64)
    np.cumsum(oc, out=optr[1:])
    col = np.empty(int(rp[-1]), dtype=np.int32)
    val = np.empty(int(rp[-1]), dtype=np.float64)
    orow = s.outer_row.astype(np.int64)
    d_out = rp[orow] + (np.arange(s.outer_count) - optr[orow])
    mrow = s.mid_rows()
    d_mid = rp[mrow] + oc[mrow] + (np.arange(s.middle_count) - s.mid_ptr[mrow])
    col[d_out], val[d_out] = s.outer_col, s.outer_val
    col[d_mid], val[d_mid] = s.mid_col, s.mid_val
    return SssMatrix(s.n, rp, col, val, s.diag)


def partition_rows(n: int, p: int) -> np.ndarray:
    """p+1 block boundaries, the first n mod p blocks one row larger (D10)."""
    if p < 1:
        raise ValueError(f"worker count must be at least 1, got {p}")
    if p > n:
        raise ValueError(f"worker count {p} exceeds the {n} available rows")
    q, r = divmod(n, p)
    sizes = np.full(p, q, dtype=np.int64)
    sizes[:r] += 1
    out = np.zeros(p + 1, dtype=np.int64)
    np.cumsum(sizes, out=out[1:])
    return out


@dataclass(frozen=True, eq=False)
class PartitionPlan:
    """Block layout + conflict classification of the middle band."""

    n: int
    p: int
    beta: int
    block_start: np.ndarray
    row_owner: np.ndarray
    safe_start: np.ndarray
    conflict_idx: np.ndarray
    conflict_ptr: np.ndarray
    conflict_target: np.ndarray
    apply_order: np.ndarray
    apply_ptr: np.ndarray
    halo_lo: np.ndarray

    def __post_init__(self):
        for name in ("block_start", "row_owner", "safe_start", "conflict_idx", "conflict_ptr",
                     "conflict_target", "apply_order", "apply_ptr", "halo_lo"):
            object.__setattr__(self, name,
                               _freeze(np.array(getattr(self, name), dtype=np.int64).ravel()))
        bs = self.block_start
        if bs.size != self.p + 1 or bs[0] != 0 or bs[-1] != self.n:
            raise StructuralError("block_start must run from 0 to n over p blocks")
        sizes = np.diff(bs)
        if np.any(sizes < 1):
            raise StructuralError("every block must own at least one row")
        if self.p and sizes.max() - sizes.min() > 1:
            raise StructuralError("block sizes must differ by at most one row")

    @property
    def conflict_count(self) -> int:
        return int(self.conflict_idx.size)


@dataclass(frozen=True)
class ConflictReport:
    """Per-worker accounting of a partition (split.py:269-300)."""

    n: int
    p: int
    beta: int
    middle_count: int
    outer_count: int
    conflict_count: int
    rows_per_worker: tuple
    safe_per_worker: tuple
    conflicts_per_worker: tuple
    incoming_per_worker: tuple
    halo_width: tuple

    def as_dict(self) -> dict:
        return {
            "n": self.n, "beta": self.beta, "nnzDiag": self.n, "nnzMiddle": self.middle_count,
            "nnzOuter": self.outer_count, "conflictCount": self.conflict_count,
            "perWorker": [{"rows": r, "safe": s, "conflicts": c} for r, s, c in
                          zip(self.rows_per_worker, self.safe_per_worker,
                              self.conflicts_per_worker)],
        }


def classify_conflicts(s: BandSplit, boundaries) -> tuple[PartitionPlan, ConflictReport]:
    """Safe/conflict classification of every middle entry against a block
    partition (split.py:303-361), computed natively."""
    import ctypes
    bs = np.array(boundaries, dtype=np.int64).ravel()
    p = bs.size - 1
    # validate like PartitionPlan would, before the native pass
    if p < 1 or bs[0] != 0 or bs[-1] != s.n:
        raise StructuralError("block_start must run from 0 to n over p blocks")
    sizes = np.diff(bs)
    if np.any(sizes < 1):
        raise StructuralError("every block must own at least one row")
    if sizes.max() - sizes.min() > 1:
        raise StructuralError("block sizes must differ by at most one row")
    L = _lib.load()
    k = _lib._c_i64()
    args = [s.n, _lib.ptr(s.mid_ptr), _lib.ptr(s.mid_col), p, _lib.ptr(bs), ctypes.byref(k)]
    _lib.check(L.pars3_classify_conflicts(*args, *([None] * 8)), "classify_conflicts")
    kk = int(k.value)
    ro = np.empty(s.n, np.int64)
    ss = np.empty(s.n, np.int64)
    ci = np.empty(max(kk, 1), np.int64)
    cp = np.empty(p + 1, np.int64)
    ct = np.empty(max(kk, 1), np.int64)
    ao = np.empty(max(kk, 1), np.int64)
    ap = np.empty(p + 1, np.int64)
    hl = np.empty(p, np.int64)
    _lib.check(L.pars3_classify_conflicts(*args, *(_lib.ptr(a) for a in
                                                   (ro, ss, ci, cp, ct, ao, ap, hl))),
               "classify_conflicts")
    plan = PartitionPlan(n=s.n, p=p, beta=s.beta, block_start=bs, row_owner=ro, safe_start=ss,
                         conflict_idx=ci[:kk], conflict_ptr=cp, conflict_target=ct[:kk],
                         apply_order=ao[:kk], apply_ptr=ap, halo_lo=hl)
    return plan, conflict_report(s, plan)


def conflict_report(s: BandSplit, plan: PartitionPlan) -> ConflictReport:
    per_conf = np.diff(plan.conflict_ptr)
    mid_w = s.mid_ptr[plan.block_start[1:]] - s.mid_ptr[plan.block_start[:-1]]
    return ConflictReport(
        n=s.n, p=plan.p, beta=s.beta, middle_count=s.middle_count, outer_count=s.outer_count,
        conflict_count=plan.conflict_count,
        rows_per_worker=tuple(int(x) for x in np.diff(plan.block_start)),
        safe_per_worker=tuple(int(a - b) for a, b in zip(mid_w, per_conf)),
        conflicts_per_worker=tuple(int(x) for x in per_conf),
        incoming_per_worker=tuple(int(x) for x in np.diff(plan.apply_ptr)),
        halo_width=tuple(int(b - h) for b, h in zip(plan.block_start[:-1], plan.halo_lo)))
