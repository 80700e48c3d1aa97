"""Bandwidth reduction by reverse Cuthill-McKee (reference reorder.py).

``rcm_order`` runs the native level-synchronous RCM in libpars3.so
(csrc/prep.cpp), which reproduces the reference's labels bit-exactly
(reorder.py:251-286; deterministic George-Liu start, (degree, index)
children, components by smallest index, isolated nodes in scan order).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .formats import CooMatrix, SssMatrix, StructuralError, coo_normalize

__all__ = ["AdjacencyPattern", "Permutation", "pattern_from_coo", "pattern_from_sss",
           "compute_bandwidth", "rcm_order", "apply_permutation", "permute_sss",
           "read_permutation", "write_permutation", "rcm_order_sss"]


@dataclass(frozen=True, eq=False)
class AdjacencyPattern:
    """Undirected adjacency, CSR with ascending neighbours (reorder.py:34-63)."""

    n: int
    indptr: np.ndarray
    indices: np.ndarray

    def __post_init__(self):
        ip = np.ascontiguousarray(self.indptr, dtype=np.int64).ravel()
        ix = np.ascontiguousarray(self.indices, dtype=np.int32).ravel()
        if ip.size != self.n + 1 or ip[0] != 0 or ip[-1] != ix.size:
            raise StructuralError("indptr must run from 0 to len(indices) with n + 1 entries")
        if np.any(ip[1:] < ip[:-1]):
            raise StructuralError("indptr must be non-decreasing")
        if ix.size and (ix.min() < 0 or ix.max() >= self.n):
            raise StructuralError("neighbor index out of range")
        ip.setflags(write=False)
        ix.setflags(write=False)
        object.__setattr__(self, "indptr", ip)
        object.__setattr__(self, "indices", ix)

    @property
    def degrees(self) -> np.ndarray:
        return np.diff(self.indptr)


@dataclass(frozen=True, eq=False)
class Permutation:
    """``forward[old] = new``, ``inverse[new] = old`` (reorder.py:66-100)."""

    forward: np.ndarray
    inverse: np.ndarray = field(init=False)

    def __post_init__(self):
        fw = np.array(self.forward, dtype=np.int64).ravel()
        n = fw.size
        if n and (fw.min() < 0 or fw.max() >= n):
            raise StructuralError("permutation image out of range")
        seen = np.zeros(n, dtype=bool)
        seen[fw] = True
        if not seen.all():
            raise StructuralError("permutation is not a bijection")
        inv = np.empty(n, dtype=np.int64)
        inv[fw] = np.arange(n, dtype=np.int64)
        fw.setflags(write=False)
        inv.setflags(write=False)
        object.__setattr__(self, "forward", fw)
        object.__setattr__(self, "inverse", inv)

    @property
    def n(self) -> int:
        return int(self.forward.size)

    @classmethod
    def identity(cls, n: int) -> "Permutation":
        return cls(np.arange(n, dtype=np.int64))


def pattern_from_coo(m: CooMatrix) -> AdjacencyPattern:
    """Symmetrised off-diagonal pattern of a triplet matrix (reorder.py:103-117).
    Explicit zeros count as edges."""
    m = coo_normalize(m)
    off = m.row != m.col
    r, c = m.row[off], m.col[off]
    key = np.unique(np.concatenate((r * m.n + c, c * m.n + r)))
    counts = np.bincount(key // m.n, minlength=m.n) if m.n else np.zeros(0, np.int64)
    ip = np.zeros(m.n + 1, dtype=np.int64)
    np.cumsum(counts, out=ip[1:])
    return AdjacencyPattern(m.n, ip, key % m.n if m.n else key)


def pattern_from_sss(m: SssMatrix) -> AdjacencyPattern:
    """Same pattern as ``pattern_from_coo(sss_to_coo(m))``, built natively
    from the skyline arrays (no 2m-key sort)."""
    L = _lib.load()
    ip = np.empty(m.n + 1, dtype=np.int64)
    ix = np.empty(2 * m.nnz_offdiag, dtype=np.int32)
    _lib.check(L.pars3_pattern_from_lower(m.n, _lib.ptr(m.row_ptr), _lib.ptr(m.col_ind),
                                          _lib.ptr(ip), _lib.ptr(ix)), "pattern_from_sss")
    return AdjacencyPattern(m.n, ip, ix)


def compute_bandwidth(m) -> int:
    """Largest |i - j| over stored off-diagonals (reorder.py:120-134)."""
    if isinstance(m, SssMatrix):
        if m.nnz_offdiag == 0:
            return 0
        return int(np.max(m.row_indices() - m.col_ind))
    if isinstance(m, CooMatrix):
        if m.nnz == 0:
            return 0
        return int(np.max(np.abs(m.row - m.col)))
    raise TypeError(f"expected CooMatrix or SssMatrix, got {type(m).__name__}")


def _upload(a, dtype, dev):
    """Host array -> device tensor (frozen arrays are read, never written)."""
    import warnings

    import torch
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)  # torch warns on read-only numpy buffers
        return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).to(dev)


def rcm_order(pattern: AdjacencyPattern, nthreads: int = 0, device=None) -> Permutation:
    """Reverse Cuthill-McKee labels, bit-identical to reorder.py:251-286.

    Host-native by default (``nthreads`` OpenMP threads); with ``device``
    (e.g. ``"cuda"``) the pattern is uploaded and ordered on the GPU
    (``pars3_rcm_order_device``), same labels."""
    L = _lib.load()
    if device is not None:
        from .device import require_cuda
        torch = require_cuda()
        dev = torch.device(device)
        ip = _upload(pattern.indptr, np.int64, dev)
        ix = _upload(pattern.indices, np.int32, dev)
        fw = torch.empty(pattern.n, dtype=torch.int64, device=dev)
        with torch.cuda.device(dev):
            _lib.check(L.pars3_rcm_order_device(pattern.n, _lib.ptr(ip), _lib.ptr(ix), _lib.ptr(fw),
                                                _lib.stream_ptr()), "rcm_order")
        return Permutation(fw.cpu().numpy())
    fw = np.empty(pattern.n, dtype=np.int64)
    _lib.check(L.pars3_rcm_order(pattern.n, _lib.ptr(pattern.indptr), _lib.ptr(pattern.indices),
                                 _lib.ptr(fw), int(nthreads)), "rcm_order")
    return Permutation(fw)


def rcm_order_sss(m: SssMatrix, device="cuda") -> Permutation:
    """``rcm_order(pattern_from_sss(m))`` on the GPU: the symmetric adjacency is
    built on the device from the skyline arrays, then ordered there."""
    from .device import require_cuda
    torch = require_cuda()
    dev = torch.device(device)
    rp = _upload(m.row_ptr, np.int64, dev)
    ci = _upload(m.col_ind, np.int32, dev)
    fw = torch.empty(m.n, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.load().pars3_rcm_order_lower_device(
            m.n, _lib.ptr(rp), _lib.ptr(ci), int(m.nnz_offdiag), _lib.ptr(fw), _lib.stream_ptr()),
            "rcm_order_sss")
    return Permutation(fw.cpu().numpy())


def apply_permutation(m: CooMatrix, perm: Permutation) -> CooMatrix:
    """Entry (i, j, v) moves to (forward[i], forward[j], v), normalized
    (reorder.py:289-297)."""
    if perm.n != m.n:
        raise ValueError(f"permutation is over {perm.n} indices, matrix has {m.n}")
    return coo_normalize(CooMatrix(m.n, perm.forward[m.row], perm.forward[m.col], m.val))


def permute_sss(m: SssMatrix, perm: Permutation, nthreads: int = 0) -> SssMatrix:
    """``coo_to_sss(apply_permutation(sss_to_coo(m), perm))`` computed
    natively on the skyline arrays (same arrays, bit for bit)."""
    if perm.n != m.n:
        raise ValueError(f"permutation is over {perm.n} indices, matrix has {m.n}")
    L = _lib.load()
    rp = np.empty(m.n + 1, dtype=np.int64)
    ci = np.empty(m.nnz_offdiag, dtype=np.int32)
    od = np.empty(m.nnz_offdiag, dtype=np.float64)
    dg = np.empty(m.n, dtype=np.float64)
    _lib.check(L.pars3_permute_lower(m.n, _lib.ptr(m.row_ptr), _lib.ptr(m.col_ind),
                                     _lib.ptr(m.off_diags), _lib.ptr(m.diags),
                                     _lib.ptr(perm.forward), _lib.ptr(rp), _lib.ptr(ci),
                                     _lib.ptr(od), _lib.ptr(dg), int(nthreads)), "permute_sss")
    return SssMatrix._trusted(m.n, rp, ci, od, dg)


def write_permutation(path, perm: Permutation) -> None:
    """Permutation text file (reorder.py:300-305), written natively."""
    from .mmio import write_permutation as _w
    _w(path, perm)


def read_permutation(path) -> Permutation:
    """Read a permutation file (reorder.py:308-333), parsed natively."""
    from .mmio import read_permutation as _r
    return _r(path)
