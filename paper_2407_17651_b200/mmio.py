"""Matrix Market coordinate, dense-vector and permutation text files.

Same names, arguments, results and errors as the reference's
``skewspmv.mmio`` (mmio.py:27-223) and its permutation files
(reorder.py:300-333).  Reading and writing run in libpars3's native
parallel parser/formatter (csrc/mmio.cpp); a file outside the canonical
fast-path syntax (or one the reference rejects) is re-read by ``_exact_*``,
a restatement of the reference's line-by-line reader, so the error raised
-- ``ParseError`` with the 1-based line number, or ``StructuralError`` -- is
the reference's.  Values round-trip bit-exactly ("%.17g", correctly rounded
parsing).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from .formats import CooMatrix, StructuralError, coo_normalize, validate_skew

__all__ = ["ParseError", "read_matrix", "write_matrix", "read_vector", "write_vector",
           "read_permutation", "write_permutation", "QUALIFIERS", "VALUE_FMT"]

QUALIFIERS = ("general", "symmetric", "skew-symmetric")
VALUE_FMT = "%.17g"  # reproduces every float64 exactly (mmio.py:24-25)


class ParseError(ValueError):
    """Malformed Matrix Market content; carries the 1-based line number."""

    def __init__(self, lineno: int, message: str):
        super().__init__(f"line {lineno}: {message}")
        self.lineno = lineno


def _path(p) -> bytes:
    return os.fsencode(os.fspath(p))


# ---------------------------------------------------------------- matrices
def _expand(n, rows, cols, vals, qual):
    """Materialise the implied triangle of a symmetric / skew file."""
    if qual != "general":
        off = rows != cols
        sign = -1.0 if qual == "skew-symmetric" else 1.0
        rows, cols, vals = (np.concatenate((rows, cols[off])), np.concatenate((cols, rows[off])),
                            np.concatenate((vals, sign * vals[off])))
    return coo_normalize(CooMatrix(n, rows, cols, vals)), qual


def read_matrix(path) -> tuple[CooMatrix, str]:
    """Read a Matrix Market ``coordinate real`` file (general, symmetric or
    skew-symmetric) into a normalized CooMatrix with both triangles, and the
    declared qualifier (mmio.py:52-149)."""
    L = _lib.load()
    h = ctypes.c_void_p()
    n, nnz, q = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
    rc = L.pars3_mm_open(_path(path), ctypes.byref(h), ctypes.byref(n), ctypes.byref(nnz),
                         ctypes.byref(q))
    if rc == _lib.PARS3_SLOW_PATH:
        return _exact_read_matrix(path)
    _lib.check(rc, "read_matrix")
    try:
        rows = np.empty(nnz.value, dtype=np.int64)
        cols = np.empty(nnz.value, dtype=np.int64)
        vals = np.empty(nnz.value, dtype=np.float64)
        rc = L.pars3_mm_fill(h, _lib.ptr(rows), _lib.ptr(cols), _lib.ptr(vals), 0)
    finally:
        L.pars3_mm_close(h)
    if rc == _lib.PARS3_SLOW_PATH:
        return _exact_read_matrix(path)
    _lib.check(rc, "read_matrix")
    return _expand(n.value, rows, cols, vals, QUALIFIERS[q.value])


def _header_qualifier(line: str, lineno: int) -> str:
    f = line.split()
    if len(f) != 5 or f[0] != "%%MatrixMarket":
        raise ParseError(lineno, f"expected a %%MatrixMarket header, got {line.rstrip()!r}")
    checks = (("object", f[1], "matrix", "only 'matrix'"),
              ("format", f[2], "coordinate", "only 'coordinate'"),
              ("field", f[3], "real", "only 'real'"))
    for what, got, want, only in checks:
        if got.lower() != want:
            raise ParseError(lineno, f"unsupported {what} {got!r}, {only}")
    qual = f[4].lower()
    if qual not in QUALIFIERS:
        raise ParseError(lineno, f"unsupported qualifier {qual!r}, expected one of {QUALIFIERS}")
    return qual


def _exact_read_matrix(path):
    """The reference reader's exact semantics, line by line (slow path)."""
    with open(path, "r", encoding="ascii") as fh:
        text = fh.readlines()
    if not text:
        raise ParseError(1, "empty file")
    qual = _header_qualifier(text[0], 1)

    def skipped(s):
        return s.startswith("%") or not s.strip()

    k = 1
    while k < len(text) and skipped(text[k]):
        k += 1
    if k == len(text):
        raise ParseError(len(text), "missing size line")
    sz = text[k].split()
    if len(sz) != 3:
        raise ParseError(k + 1, f"size line must be 'rows cols nnz', got {text[k].rstrip()!r}")
    try:
        nrows, ncols, nnz = int(sz[0]), int(sz[1]), int(sz[2])
    except ValueError:
        raise ParseError(k + 1, f"non-integer size line {text[k].rstrip()!r}") from None
    if nrows != ncols:
        raise StructuralError(f"matrix must be square, got {nrows}x{ncols}")
    if nnz < 0:
        raise ParseError(k + 1, f"negative entry count {nnz}")
    rows = np.empty(nnz, dtype=np.int64)
    cols = np.empty(nnz, dtype=np.int64)
    vals = np.empty(nnz, dtype=np.float64)
    got = 0
    for idx in range(k + 1, len(text)):
        s = text[idx]
        if skipped(s):
            continue
        ln = idx + 1
        f = s.split()
        if len(f) != 3:
            raise ParseError(ln, f"entry line must be 'row col value', got {s.rstrip()!r}")
        try:
            i, j, v = int(f[0]), int(f[1]), float(f[2])
        except ValueError:
            raise ParseError(ln, f"malformed entry {s.rstrip()!r}") from None
        if got >= nnz:
            raise StructuralError(f"file contains more than the declared {nnz} entries")
        if not (1 <= i <= nrows and 1 <= j <= ncols):
            raise StructuralError(f"line {ln}: entry ({i}, {j}) outside declared {nrows}x{ncols} matrix")
        if qual != "general" and j > i:
            raise StructuralError(f"line {ln}: {qual} file must store only the lower triangle, "
                                  f"got entry ({i}, {j})")
        if qual == "skew-symmetric" and i == j and v != 0.0:
            raise StructuralError(f"line {ln}: skew-symmetric file has nonzero diagonal entry "
                                  f"({i}, {i}) = {f[2]}")
        rows[got], cols[got], vals[got] = i - 1, j - 1, v
        got += 1
    if got != nnz:
        raise StructuralError(f"declared {nnz} entries but file contains {got}")
    return _expand(nrows, rows, cols, vals, qual)


def _is_symmetric(m: CooMatrix) -> bool:
    """Every stored (i, j) has (j, i) with the same value (zeros may be lone)."""
    if m.nnz == 0:
        return True
    key = m.row * m.n + m.col
    want = m.col * m.n + m.row
    pos = np.searchsorted(key, want)
    at = np.minimum(pos, key.size - 1)
    hit = (pos < key.size) & (key[at] == want)
    if not np.all(hit | (m.val == 0.0)):
        return False
    return bool(np.all(m.val[hit] == m.val[at[hit]]))


def write_matrix(path, m: CooMatrix, qualifier: str = "general") -> None:
    """Write triplets as Matrix Market text (mmio.py:152-187): symmetric and
    skew-symmetric qualifiers are validated and store the lower triangle
    only; values with 17 significant digits."""
    if qualifier not in QUALIFIERS:
        raise ValueError(f"qualifier must be one of {QUALIFIERS}, got {qualifier!r}")
    m = coo_normalize(m)
    if qualifier == "skew-symmetric":
        rep = validate_skew(m)
        if rep.asymmetry_count or rep.violation_count or rep.diagonal_class != "zero":
            raise StructuralError(
                "matrix is not strictly skew-symmetric: "
                f"{rep.asymmetry_count} pattern asymmetries, "
                f"{rep.violation_count} value violations, "
                f"diagonal class {rep.diagonal_class!r}")
        keep = m.row > m.col
    elif qualifier == "symmetric":
        if not _is_symmetric(m):
            raise StructuralError("matrix is not symmetric; cannot write 'symmetric' qualifier")
        keep = m.row >= m.col
    else:
        keep = np.ones(m.nnz, dtype=bool)
    r = np.ascontiguousarray(m.row[keep])
    c = np.ascontiguousarray(m.col[keep])
    v = np.ascontiguousarray(m.val[keep])
    _lib.check(_lib.load().pars3_mm_write(_path(path), qualifier.encode(), m.n, r.size,
                                          _lib.ptr(r), _lib.ptr(c), _lib.ptr(v), 0),
               "write_matrix")


# ----------------------------------------------------------------- vectors
def read_vector(path) -> np.ndarray:
    """One real per line; blank and '%' lines skipped (mmio.py:203-215)."""
    L = _lib.load()
    cnt = ctypes.c_int64()
    rc = L.pars3_vector_read(_path(path), None, ctypes.byref(cnt), 0)
    if rc == _lib.PARS3_OK:
        x = np.empty(cnt.value, dtype=np.float64)
        rc = L.pars3_vector_read(_path(path), _lib.ptr(x), ctypes.byref(cnt), 0)
        if rc == _lib.PARS3_OK:
            return x
    if rc != _lib.PARS3_SLOW_PATH:
        _lib.check(rc, "read_vector")
    vals = []
    with open(path, "r", encoding="ascii") as fh:
        for ln, line in enumerate(fh, start=1):
            s = line.strip()
            if s and not s.startswith("%"):
                try:
                    vals.append(float(s))
                except ValueError:
                    raise ParseError(ln, f"malformed vector entry {s!r}") from None
    return np.array(vals, dtype=np.float64)


def write_vector(path, x) -> None:
    """One value per line with 17 significant digits (mmio.py:218-223)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64).ravel())
    _lib.check(_lib.load().pars3_vector_write(_path(path), x.size, _lib.ptr(x), 0), "write_vector")


# ------------------------------------------------------------ permutations
def write_permutation(path, perm) -> None:
    """Count line, then ``old new`` pairs (reorder.py:300-305)."""
    fw = np.ascontiguousarray(perm.forward, dtype=np.int64)
    _lib.check(_lib.load().pars3_permutation_write(_path(path), fw.size, _lib.ptr(fw), 0),
               "write_permutation")


def read_permutation(path):
    """Read a file written by :func:`write_permutation` (reorder.py:308-333)."""
    from .reorder import Permutation
    L = _lib.load()
    n = ctypes.c_int64()
    rc = L.pars3_permutation_read(_path(path), ctypes.byref(n), None, None, 0)
    if rc == _lib.PARS3_OK:
        old = np.empty(n.value, dtype=np.int64)
        new = np.empty(n.value, dtype=np.int64)
        rc = L.pars3_permutation_read(_path(path), ctypes.byref(n), _lib.ptr(old), _lib.ptr(new), 0)
        if rc == _lib.PARS3_OK:
            return Permutation(_checked_forward(n.value, old, new))
    if rc != _lib.PARS3_SLOW_PATH:
        _lib.check(rc, "read_permutation")
    return _exact_read_permutation(path)


def _checked_forward(n, old, new):
    """forward[old] = new with the reference's first-offending-pair errors:
    an out-of-range source, then a source listed twice, in file order."""
    bad_range = np.flatnonzero((old < 0) | (old >= n))
    first_bad = int(bad_range[0]) if bad_range.size else n
    ok = old[:first_bad]
    order = np.argsort(ok, kind="stable")
    srt = ok[order]
    dup_pos = order[1:][srt[1:] == srt[:-1]]  # later occurrences of a repeated source
    first_dup = int(dup_pos.min()) if dup_pos.size else n
    if first_bad < n and first_bad <= first_dup:
        raise StructuralError(f"source index {int(old[first_bad])} out of range")
    if first_dup < n:
        raise StructuralError(f"source index {int(old[first_dup])} listed twice")
    forward = np.empty(n, dtype=np.int64)
    forward[old] = new
    return forward


def _exact_read_permutation(path):
    from .reorder import Permutation
    with open(path, "r", encoding="ascii") as fh:
        lines = [s for s in (ln.strip() for ln in fh) if s]
    if not lines:
        raise StructuralError("empty permutation file")
    try:
        n = int(lines[0])
    except ValueError:
        raise StructuralError(f"first line must be the index count, got {lines[0]!r}") from None
    if len(lines) != n + 1:
        raise StructuralError(f"expected {n} pairs after the count line, got {len(lines) - 1}")
    forward = np.empty(n, dtype=np.int64)
    seen = np.zeros(n, dtype=bool)
    for s in lines[1:]:
        f = s.split()
        if len(f) != 2:
            raise StructuralError(f"malformed pair {s!r}")
        a, b = int(f[0]), int(f[1])
        if not 0 <= a < n:
            raise StructuralError(f"source index {a} out of range")
        if seen[a]:
            raise StructuralError(f"source index {a} listed twice")
        seen[a] = True
        forward[a] = b
    return Permutation(forward)
