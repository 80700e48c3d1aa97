"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference measures on SuiteSparse matrices that are not
available here; BASELINE.json instead names five synthetic configurations,
and these generators produce them.  The same arrays feed the reference (for
the golden fixtures), the CPU oracle and the GPU path, so no RNG-version
parity across implementations is needed.

Every generator returns the strictly-lower skyline (SSS) arrays of the
matrix *before* RCM, in canonical order (rows ascending, columns strictly
ascending within a row), exactly what ``coo_to_sss`` (formats.py:413-475)
would produce from the both-triangle triplets:

    (n, row_ptr[int64, n+1], col_ind[int32], off_diags[float64], diags[float64])

Conventions:

* graph configurations get a random symmetric relabel drawn from
  ``default_rng(seed_perm).permutation(n)`` (``new = perm[old]``), except
  c5, which keeps the natural grid order;
* values are drawn in canonical storage order from ``default_rng(seed_val)``
  (``uniform(-1, 1)``; R-MAT uses ``standard_normal``);
* ``x`` is ``default_rng(seed_x).uniform(-1, 1, n)``, matching the reference
  tests' ``rng_vector`` (tests/conftest.py:82-84) and bench.py:150-151.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["LowerSss", "CONFIGS", "make_config", "make_x", "grid5", "stencil7", "stencil27",
           "random_band", "rmat", "lower_to_coo_entries"]


@dataclass
class LowerSss:
    n: int
    row_ptr: np.ndarray
    col_ind: np.ndarray
    off_diags: np.ndarray
    diags: np.ndarray
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.col_ind.size)


def _from_pairs(n, r, c, relabel_seed, val_seed, values="uniform", alpha=0.0, name=""):
    """Undirected pairs (r > c or r < c, no self loops, unique) -> LowerSss."""
    r = np.asarray(r, dtype=np.int64)
    c = np.asarray(c, dtype=np.int64)
    if relabel_seed is not None:
        perm = np.random.default_rng(relabel_seed).permutation(n).astype(np.int64)
        r, c = perm[r], perm[c]
    lo_r = np.maximum(r, c)
    lo_c = np.minimum(r, c)
    del r, c
    key = lo_r * n + lo_c
    del lo_r, lo_c
    key.sort(kind="stable")
    rows = key // n
    cols = (key - rows * n).astype(np.int32)
    del key
    counts = np.bincount(rows, minlength=n)
    del rows
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    rng = np.random.default_rng(val_seed)
    if values == "normal":
        val = rng.standard_normal(cols.size)
    else:
        val = rng.uniform(-1.0, 1.0, cols.size)
    return LowerSss(n, row_ptr, cols, val, np.full(n, float(alpha)), name)


def _sorted_unique(key: np.ndarray) -> np.ndarray:
    """np.unique for large int64 keys via an in-place sort (np.unique's hash
    path is several times slower at 10^8 keys); same result."""
    key.sort()
    if key.size < 2:
        return key
    keep = np.empty(key.size, dtype=bool)
    keep[0] = True
    np.not_equal(key[1:], key[:-1], out=keep[1:])
    return key[keep]


def _grid_pairs(k, dims, stencil):
    """Lower neighbour pairs (i, j) with j < i of a k^dims grid, natural ids."""
    n = k ** dims
    ids = np.arange(n, dtype=np.int64)
    coords = []
    rem = ids
    for _ in range(dims):
        coords.append(rem % k)
        rem = rem // k
    # coords[0] is the fastest axis
    offs = []
    if stencil == "star":
        for ax in range(dims):
            o = [0] * dims
            o[ax] = -1
            offs.append(tuple(o))
    else:  # box: all offsets lexicographically negative
        import itertools
        for o in itertools.product((-1, 0, 1), repeat=dims):
            o = tuple(reversed(o))  # o[0] fastest axis
            delta = sum(o[a] * k ** a for a in range(dims))
            if delta < 0:
                offs.append(o)
    rs, cs = [], []
    for o in offs:
        ok = np.ones(n, dtype=bool)
        for a in range(dims):
            if o[a]:
                t = coords[a] + o[a]
                ok &= (t >= 0) & (t < k)
        delta = sum(o[a] * k ** a for a in range(dims))
        i = ids[ok]
        rs.append(i)
        cs.append(i + delta)
    return n, np.concatenate(rs), np.concatenate(cs)


def grid5(k, seed_perm=None, seed_val=0, alpha=0.0, name="grid5"):
    """2-D 5-point stencil graph on a k x k grid."""
    n, r, c = _grid_pairs(k, 2, "star")
    return _from_pairs(n, r, c, seed_perm, seed_val, alpha=alpha, name=name)


def stencil7(k, seed_perm=None, seed_val=0, alpha=0.0, name="stencil7"):
    """3-D 7-point stencil graph on a k^3 grid."""
    n, r, c = _grid_pairs(k, 3, "star")
    return _from_pairs(n, r, c, seed_perm, seed_val, alpha=alpha, name=name)


def stencil27(k, seed_perm=None, seed_val=0, alpha=0.0, name="stencil27"):
    """3-D 27-point stencil graph on a k^3 grid (non-periodic).

    Without a relabel the lower columns of each row come out ascending
    directly (the 13 negative offsets in ascending id delta), so the arrays
    are built row-major without a global sort; this is what keeps the
    256^3 configuration (216 M entries) cheap to generate."""
    if seed_perm is not None:
        n, r, c = _grid_pairs(k, 3, "box")
        return _from_pairs(n, r, c, seed_perm, seed_val, alpha=alpha, name=name)
    n = k ** 3
    import itertools
    offs = []
    for dz, dy, dx in itertools.product((-1, 0, 1), repeat=3):
        delta = dz * k * k + dy * k + dx
        if delta < 0:
            offs.append((delta, dz, dy, dx))
    offs.sort()
    cols = np.full((n, len(offs)), -1, dtype=np.int32)
    ids = np.arange(n, dtype=np.int64)
    x = ids % k
    y = (ids // k) % k
    z = ids // (k * k)
    del ids
    for j, (delta, dz, dy, dx) in enumerate(offs):
        ok = np.ones(n, dtype=bool)
        for comp, d in ((x, dx), (y, dy), (z, dz)):
            if d < 0:
                ok &= comp > 0
            elif d > 0:
                ok &= comp < k - 1
        idx = np.flatnonzero(ok)
        cols[idx, j] = (idx + delta).astype(np.int32)
    del x, y, z
    valid = cols >= 0
    counts = valid.sum(axis=1)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    col_ind = cols[valid]
    del cols, valid
    val = np.random.default_rng(seed_val).uniform(-1.0, 1.0, col_ind.size)
    return LowerSss(n, row_ptr, col_ind, val, np.full(n, float(alpha)), name)


def random_band(n, half_width=2048, per_row=16, far_frac=0.01, seed_struct=0, seed_perm=None,
                seed_val=0, alpha=0.0, name="random_band"):
    """Random band: per row ``per_row`` distinct lower columns uniform in
    ``[i - half_width, i)`` (clipped at 0), plus ``far_frac`` of that count
    as extra entries uniformly far off-band (``i - j > half_width``)."""
    rng = np.random.default_rng(seed_struct)
    i = np.arange(n, dtype=np.int64)
    width = np.minimum(i, half_width)  # available columns [i-width, i)
    k = per_row
    d = 1 + (rng.random((n, k)) * np.maximum(width, 1)[:, None]).astype(np.int64)
    # resample duplicates within a row until all offsets are distinct
    while True:
        d.sort(axis=1)
        dup = np.zeros_like(d, dtype=bool)
        dup[:, 1:] = d[:, 1:] == d[:, :-1]
        dup &= (width >= k)[:, None]
        nd = int(dup.sum())
        if nd == 0:
            break
        rows_dup = np.nonzero(dup)[0]
        d[dup] = 1 + (rng.random(nd) * width[rows_dup]).astype(np.int64)
    # rows with fewer than k available columns take all of them
    short = width < k
    r_band = np.repeat(i, k)
    c_band = (i[:, None] - d).ravel()
    keep = np.ones(n * k, dtype=bool)
    if short.any():
        keep = np.repeat(~short, k)
        rs = np.concatenate([np.full(w, row) for row, w in zip(i[short], width[short])]) \
            if width[short].sum() else np.zeros(0, np.int64)
        cs = np.concatenate([np.arange(w) for w in width[short]]) \
            if width[short].sum() else np.zeros(0, np.int64)
    else:
        rs = cs = np.zeros(0, np.int64)
    r_band = np.concatenate((r_band[keep], rs))
    c_band = np.concatenate((c_band[keep], cs))
    m_band = r_band.size
    n_far = int(round(far_frac * m_band))
    if n_far and n > half_width + 1:
        fr = rng.integers(half_width + 1, n, size=n_far)
        fc = (rng.random(n_far) * (fr - half_width)).astype(np.int64)
        key = _sorted_unique(fr * n + fc)
        fr, fc = key // n, key % n
        r_band = np.concatenate((r_band, fr))
        c_band = np.concatenate((c_band, fc))
    return _from_pairs(n, r_band, c_band, seed_perm, seed_val, alpha=alpha, name=name)


def rmat(scale, edge_factor=16, abcd=(0.57, 0.19, 0.19, 0.05), seed_struct=0, seed_perm=None,
         seed_val=0, name="rmat"):
    """R-MAT graph (Graph500-style ``edge_factor * 2^scale`` samples),
    symmetrised, self loops and duplicates removed; values N(0, 1)."""
    n = 1 << scale
    e = edge_factor * n
    a, b, c, _ = abcd
    rng = np.random.default_rng(seed_struct)
    src = np.zeros(e, dtype=np.int32)
    dst = np.zeros(e, dtype=np.int32)
    ge_a = np.empty(e, dtype=bool)
    ge_ab = np.empty(e, dtype=bool)
    ge_abc = np.empty(e, dtype=bool)
    for bit in range(scale):
        u = rng.random(e)
        np.greater_equal(u, a, out=ge_a)
        np.greater_equal(u, a + b, out=ge_ab)
        np.greater_equal(u, a + b + c, out=ge_abc)
        del u
        # source bit: quadrant c or d; destination bit: quadrant b or d
        src |= ge_ab.view(np.int8).astype(np.int32) << bit
        np.logical_xor(ge_a, ge_ab, out=ge_a)
        np.logical_or(ge_a, ge_abc, out=ge_a)
        dst |= ge_a.view(np.int8).astype(np.int32) << bit
    src = src.astype(np.int64)
    dst = dst.astype(np.int64)
    keep = src != dst
    src, dst = src[keep], dst[keep]
    lo_r = np.maximum(src, dst)
    lo_c = np.minimum(src, dst)
    del src, dst
    key = _sorted_unique(lo_r * n + lo_c)
    r, cc = key // n, key % n
    return _from_pairs(n, r, cc, seed_perm, seed_val, values="normal", name=name)


# BASELINE.json configs[0..4].  Seeds: (struct, perm, val, x).
CONFIGS = {
    "c1": dict(desc="2D 5-pt 100x100, random relabel, U(-1,1), zero diagonal",
               fn=lambda: grid5(100, seed_perm=11, seed_val=12, name="c1"), seed_x=13),
    "c2": dict(desc="3D 7-pt 64^3, random relabel, U(-1,1), zero diagonal",
               fn=lambda: stencil7(64, seed_perm=21, seed_val=22, name="c2"), seed_x=23),
    "c3": dict(desc="random band n=2^22, half-width 2048, 16/row + 1% far, random relabel",
               fn=lambda: random_band(1 << 22, 2048, 16, 0.01, seed_struct=30, seed_perm=31,
                                      seed_val=32, name="c3"), seed_x=33),
    "c4": dict(desc="R-MAT 2^22, edge factor 16, (0.57,0.19,0.19,0.05), N(0,1), random relabel",
               fn=lambda: rmat(22, 16, seed_struct=40, seed_perm=41, seed_val=42, name="c4"),
               seed_x=43),
    "c5": dict(desc="0.5*I + 27-pt 256^3 (natural order), U(-1,1)",
               fn=lambda: stencil27(256, seed_val=52, alpha=0.5, name="c5"), seed_x=53),
}


def make_config(name: str) -> LowerSss:
    return CONFIGS[name]["fn"]()


def make_x(n: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def lower_to_coo_entries(m: LowerSss):
    """Both-triangle triplets (plus the diagonal when non-zero) of a LowerSss,
    i.e. what the reference's CooMatrix holds for the same matrix."""
    rows = np.repeat(np.arange(m.n, dtype=np.int64), np.diff(m.row_ptr))
    cols = m.col_ind.astype(np.int64)
    r = [rows, cols]
    c = [cols, rows]
    v = [m.off_diags, -m.off_diags]
    if np.any(m.diags != 0.0):
        d = np.arange(m.n, dtype=np.int64)
        r.append(d)
        c.append(d)
        v.append(m.diags)
    return np.concatenate(r), np.concatenate(c), np.concatenate(v)
