"""The host plan builders (csrc/tileplan.cpp, csrc/fullcsr.cpp) without a
GPU: the tile plan and the row-major plan decoded back into (row, column,
value) triples must be exactly the split's entries, and their structural
invariants must hold (rows owned once, windows within the local space, slice
records well formed, lanes and spans consistent)."""

import ctypes

import numpy as np
import pytest

import paper_2407_17651_b200 as P
from paper_2407_17651_b200 import _lib
from paper_2407_17651_b200 import generators as G

SINK2 = 3201  # Layout<2>::kSink (tiles.cu): padding lanes and entries of two-word plans


def _split(g, beta=None):
    m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    m = P.permute_sss(m0, P.rcm_order(P.pattern_from_sss(m0)))
    b = P.default_beta(m.n, P.compute_bandwidth(m)) if beta is None else beta
    return m, P.split_bands(m, b)


def _view(s):
    keep = dict(diag=np.ascontiguousarray(s.diag, np.float64), mp=np.ascontiguousarray(s.mid_ptr, np.int64),
                mc=np.ascontiguousarray(s.mid_col, np.int32), mv=np.ascontiguousarray(s.mid_val, np.float64),
                orow=np.ascontiguousarray(s.outer_row, np.int32), oc=np.ascontiguousarray(s.outer_col, np.int32),
                ov=np.ascontiguousarray(s.outer_val, np.float64))
    v = _lib.SplitView(s.n, s.beta, _lib.ptr(keep["diag"]), _lib.ptr(keep["mp"]), _lib.ptr(keep["mc"]),
                       _lib.ptr(keep["mv"]), int(keep["oc"].size), _lib.ptr(keep["orow"]), _lib.ptr(keep["oc"]),
                       _lib.ptr(keep["ov"]))
    return v, keep


def _entries(s):
    rows = np.concatenate([s.outer_row.astype(np.int64), np.repeat(np.arange(s.n), np.diff(s.mid_ptr))])
    cols = np.concatenate([s.outer_col.astype(np.int64), s.mid_col.astype(np.int64)])
    vals = np.concatenate([s.outer_val, s.mid_val])
    o = np.lexsort((cols, rows))
    return rows[o], cols[o], vals[o]


def host_plan(s, words=2, options=()):
    L = _lib.load()
    v, keep = _view(s)
    opts = _lib.PlanOptions(*(tuple(options) + (0, 0, 0, -1, 0, 0, 0)[len(options):]))
    sizes = np.zeros(9, dtype=np.int64)
    args = (ctypes.byref(v), ctypes.byref(opts), words, 0, _lib.ptr(sizes))
    _lib.check(L.pars3_tile_plan_arrays(*args, None, None, None, None, None))
    tiles = np.zeros((int(sizes[0]), 12), dtype=np.int32)
    wins = np.zeros((max(1, int(sizes[1])), 4), dtype=np.int32)
    soff = np.zeros(int(sizes[2]) + 1, dtype=np.int64)
    rec = np.zeros(max(1, int(sizes[3])), dtype=np.uint8)
    ucol = np.zeros(max(1, int(sizes[8])), dtype=np.int32)
    _lib.check(L.pars3_tile_plan_arrays(*args, _lib.ptr(tiles), _lib.ptr(wins), _lib.ptr(soff), _lib.ptr(rec),
                                        _lib.ptr(ucol)))
    return sizes, tiles, wins, soff, rec, ucol


def decode(sizes, tiles, wins, soff, rec, ucol, sink):
    """(row, col, val) of every stored entry, from the slice records."""
    R, C, V = [], [], []
    for t in tiles:
        r0, r1, w0, w1, u0, s0, s1, local = (int(x) for x in t[:8])
        if u0 >= 0:
            glob = ucol[u0:u0 + local].astype(np.int64)
        else:
            glob = np.concatenate([np.arange(lo, lo + ln, dtype=np.int64) for lo, ln, _, _ in wins[w0:w1]]
                                  or [np.zeros(0, np.int64)])
            offs = [int(w[2]) for w in wins[w0:w1]]
            assert offs == list(np.cumsum([0] + [int(w[1]) for w in wins[w0:w1]])[:-1])
            assert w1 - w0 <= 8
        assert glob.size == local and np.all(np.diff(glob) > 0)
        for sl in range(s0, s1):
            a, b = int(soff[sl]) * 16, int(soff[sl + 1]) * 16
            ns = (b - a - 64) // 320
            assert 1 <= ns <= 8 and 64 + 320 * ns == b - a
            rowl = rec[a:a + 64].view(np.uint16).astype(np.int64)
            val = rec[a + 64:a + 64 + ns * 256].view(np.float64).reshape(ns, 32)
            lidx = rec[a + 64 + ns * 256:b].view(np.uint16).astype(np.int64).reshape(ns, 32)
            for lane in range(32):
                if rowl[lane] == sink:
                    assert np.all(lidx[:, lane] == sink) and np.all(val[:, lane] == 0.0)
                    continue
                row = glob[rowl[lane]]
                live = lidx[:, lane] != sink
                assert np.all(val[~live, lane] == 0.0)
                R += [row] * int(live.sum())
                C += list(glob[lidx[live, lane]])
                V += list(val[live, lane])
    R, C, V = np.array(R, np.int64), np.array(C, np.int64), np.array(V)
    o = np.lexsort((C, R))
    return R[o], C[o], V[o]


CASES = [
    ("stencil27", lambda: G.stencil27(9, seed_perm=3, seed_val=4, alpha=0.5), ()),
    ("grid5", lambda: G.grid5(40, seed_perm=7, seed_val=8), ()),
    ("band_far", lambda: G.random_band(4000, 300, 10, 0.02, seed_struct=1, seed_perm=2, seed_val=3), ()),
    ("rmat_hubs", lambda: G.rmat(10, 16, seed_struct=3, seed_perm=4, seed_val=5), ()),
    ("tiny_tiles", lambda: G.stencil27(8, seed_perm=1, seed_val=2), (64, 128, 8, 0)),
    ("narrow_segments", lambda: G.rmat(9, 8, seed_struct=5, seed_perm=6, seed_val=7), (32, 64, 4, 2)),
]


@pytest.mark.parametrize("name,make,options", CASES, ids=[c[0] for c in CASES])
def test_tile_plan_decodes_to_the_split(name, make, options, lib_built):
    m, s = _split(make())
    sizes, tiles, wins, soff, rec, ucol = host_plan(s, 2, options)
    assert int(sizes[4]) == s.mid_col.size + s.outer_col.size
    R, C, V = decode(sizes, tiles, wins, soff, rec, ucol, SINK2)
    r, c, v = _entries(s)
    assert np.array_equal(R, r) and np.array_equal(C, c) and np.array_equal(V, v), name
    # every row is owned by exactly one tile (helper tiles own none), in order
    owned = np.zeros(s.n, dtype=np.int32)
    last = 0
    for t in tiles:
        assert t[0] >= last or t[0] == t[1]
        owned[t[0]:t[1]] += 1
        last = max(last, int(t[1]))
    assert np.all(owned == 1)
    cap = options[1] if len(options) > 1 and options[1] else 3200
    assert int(tiles[:, 7].max()) <= cap
    assert int(sizes[7]) == int((tiles[:, 4] >= 0).sum())


def test_one_window_for_a_fragmented_range(lib_built):
    """A range too fragmented for gap-merged windows whose whole column span fits
    the local space is one dense window, not a column list."""
    n = 3000
    rng = np.random.default_rng(5)
    rows, cols = [], []
    for i in range(40, n):            # every row: 12 scattered columns within 600 of the diagonal
        cs = np.unique(i - 1 - rng.choice(np.arange(0, 600, 11), size=12, replace=False))
        cs = cs[cs >= 0]
        rows += [i] * cs.size
        cols += list(cs)
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, np.array(rows) + 1, 1)
    np.cumsum(rp, out=rp)
    o = np.lexsort((cols, rows))
    m = P.SssMatrix(n, rp, np.array(cols)[o], rng.uniform(-1, 1, len(cols)), np.zeros(n))
    s = P.split_bands(m, n)
    sizes, tiles, wins, soff, rec, ucol = host_plan(s, 2)
    assert int(sizes[7]) == 0 and np.all(tiles[:, 3] - tiles[:, 2] <= 8)
    R, C, V = decode(sizes, tiles, wins, soff, rec, ucol, SINK2)
    r, c, v = _entries(s)
    assert np.array_equal(R, r) and np.array_equal(C, c) and np.array_equal(V, v)


@pytest.mark.parametrize("name", ["rmat", "stencil27", "band_far"])
def test_full_csr_host_is_the_whole_matrix(name, lib_built, oracle):
    """The row-major plan (csrc/fullcsr.cpp): rows ascending in column with the
    diagonal and the negated mirrors; y = (CSR) x equals the oracle's product;
    lane rows, row-start masks and spans consistent with the row pointer."""
    g = {"rmat": lambda: G.rmat(10, 16, seed_struct=7, seed_perm=8, seed_val=9),
         "stencil27": lambda: G.stencil27(8, seed_val=6, alpha=0.5),
         "band_far": lambda: G.random_band(3001, 200, 9, 0.03, seed_struct=1, seed_perm=2, seed_val=3)}[name]()
    m, s = _split(g)
    L = _lib.load()
    v, keep = _view(s)
    sizes = np.zeros(4, dtype=np.int64)
    _lib.check(L.pars3_full_csr_host(ctypes.byref(v), _lib.ptr(sizes), *([None] * 7)))
    nep, ne, nl, nsp = (int(t) for t in sizes)
    col, val = np.zeros(nep, np.int32), np.zeros(nep, np.float64)
    lrow, lflags = np.zeros(nl, np.int32), np.zeros(nl, np.uint32)
    srow, sw0, sw1 = (np.zeros(max(nsp, 1), np.int32) for _ in range(3))
    _lib.check(L.pars3_full_csr_host(ctypes.byref(v), _lib.ptr(sizes), _lib.ptr(col), _lib.ptr(val), _lib.ptr(lrow),
                                     _lib.ptr(lflags), _lib.ptr(srow), _lib.ptr(sw0), _lib.ptr(sw1)))
    m_entries = s.mid_col.size + s.outer_col.size
    assert ne == 2 * m_entries + s.n and nep % 512 == 0 and nl == nep // 16
    # row starts from the masks
    starts = np.zeros(nep + 1, dtype=bool)
    for l in range(nl):
        for k in range(17):
            if (int(lflags[l]) >> k) & 1:
                starts[l * 16 + k] = True
    rp = np.flatnonzero(starts[:ne])
    assert rp.size == s.n and rp[0] == 0
    rp = np.append(rp, ne)
    rows = np.repeat(np.arange(s.n), np.diff(rp))
    for i in (0, s.n // 2, s.n - 1):
        assert np.all(np.diff(col[rp[i]:rp[i + 1]]) > 0)
    assert np.array_equal(lrow, rows[np.minimum(np.arange(nl) * 16, ne - 1)])
    x = G.make_x(s.n, 3)
    y = np.zeros(s.n)
    np.add.at(y, rows, val[:ne] * x[col[:ne]])
    ref = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
    assert oracle.rel_err(y, ref) <= 1e-13
    # spans: exactly the rows that cross a warp of 512 entries
    last = np.append(rp[1:-1] - 1, nep - 1)
    cross = np.flatnonzero(last // 512 > rp[:-1] // 512)
    assert np.array_equal(srow[:nsp], cross)
    assert np.array_equal(sw0[:nsp], rp[cross] // 512) and np.array_equal(sw1[:nsp], last[cross] // 512)
