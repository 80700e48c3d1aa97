"""The internal locality order of the device plan (csrc/locality.cpp), host
side: a valid, deterministic permutation that recovers a band scrambled by
random long-range entries (BASELINE c3's structure).  The GPU side (the plan
gathering x / y through it) is tests/test_gpu_parity.py::test_locality_order."""

import numpy as np

import paper_2407_17651_b200 as P
from paper_2407_17651_b200 import generators as G


def _rcm_split(g):
    m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    m = P.permute_sss(m0, P.rcm_order(P.pattern_from_sss(m0)))
    return m, P.split_bands(m, P.default_beta(m.n, P.compute_bandwidth(m)))


def _near(m, fw, w):
    r = np.repeat(np.arange(m.n), np.diff(m.row_ptr))
    return float(np.mean(np.abs(fw[r] - fw[m.col_ind]) <= w))


def test_locality_order_recovers_band():
    g = G.random_band(100000, 1024, 16, 0.01, seed_struct=21, seed_perm=22, seed_val=23)
    m, s = _rcm_split(g)
    perm, dropped = P.locality_order(s)
    fw = perm.forward
    assert np.array_equal(np.sort(fw), np.arange(m.n))
    # the filter removes (at least) the far entries: 1 % of 1.6 M, both directions
    assert dropped >= 2 * 0.8 * 0.01 * m.nnz_offdiag
    ident = np.arange(m.n)
    before, after = _near(m, ident, 2048), _near(m, fw, 2048)
    assert after >= 0.9 and after > 2 * before, (before, after)
    perm2, dropped2 = P.locality_order(s)          # deterministic
    assert np.array_equal(perm2.forward, fw) and dropped2 == dropped


def test_locality_order_keeps_structured_and_small():
    # a 27-point stencil keeps every edge (each one closes many short cycles)
    g = G.stencil27(10, seed_perm=3, seed_val=4)
    m, s = _rcm_split(g)
    perm, dropped = P.locality_order(s)
    assert dropped == 0
    assert np.array_equal(np.sort(perm.forward), np.arange(m.n))
    # tiny and empty matrices
    for n in (0, 1, 2):
        m = P.SssMatrix(n, np.zeros(n + 1, np.int64), np.zeros(0, np.int64), np.zeros(0),
                        np.zeros(n))
        perm, dropped = P.locality_order(P.split_bands(m, 1))
        assert perm.forward.tolist() == list(range(n)) and dropped == 0
