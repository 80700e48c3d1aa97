"""The product's native preprocessing (libpars3 host functions) against the
reference's outputs: RCM labels, relabelled skyline, split and plan arrays
must match bit for bit (north star: integer/indexing work is bit-exact)."""

import numpy as np
import pytest

import paper_2407_17651_b200 as P
from conftest import PLAN_FIELDS, SPLIT_FIELDS, sha


def _sss(g):
    return P.SssMatrix(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)


def test_rcm_corpus(lib_built, golden_corpus):
    for name, g in golden_corpus.items():
        m = _sss(g)
        for nt in (1, 4):
            assert np.array_equal(P.rcm_order(P.pattern_from_sss(m), nthreads=nt).forward,
                                  g.rcm_forward), (name, nt)


def test_pattern_from_coo_matches_sss_route(lib_built, golden_corpus):
    for name, g in golden_corpus.items():
        m = _sss(g)
        a = P.pattern_from_sss(m)
        b = P.pattern_from_coo(P.sss_to_coo(m))
        assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices), name


def test_split_and_plan_corpus(lib_built, golden_corpus):
    for name, g in golden_corpus.items():
        m = _sss(g)
        for beta in g.betas:
            s = P.split_bands(m, beta)
            want = g.split(beta)
            for f in SPLIT_FIELDS:
                assert np.array_equal(getattr(s, f), want[f]), (name, beta, f)
            assert P.merge_splits(s).equals(m), (name, beta)
            for p in g.ps():
                plan, rep = P.classify_conflicts(s, P.partition_rows(m.n, p))
                for f in PLAN_FIELDS:
                    assert np.array_equal(getattr(plan, f), g.plan(beta, p)[f]), (name, beta, p, f)
                assert rep.as_dict() == g.report(beta, p), (name, beta, p)


def test_c1_chain(lib_built, golden_c1):
    from paper_2407_17651_b200 import generators as G
    z = golden_c1
    g = G.make_config("c1")
    m0 = P.SssMatrix(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    perm = P.rcm_order(P.pattern_from_sss(m0))
    assert np.array_equal(perm.forward, z["rcm_forward"])
    m = P.permute_sss(m0, perm)
    for k in ("row_ptr", "col_ind", "off_diags", "diags"):
        assert np.array_equal(getattr(m, k), z[k]), k
    assert P.compute_bandwidth(m) == int(z["bandwidth"])
    for b in (int(z["beta"]), int(z["bandwidth"])):
        s = P.split_bands(m, b)
        for f in SPLIT_FIELDS:
            assert np.array_equal(getattr(s, f), z[f"b{b}/{f}"]), (b, f)
        for p in (1, 2, 4, 8):
            plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, p))
            for f in PLAN_FIELDS:
                assert np.array_equal(getattr(plan, f), z[f"b{b}/p{p}/{f}"]), (b, p, f)


def test_rcm_disconnected_and_isolated(lib_built, oracle):
    """Several components + isolated nodes (D8/D9) against the oracle."""
    from paper_2407_17651_b200 import generators as G
    g = G.rmat(12, 4, seed_struct=7, seed_perm=8, seed_val=9)  # many isolated nodes
    m = P.SssMatrix(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    ip, ix = oracle.pattern_from_sss(g.n, g.row_ptr, g.col_ind)
    assert np.array_equal(P.rcm_order(P.pattern_from_sss(m)).forward,
                          oracle.rcm_order(g.n, ip, ix))


def test_permute_matches_oracle_random_labels(lib_built, oracle):
    from paper_2407_17651_b200 import generators as G
    g = G.random_band(3000, 100, 8, 0.02, seed_struct=1, seed_perm=2, seed_val=3)
    m = P.SssMatrix(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    fw = np.random.default_rng(5).permutation(g.n)
    out = P.permute_sss(m, P.Permutation(fw))
    want = oracle.permute_sss(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags, fw)
    for a, b in zip((out.row_ptr, out.col_ind, out.off_diags, out.diags), want):
        assert np.array_equal(a, b)
    # and the result is a valid skyline matrix
    P.SssMatrix(out.n, out.row_ptr, out.col_ind, out.off_diags, out.diags)
