"""Pin the CPU oracle against the reference's own outputs (golden fixtures).

The oracle (oracle/) is the checker for every GPU parity test, so it is
itself checked here first: bit-exact on integer arrays and -- because it
restates the reference's arithmetic order without FMA contraction -- also
bit-exact on the serial and pars3 products.
"""

import numpy as np
import pytest

from conftest import PLAN_FIELDS, SPLIT_FIELDS, sha


def test_corpus_serial_bit_exact(oracle, golden_corpus):
    for name, g in golden_corpus.items():
        y = oracle.spmv_serial(g.row_ptr, g.col_ind, g.off_diags, g.diags, g.x)
        assert np.array_equal(y, g.y_serial), name


def test_corpus_rcm_bit_exact(oracle, golden_corpus):
    for name, g in golden_corpus.items():
        ip, ix = oracle.pattern_from_sss(g.n, g.row_ptr, g.col_ind)
        # the reference computed RCM on the unpermuted corpus matrix
        assert np.array_equal(oracle.rcm_order(g.n, ip, ix), g.rcm_forward), name


def test_corpus_split_plan_pars3_bit_exact(oracle, golden_corpus):
    for name, g in golden_corpus.items():
        for beta in g.betas:
            s = oracle.split_bands(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags, beta)
            want = g.split(beta)
            for f in SPLIT_FIELDS:
                assert np.array_equal(s[f], want[f]), (name, beta, f)
            for p in g.ps():
                plan = oracle.classify_conflicts(s, oracle.partition_rows(g.n, p))
                for f in PLAN_FIELDS:
                    assert np.array_equal(plan[f], g.plan(beta, p)[f]), (name, beta, p, f)
                y = oracle.spmv_pars3(s, plan, g.x)
                assert np.array_equal(y, g.y_pars3(beta, p)), (name, beta, p)


def test_worked_example_known_answer(oracle, golden_corpus):
    # test_serial.py:14-18 / test_formats.py:135-142 of the reference
    g = golden_corpus["tiny4"]
    assert g.row_ptr.tolist() == [0, 0, 1, 2, 4]
    assert g.col_ind.tolist() == [0, 1, 0, 2]
    assert g.off_diags.tolist() == [2.0, 3.0, 5.0, 1.0]
    y = oracle.spmv_serial(g.row_ptr, g.col_ind, g.off_diags, g.diags, np.ones(4))
    assert y.tolist() == [-7.0, -1.0, 2.0, 6.0]


def test_default_beta_and_partition_known_answers(oracle):
    # test_split.py:76-79, 216-222 of the reference
    assert oracle.partition_rows(10, 4).tolist() == [0, 3, 6, 8, 10]
    assert oracle.partition_rows(30, 4).tolist() == [0, 8, 16, 23, 30]
    assert [oracle.default_beta(*a) for a in ((500, 30), (10000, 30), (10000, 4), (100, 0), (2, 1))] \
        == [8, 10, 4, 1, 1]


def _c1_chain(oracle):
    from paper_2407_17651_b200 import generators as G
    g = G.make_config("c1")
    ip, ix = oracle.pattern_from_sss(g.n, g.row_ptr, g.col_ind)
    fw = oracle.rcm_order(g.n, ip, ix)
    rp, ci, od, dg = oracle.permute_sss(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags, fw)
    return g, fw, rp, ci, od, dg


def test_c1_full_chain_bit_exact(oracle, golden_c1):
    g, fw, rp, ci, od, dg = _c1_chain(oracle)
    z = golden_c1
    assert np.array_equal(fw, z["rcm_forward"])
    for a, k in ((rp, "row_ptr"), (ci, "col_ind"), (od, "off_diags"), (dg, "diags")):
        assert np.array_equal(a, z[k]), k
    assert oracle.compute_bandwidth(g.n, rp, ci) == int(z["bandwidth"])
    beta = oracle.default_beta(g.n, int(z["bandwidth"]))
    assert beta == int(z["beta"])
    x = z["x"]
    assert np.array_equal(oracle.spmv_serial(rp, ci, od, dg, x), z["y_serial"])
    for b in (beta, int(z["bandwidth"])):
        s = oracle.split_bands(g.n, rp, ci, od, dg, b)
        for f in SPLIT_FIELDS:
            assert np.array_equal(s[f], z[f"b{b}/{f}"]), (b, f)
        for p in (1, 2, 4, 8):
            plan = oracle.classify_conflicts(s, oracle.partition_rows(g.n, p))
            for f in PLAN_FIELDS:
                assert np.array_equal(plan[f], z[f"b{b}/p{p}/{f}"]), (b, p, f)
            assert np.array_equal(oracle.spmv_pars3(s, plan, x), z[f"b{b}/p{p}/y_pars3"])
