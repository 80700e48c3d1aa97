"""BASELINE configs c2-c4 through the full chain, pinned to the reference.

tests/golden/hashes.json holds the SHA-256 of every array the unmodified
reference chain produced for these configs (make_golden.py; c3/c4 with
--big).  Each config is generated once and checked twice: the CPU oracle's
chain and the product's native chain must both reproduce every hash."""

import numpy as np
import pytest

import paper_2407_17651_b200 as P
from conftest import PLAN_FIELDS, SPLIT_FIELDS, sha


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4"])
def test_config_chain_hashes(cfg, oracle, lib_built, golden_hashes):
    if cfg not in golden_hashes:
        pytest.skip(f"{cfg} hashes not generated")
    from paper_2407_17651_b200 import generators as G
    h = golden_hashes[cfg]
    g = G.make_config(cfg)
    x = G.make_x(g.n, G.CONFIGS[cfg]["seed_x"])
    assert sha(x) == h["x"]
    beta = int(h["beta"])

    # product: native pattern -> RCM -> relabel -> split -> plan
    m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    perm = P.rcm_order(P.pattern_from_sss(m0))
    assert sha(perm.forward) == h["rcm_forward"]
    m = P.permute_sss(m0, perm)
    for k in ("row_ptr", "col_ind", "off_diags", "diags"):
        assert sha(getattr(m, k)) == h[k], k
    assert P.default_beta(m.n, P.compute_bandwidth(m)) == beta
    s = P.split_bands(m, beta)
    for f in SPLIT_FIELDS:
        assert sha(getattr(s, f)) == h[f"b{beta}/{f}"], f
    plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, 8))
    for f in PLAN_FIELDS:
        assert sha(getattr(plan, f)) == h[f"b{beta}/p8/{f}"], f

    # oracle: the same chain restated (C RCM, numpy split/classify), and its
    # serial/pars3 products bit-identical to the reference's
    ip, ix = oracle.pattern_from_sss(g.n, g.row_ptr, g.col_ind)
    fw = oracle.rcm_order(g.n, ip, ix)
    del ip, ix
    assert np.array_equal(fw, perm.forward)
    assert sha(oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)) == h["y_serial"]
    so = oracle.split_bands(g.n, m.row_ptr, m.col_ind, m.off_diags, m.diags, beta)
    po = oracle.classify_conflicts(so, oracle.partition_rows(g.n, 8))
    for f in PLAN_FIELDS:
        assert sha(po[f]) == h[f"b{beta}/p8/{f}"], f
    assert sha(oracle.spmv_pars3(so, po, x)) == h[f"b{beta}/p8/y_pars3"]


def test_oracle_permute_matches_reference_chain_c2(oracle, golden_hashes):
    """The oracle's own permute restatement (numpy) on c2."""
    from paper_2407_17651_b200 import generators as G
    h = golden_hashes["c2"]
    g = G.make_config("c2")
    ip, ix = oracle.pattern_from_sss(g.n, g.row_ptr, g.col_ind)
    fw = oracle.rcm_order(g.n, ip, ix)
    rp, ci, od, dg = oracle.permute_sss(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags, fw)
    for a, k in ((rp, "row_ptr"), (ci, "col_ind"), (od, "off_diags"), (dg, "diags")):
        assert sha(a) == h[k], k
