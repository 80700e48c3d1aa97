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


def _check_chain_c5(h, perm, m, s, beta):
    assert sha(perm.forward) == h["rcm_forward"]
    for k in ("row_ptr", "col_ind", "off_diags", "diags"):
        assert sha(getattr(m, k)) == h[k], k
    assert beta == int(h["beta"])
    for f in SPLIT_FIELDS:
        assert sha(getattr(s, f)) == h[f"b{beta}/{f}"], f
    for p in (1, 2, 4, 8):
        plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, p))
        for f in PLAN_FIELDS:
            assert sha(getattr(plan, f)) == h[f"b{beta}/p{p}/{f}"], (p, f)


def test_config_chain_hashes_c5(oracle, lib_built, golden_hashes):
    """The headline config c5 (n = 16.7 M, m = 216 M): the reference's own
    rcm_order / SssMatrix / split_bands / classify_conflicts outputs
    (make_golden.py --c5) reproduced bit for bit by the product's native
    host chain and by the oracle's chain (the reference arm's inputs)."""
    if "c5" not in golden_hashes:
        pytest.skip("c5 hashes not generated")
    from paper_2407_17651_b200 import generators as G
    h = golden_hashes["c5"]
    g = G.make_config("c5")
    assert g.n == h["n"] and g.nnz == h["nnz"]
    x = G.make_x(g.n, G.CONFIGS["c5"]["seed_x"])
    assert sha(x) == h["x"]
    del x
    m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    perm = P.rcm_order(P.pattern_from_sss(m0))
    m = P.permute_sss(m0, perm)
    beta = P.default_beta(m.n, P.compute_bandwidth(m))
    assert P.compute_bandwidth(m) == h["bandwidth"]
    s = P.split_bands(m, beta)
    _check_chain_c5(h, perm, m, s, beta)
    del s
    # oracle chain: C RCM, numpy permute / split / classify
    ip, ix = oracle.pattern_from_sss(g.n, g.row_ptr, g.col_ind)
    fw = oracle.rcm_order(g.n, ip, ix)
    del ip, ix
    assert sha(fw) == h["rcm_forward"]
    rp, ci, od, dg = oracle.permute_sss(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags, fw)
    for a, k in ((rp, "row_ptr"), (ci, "col_ind"), (od, "off_diags"), (dg, "diags")):
        assert sha(a) == h[k], k
    so = oracle.split_bands(g.n, rp, ci, od, dg, beta)
    for f in SPLIT_FIELDS:
        assert sha(so[f]) == h[f"b{beta}/{f}"], f
    po = oracle.classify_conflicts(so, oracle.partition_rows(g.n, 8))
    for f in PLAN_FIELDS:
        assert sha(po[f]) == h[f"b{beta}/p8/{f}"], f


@pytest.mark.gpu
def test_gpu_chain_hashes_c5(lib_built, golden_hashes):
    """The GPU preprocessing chain (prepare_gpu: RCM, relabel, bandwidth and
    split on the device) reproduces the reference's c5 hashes; this is the
    chain bench.py times the product on."""
    if "c5" not in golden_hashes:
        pytest.skip("c5 hashes not generated")
    from paper_2407_17651_b200 import generators as G
    from paper_2407_17651_b200.pipeline import prepare_gpu
    h = golden_hashes["c5"]
    g = G.make_config("c5")
    m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    del g
    perm, m, s, bw, plan8 = prepare_gpu(m0, boundaries=P.partition_rows(m0.n, 8))
    assert bw == h["bandwidth"]
    # classify_conflicts on the device-resident split (p = 8), then the host function (every p)
    for f in PLAN_FIELDS:
        assert sha(getattr(plan8, f)) == h[f"b{s.beta}/p8/{f}"], ("gpu classify", f)
    _check_chain_c5(h, perm, m, s, s.beta)
