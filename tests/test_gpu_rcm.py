"""GPU reverse Cuthill-McKee (csrc/rcm.cu) against the host-native RCM,
which is pinned bit-exactly to the reference (test_prep_parity.py,
test_config_hashes.py), and against the reference's own labels for the
BASELINE configs c2-c4 (tests/golden/hashes.json)."""

import numpy as np
import pytest

import paper_2407_17651_b200 as P
from conftest import sha

pytestmark = pytest.mark.gpu


def _sss(g):
    return P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)


def _lower_from_pairs(n, pairs):
    """Strictly-lower SSS of an undirected edge set (values 1)."""
    pairs = {(max(a, b), min(a, b)) for a, b in pairs if a != b}
    rows = np.array(sorted(pairs), dtype=np.int64).reshape(-1, 2)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, rows[:, 0] + 1, 1)
    np.cumsum(rp, out=rp)
    return P.SssMatrix(n, rp, rows[:, 1], np.ones(len(rows)), np.zeros(n))


def _graphs():
    from paper_2407_17651_b200 import generators as G
    rng = np.random.default_rng(5)
    yield "rmat12", _sss(G.rmat(12, 16, seed_struct=3, seed_perm=4, seed_val=5))
    yield "rmat14_ef4", _sss(G.rmat(14, 4, seed_struct=6, seed_perm=7, seed_val=8))
    yield "band", _sss(G.random_band(20000, 300, 8, 0.01, seed_struct=1, seed_perm=2, seed_val=3))
    yield "stencil27", _sss(G.stencil27(20, seed_perm=9, seed_val=6))
    yield "grid5", _sss(G.grid5(60, seed_perm=7, seed_val=8))
    # many small components of different shapes, isolated nodes between them
    pairs, base = [], 0
    for k in range(300):
        size = int(rng.integers(1, 9))
        kind = k % 3
        nodes = base + rng.permutation(size)
        if kind == 0:
            pairs += [(nodes[i], nodes[i + 1]) for i in range(size - 1)]          # path
        elif kind == 1:
            pairs += [(nodes[0], nodes[i]) for i in range(1, size)]              # star
        else:
            pairs += [(nodes[i], nodes[j]) for i in range(size) for j in range(i)]  # clique
        base += size + int(rng.integers(0, 3))
    perm = rng.permutation(base)
    yield "small_components", _lower_from_pairs(base, [(perm[a], perm[b]) for a, b in pairs])
    yield "all_isolated", P.SssMatrix(7, np.zeros(8, np.int64), [], [], np.zeros(7))
    yield "single", P.SssMatrix(1, np.zeros(2, np.int64), [], [], np.zeros(1))
    yield "two_paths_reversed", _lower_from_pairs(10, [(9, 8), (8, 7), (0, 5), (5, 3), (3, 1)])


@pytest.mark.parametrize("name,m", list(_graphs()), ids=lambda v: v if isinstance(v, str) else "")
def test_gpu_rcm_equals_native(name, m, lib_built):
    pat = P.pattern_from_sss(m)
    want = P.rcm_order(pat).forward
    assert np.array_equal(P.rcm_order(pat, device="cuda").forward, want), name
    assert np.array_equal(P.rcm_order_sss(m).forward, want), name


def test_gpu_rcm_empty(lib_built):
    m = P.SssMatrix(0, np.zeros(1, np.int64), [], [], np.zeros(0))
    assert P.rcm_order_sss(m).n == 0


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4"])
def test_gpu_rcm_reference_labels(cfg, golden_hashes, lib_built):
    from paper_2407_17651_b200 import generators as G
    g = G.make_config(cfg)
    assert sha(P.rcm_order_sss(_sss(g)).forward) == golden_hashes[cfg]["rcm_forward"]


@pytest.mark.parametrize("name,m", [g for g in _graphs() if g[0] in ("rmat12", "band", "stencil27",
                                                                    "small_components", "all_isolated",
                                                                    "single")],
                         ids=lambda v: v if isinstance(v, str) else "")
@pytest.mark.parametrize("beta", [None, 1, 7])
def test_gpu_chain_equals_host_chain(name, m, beta, lib_built):
    """prepare_gpu: RCM -> permute -> bandwidth -> split on the device, every
    array equal to the host chain's."""
    from paper_2407_17651_b200.pipeline import prepare_gpu
    perm = P.rcm_order(P.pattern_from_sss(m))
    mh = P.permute_sss(m, perm)
    bw = P.compute_bandwidth(mh)
    b = P.default_beta(mh.n, bw) if beta is None else beta
    sh = P.split_bands(mh, b)
    pg, mg, sg, bwg = prepare_gpu(m, beta)
    assert np.array_equal(pg.forward, perm.forward) and bwg == bw and sg.beta == b
    assert mg.equals(mh), name
    for f in ("diag", "mid_ptr", "mid_col", "mid_val", "outer_row", "outer_col", "outer_val"):
        assert np.array_equal(getattr(sg, f), getattr(sh, f)), (name, f)


def test_gpu_chain_reference_hashes_c2(golden_hashes, lib_built):
    from conftest import SPLIT_FIELDS
    from paper_2407_17651_b200 import generators as G
    from paper_2407_17651_b200.pipeline import prepare_gpu
    h = golden_hashes["c2"]
    perm, m, s, bw = prepare_gpu(_sss(G.make_config("c2")))
    assert sha(perm.forward) == h["rcm_forward"]
    for k in ("row_ptr", "col_ind", "off_diags", "diags"):
        assert sha(getattr(m, k)) == h[k], k
    beta = int(h["beta"])
    assert s.beta == beta
    for f in SPLIT_FIELDS:
        assert sha(getattr(s, f)) == h[f"b{beta}/{f}"], f


def test_page_locked_download(lib_built):
    """pipeline._download (page-locked return path of prepare_gpu): every
    dtype the chain returns, empty and multi-chunk tensors, bytes unchanged."""
    import torch

    from paper_2407_17651_b200 import pipeline
    rng = np.random.default_rng(11)
    hs = [rng.integers(-2**40, 2**40, 3_000_001, dtype=np.int64),
          rng.integers(-2**31, 2**31 - 1, 20_000_003, dtype=np.int32),  # > one 64 MB chunk
          rng.uniform(-1, 1, 12_345).astype(np.float64),
          np.empty(0, dtype=np.float64), np.empty(0, dtype=np.int32)]
    ds = [torch.from_numpy(h).cuda() for h in hs]
    outs = pipeline._download(ds, torch)
    for h, o in zip(hs, outs):
        assert o.dtype == h.dtype and o.shape == h.shape
        assert np.array_equal(o, h)
        assert o.flags.writeable and o.flags.c_contiguous


@pytest.mark.parametrize("name,m", [(n, m) for n, m in _graphs()
                                    if n in ("rmat12", "band", "stencil27", "grid5", "small_components",
                                             "single")],
                         ids=lambda v: v if isinstance(v, str) else "")
@pytest.mark.parametrize("p", [1, 2, 3, 8])
def test_gpu_classify_equals_host(name, m, p, lib_built):
    """classify_conflicts on the device (split.py:303-361): every PartitionPlan
    array and the ConflictReport equal to the host-native function's, both
    standalone and inside prepare_gpu (device-resident split)."""
    from conftest import PLAN_FIELDS
    from paper_2407_17651_b200.pipeline import classify_conflicts_gpu, prepare_gpu
    perm = P.rcm_order(P.pattern_from_sss(m))
    mh = P.permute_sss(m, perm)
    if p > mh.n:
        pytest.skip("more workers than rows")
    for beta in (None, 3):
        b = P.default_beta(mh.n, P.compute_bandwidth(mh)) if beta is None else beta
        sh = P.split_bands(mh, b)
        bounds = P.partition_rows(mh.n, p)
        want, wrep = P.classify_conflicts(sh, bounds)
        got, grep = classify_conflicts_gpu(sh, bounds)
        chain = prepare_gpu(m, beta, boundaries=bounds)[4]
        for f in PLAN_FIELDS:
            assert np.array_equal(getattr(got, f), getattr(want, f)), (name, p, f)
            assert np.array_equal(getattr(chain, f), getattr(want, f)), (name, p, f, "chain")
        assert grep == wrep


def test_gpu_classify_errors(lib_built):
    from paper_2407_17651_b200.pipeline import classify_conflicts_gpu
    from paper_2407_17651_b200 import generators as G
    m = _sss(G.grid5(12, seed_perm=1, seed_val=2))
    s = P.split_bands(m, 5)
    for bad in ([0, 10], [1, m.n], [0, 5, 5, m.n], [0, 1, m.n]):
        with pytest.raises(P.StructuralError):
            classify_conflicts_gpu(s, bad)
