"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's golden outputs.

Contract (north star, SPEC.md D14, reference test_acceptance.py:101-130):
``||y - y_ref||_inf / max(1, ||y_ref||_inf) <= 1e-12`` with ``y_ref`` the
reference's serial SSS product.
"""

import numpy as np
import pytest

import paper_2407_17651_b200 as P
from conftest import mixed_tol, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2407_17651_b200 import _lib
    _lib.load()


def _sss(g):
    return P.SssMatrix(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)


def test_worked_example_exact(golden_corpus):
    g = golden_corpus["tiny4"]
    m = _sss(g)
    s = P.split_bands(m, 2)
    plan, _ = P.classify_conflicts(s, P.partition_rows(4, 2))
    y = P.spmv_pars3(s, plan, np.ones(4))
    assert y.tolist() == [-7.0, -1.0, 2.0, 6.0]
    assert P.spmv_serial(m, np.ones(4)).tolist() == [-7.0, -1.0, 2.0, 6.0]


def test_corpus_all_betas_and_workers(golden_corpus):
    for name, g in golden_corpus.items():
        m = _sss(g)
        for beta in g.betas:
            s = P.split_bands(m, beta)
            for p in g.ps():
                plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, p))
                y = P.spmv_pars3(s, plan, g.x)
                assert np.max(np.abs(y - g.y_serial), initial=0.0) <= mixed_tol(g.y_serial, TOL), \
                    (name, beta, p)
                # and against the reference's own pars3 output
                assert rel_err(y, g.y_pars3(beta, p)) <= TOL, (name, beta, p)


def test_spmv_serial_and_atomic_corpus(golden_corpus):
    for name, g in golden_corpus.items():
        m = _sss(g)
        assert rel_err(P.spmv_serial(m, g.x), g.y_serial) <= TOL, name
        assert rel_err(P.spmv_atomic(m, g.x, 4), g.y_serial) <= TOL, name
        assert rel_err(P.spmv_serial(m, g.x), g.y_dense) <= 1e-13 * 10, name


def test_c1_against_golden(golden_c1):
    z = golden_c1
    m = P.SssMatrix(int(z["n"]), z["row_ptr"], z["col_ind"], z["off_diags"], z["diags"])
    for b in (int(z["beta"]), int(z["bandwidth"])):
        s = P.split_bands(m, b)
        for p in (1, 2, 4, 8):
            plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, p))
            assert rel_err(P.spmv_pars3(s, plan, z["x"]), z["y_serial"]) <= TOL, (b, p)


def test_torch_in_torch_out(golden_corpus):
    import torch
    g = golden_corpus["gen500"]
    m = _sss(g)
    s = P.split_bands(m, 8)
    plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, 4))
    xd = torch.from_numpy(g.x).cuda()
    y = P.spmv_pars3(s, plan, xd)
    assert isinstance(y, torch.Tensor) and y.is_cuda
    assert rel_err(y.cpu().numpy(), g.y_serial) <= TOL


def test_errors_match_reference(golden_corpus):
    g = golden_corpus["tiny4"]
    m = _sss(g)
    s2, s3 = P.split_bands(m, 2), P.split_bands(m, 3)
    plan, _ = P.classify_conflicts(s2, P.partition_rows(4, 2))
    with pytest.raises(ValueError):
        P.spmv_pars3(s3, plan, np.ones(4))
    with pytest.raises(ValueError):
        P.spmv_pars3(s2, plan, np.ones(4), p=3)
    with pytest.raises(ValueError):
        P.spmv_pars3(s2, plan, np.ones(5))
    with pytest.raises(ValueError):
        P.spmv_atomic(m, np.ones(4), 0)


def _pipeline(g, beta=None, p=1):
    m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    m = P.permute_sss(m0, P.rcm_order(P.pattern_from_sss(m0)))
    if beta is None:
        beta = P.default_beta(m.n, P.compute_bandwidth(m))
    s = P.split_bands(m, beta)
    plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, p))
    return m, s, plan


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4", "c5"])
def test_baseline_configs_full_size(cfg, oracle):
    """Every BASELINE configuration at full size against the oracle's serial
    product (itself pinned to the reference, test_oracle_golden.py)."""
    from paper_2407_17651_b200 import generators as G
    g = G.make_config(cfg)
    m, s, plan = _pipeline(g, p=8)
    x = G.make_x(m.n, G.CONFIGS[cfg]["seed_x"])
    y_ref = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
    y = P.spmv_pars3(s, plan, x)
    assert rel_err(y, y_ref) <= TOL, cfg


def test_skew_identity_large():
    """x . (S x) = 0 for strict skew S (reference test_acceptance.py:133-160)."""
    from paper_2407_17651_b200 import generators as G
    g = G.stencil27(48, seed_val=3)
    m, s, plan = _pipeline(g)
    x = G.make_x(m.n, 4)
    y = P.spmv_pars3(s, plan, x)
    assert abs(float(x @ y)) <= 1e-10 * float(x @ x) * float(np.max(np.abs(m.off_diags)))


OPTION_SETS = [
    # (tile_rows, local_slots, seg_max, gap, mode[, flags, max_ctas])
    (0, 0, 0, -1, 0),         # defaults (auto accumulation)
    (0, 0, 0, -1, 1),         # three-word fixed point forced
    (0, 0, 0, -1, 2),         # fp64 shared accumulators forced
    (0, 0, 0, -1, 3),         # two-word fixed point forced (refused for hub-heavy plans)
    (64, 128, 8, 0, 1),       # tiny tiles: splits, list-mode tiles, hub chunks
    (64, 128, 8, 0, 2),
    (64, 128, 8, 0, 3),
    (32, 64, 4, 2, 1),        # smallest local space: every wide row is chunked
    (4096, 65535, 64, 64, 1),   # clamped to the shared-memory budget
    (0, 0, 0, -1, 0, 0, 37),  # persistent grid capped at 37 CTAs
]


@pytest.mark.parametrize("opts", OPTION_SETS)
def test_tile_plan_options(opts, oracle):
    """The windowed tile plan under extreme options (tile splits, hub-row
    chunking into helper tiles, many tiny windows, every accumulation mode)
    against the oracle."""
    from paper_2407_17651_b200 import generators as G
    from paper_2407_17651_b200.device import operator_for_sss
    import torch
    cases = [G.rmat(12, 16, seed_struct=3, seed_perm=4, seed_val=5),        # hubs + isolated
             G.random_band(5000, 300, 12, 0.02, seed_struct=1, seed_perm=2, seed_val=3),
             G.stencil27(14, seed_val=6, alpha=0.5), G.grid5(40, seed_perm=7, seed_val=8)]
    for g in cases:
        m = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
        x = G.make_x(m.n, 9)
        y_ref = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
        try:
            op = operator_for_sss(m, options=opts)
        except ValueError as e:  # two words cannot hold a hub column's terms
            assert opts[4] == 3 and "two-word" in str(e), (g.name, opts, e)
            continue
        y = op.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
        assert rel_err(y, y_ref) <= TOL, (g.name, opts, op.stats())
        for _ in range(3):  # repeated launches reuse the plan
            y2 = op.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
            assert rel_err(y2, y_ref) <= TOL


def test_accumulating_plans_and_skip_empty(oracle):
    """Two partial plans (rows split by parity) accumulate into one y
    (pars3_plan_spmv_acc); the diagonal lives in the first, the second skips
    its empty rows (PARS3_PLAN_SKIP_EMPTY)."""
    import torch
    from paper_2407_17651_b200 import generators as G
    from paper_2407_17651_b200.device import Pars3Operator
    g = G.stencil27(16, seed_val=2, alpha=0.5)
    m = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    rows = np.repeat(np.arange(m.n), np.diff(m.row_ptr))
    x = G.make_x(m.n, 3)
    y_ref = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
    e = np.zeros(0, np.int32)
    ops = []
    for parity, diag, flags in ((0, m.diags, 0), (1, np.zeros(m.n), 1)):
        keep_row = (np.arange(m.n) % 2) == parity
        keep = keep_row[rows]
        rp = np.zeros(m.n + 1, dtype=np.int64)
        np.cumsum(np.where(keep_row, np.diff(m.row_ptr), 0), out=rp[1:])
        ops.append(Pars3Operator(m.n, m.n, diag, rp, m.col_ind[keep], m.off_diags[keep], e, e,
                                 np.zeros(0), options=(0, 0, 0, -1, 0, flags, 0)))
    xd = torch.from_numpy(x).cuda()
    y = torch.full((m.n,), 7.0, dtype=torch.float64, device="cuda")
    ops[0].matvec(xd, y)                     # overwrites y
    ops[1].matvec(xd, y, accumulate=True)    # adds
    assert rel_err(y.cpu().numpy(), y_ref) <= TOL


def test_spmv_dot(oracle):
    import torch
    from paper_2407_17651_b200 import generators as G
    g = G.stencil27(20, seed_val=1, alpha=0.5)
    m, s, plan = _pipeline(g)
    op = P.prepare(s, plan)
    x = torch.from_numpy(G.make_x(m.n, 2)).cuda()
    y, dot = op.matvec_dot(x, None)
    yh = y.cpu().numpy()
    assert abs(float(dot.item()) - float(yh @ yh)) <= 1e-12 * float(yh @ yh)


@pytest.mark.parametrize("overlap", [False, True])
@pytest.mark.parametrize("p", [2, 3, 8])
def test_multirank_protocol_on_one_gpu(p, overlap, oracle):
    """The p-rank sharding with the GPU tile kernel as each rank's local
    product, exchanges emulated in-process (one GPU is available)."""
    import torch
    from paper_2407_17651_b200 import generators as G
    from paper_2407_17651_b200.device import Pars3Operator
    from paper_2407_17651_b200.distributed import emulate_ranks
    for g, beta in ((G.stencil27(40, seed_val=4, alpha=0.5), None),
                    (G.random_band(40000, 300, 8, 0.01, seed_struct=1, seed_perm=2, seed_val=3), 16)):
        m, s, plan = _pipeline(g, beta=beta, p=p)
        x = G.make_x(m.n, 11)

        def make_local(sh, boundary):
            e = np.zeros(0, np.int32)
            # boundary parts skip their empty rows (flags = PARS3_PLAN_SKIP_EMPTY)
            op = Pars3Operator(sh.n_ext, max(1, sh.n_ext), sh.diags, sh.row_ptr, sh.col_ind,
                               sh.off_diags, e, e, np.zeros(0),
                               options=(0, 0, 0, -1, 0, 1 if boundary else 0, 0))
            return lambda xe: op.matvec(xe)

        y = emulate_ranks(s, plan, torch.from_numpy(x).cuda(), make_local,
                          overlap=overlap).cpu().numpy()
        y_ref = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
        assert rel_err(y, y_ref) <= TOL, (g.name, p)


def test_host_pipeline_non_blocking(oracle):
    """Pinned host vectors through spmv_pars3(non_blocking=True): five calls
    in flight on the copy pipeline (double-buffered device vectors), each
    result checked after one synchronize; then a blocking call."""
    import torch
    from paper_2407_17651_b200 import generators as G
    g = G.stencil27(24, seed_val=5, alpha=0.5)
    m, s, plan = _pipeline(g)
    xs = [torch.from_numpy(G.make_x(m.n, 20 + k)).pin_memory() for k in range(5)]
    outs = [torch.empty(m.n, dtype=torch.float64).pin_memory() for _ in range(5)]
    for x, o in zip(xs, outs):
        P.spmv_pars3(s, plan, x, out=o, non_blocking=True)
    torch.cuda.synchronize()
    for x, o in zip(xs, outs):
        y_ref = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x.numpy())
        assert rel_err(o.numpy(), y_ref) <= TOL
    y = P.spmv_pars3(s, plan, xs[0])  # blocking; the grid product is bitwise repeatable
    assert not y.is_cuda and np.array_equal(y.numpy(), outs[0].numpy())


def _ieee_close(y, y_ref, name):
    """IEEE agreement: the same nan / inf pattern and infinities, finite
    entries within 1e-12 * max(1, ||y_ref||_inf) (or relative for tiny y)."""
    fin = np.isfinite(y_ref)
    assert np.array_equal(np.isnan(y), np.isnan(y_ref)), name
    assert np.array_equal(np.isinf(y), np.isinf(y_ref)), name
    assert np.array_equal(y[np.isinf(y)], y_ref[np.isinf(y_ref)]), name
    if not fin.any():
        return
    scale = max(np.max(np.abs(y_ref[fin])), np.finfo(float).tiny)
    err = np.max(np.abs(y[fin] - y_ref[fin]))
    assert err <= 1e-12 * max(1.0, scale) if scale >= 1 else err <= 1e-12 * scale, (name, err, scale)


def _entry_points(s, plan, m):
    """Every product entry point: y for a host numpy x."""
    import torch

    def pars3_numpy(x):
        return P.spmv_pars3(s, plan, x)

    def pars3_cuda(x):
        return P.spmv_pars3(s, plan, torch.from_numpy(x).cuda()).cpu().numpy()

    def serial_cuda(x):
        return P.spmv_serial(m, torch.from_numpy(x).cuda()).cpu().numpy()

    def matvec_dot(x):
        op = P.prepare(s, plan)
        y, dot = op.matvec_dot(torch.from_numpy(x).cuda(), None)
        yh = y.cpu().numpy()
        with np.errstate(all="ignore"):
            ref = float(yh @ yh)
        d = float(dot.item())
        assert (np.isnan(d) and np.isnan(ref)) or d == ref or abs(d - ref) <= 1e-12 * abs(ref)
        return yh

    def accumulate(x):
        op = P.prepare(s, plan)
        y = torch.zeros(m.n, dtype=torch.float64, device="cuda")
        op.matvec(torch.from_numpy(x).cuda(), y, accumulate=True)
        return y.cpu().numpy()

    def host_pipeline(x):
        out = torch.empty(m.n, dtype=torch.float64).pin_memory()
        P.spmv_pars3(s, plan, torch.from_numpy(x).pin_memory(), out=out, non_blocking=True)
        torch.cuda.synchronize()
        return out.numpy().copy()

    return {"pars3_numpy": pars3_numpy, "pars3_cuda": pars3_cuda, "serial_cuda": serial_cuda,
            "matvec_dot": matvec_dot, "accumulate": accumulate, "host_pipeline": host_pipeline}


@pytest.mark.parametrize("entry", ["pars3_numpy", "pars3_cuda", "serial_cuda", "matvec_dot",
                                   "accumulate", "host_pipeline"])
def test_nonfinite_and_extreme_inputs(entry, oracle):
    """x with inf / nan / subnormal / huge / tiny entries through every entry
    point returns the IEEE result of the reference's arithmetic without any
    host-side check (the grid product raises a device flag and k_finish
    redoes it with fp64 accumulators; the RED form re-streams single tiles)."""
    import warnings

    from paper_2407_17651_b200 import generators as G
    g = G.stencil27(12, seed_val=3, alpha=0.5)
    m, s, plan = _pipeline(g)
    base = G.make_x(m.n, 5)
    cases = {}
    x = base.copy(); x[7] = np.inf; cases["inf"] = x
    x = base.copy(); x[100] = np.nan; cases["nan"] = x
    x = base.copy(); x[::3] *= 1e-310; cases["subnormal"] = x
    x = base.copy() * 1e290; cases["huge"] = x
    x = base.copy() * 1e-290; cases["tiny"] = x
    x = base.copy(); x[3] = -np.inf; x[50] = np.inf; cases["inf_both"] = x
    fn = _entry_points(s, plan, m)[entry]
    for name, x in list(cases.items()) + [("base", base)]:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            y_ref = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
            y = fn(x)
        _ieee_close(y, y_ref, (entry, name))
    # extreme matrix values: fp64 accumulators at plan creation
    big = P.SssMatrix(m.n, m.row_ptr, m.col_ind, m.off_diags * 1e295, m.diags)
    sb = P.split_bands(big, s.beta)
    pb, _ = P.classify_conflicts(sb, P.partition_rows(m.n, 2))
    y = _entry_points(sb, pb, big)[entry](base)
    y_ref = oracle.spmv_serial(big.row_ptr, big.col_ind, big.off_diags, big.diags, base)
    assert np.max(np.abs(y - y_ref)) <= 1e-12 * np.max(np.abs(y_ref))
    assert P.prepare(sb, pb).stats()["accum_words"] == 0


@pytest.mark.parametrize("entry", ["pars3_cuda", "matvec_dot", "accumulate"])
def test_value_spread_correlated_x(entry, oracle):
    """a tile holding v = 1e10 met only by x ~ 1e-10 next
    to v ~ 1 met by x ~ 1 must not round every term to the unit its largest
    |v| * |x| bound implies.  Values spanning 1e-10 .. 1e10 with x ~ 1/|v|
    of the rows: the per-tile guard / the grid's accuracy check send such
    products to fp64 accumulators; the result meets the 1e-12 contract."""
    from paper_2407_17651_b200 import generators as G
    g = G.stencil27(14, seed_val=8, alpha=0.5)
    m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    rng = np.random.default_rng(4)
    rows = np.repeat(np.arange(m0.n), np.diff(m0.row_ptr))
    scale_row = 10.0 ** rng.uniform(-10, 10, m0.n)
    vals = m0.off_diags * scale_row[rows]
    m1 = P.SssMatrix._trusted(m0.n, m0.row_ptr, m0.col_ind, vals, m0.diags)
    m = P.permute_sss(m1, P.rcm_order(P.pattern_from_sss(m1)))
    beta = P.default_beta(m.n, P.compute_bandwidth(m))
    s = P.split_bands(m, beta)
    plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, 1))
    # x ~ 1 / (the row's scale): large values meet small x
    perm = P.rcm_order(P.pattern_from_sss(m1))
    xs = np.empty(m.n)
    xs[perm.forward] = 1.0 / scale_row
    x = xs * G.make_x(m.n, 6)
    y_ref = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
    y = _entry_points(s, plan, m)[entry](x)
    assert rel_err(y, y_ref) <= TOL, (entry, rel_err(y, y_ref))
    # the advisor's example, directly: one tile, v = 1e10 met by x = 3e-10 on
    # both sides, v = 0.7 met by x = 0.9
    e = np.zeros(0, np.int32)
    from paper_2407_17651_b200.device import Pars3Operator
    import torch
    rp = np.array([0, 0, 1, 1, 2], dtype=np.int64)
    ci = np.array([0, 2], dtype=np.int32)
    ov = np.array([1e10, 0.7])
    op = Pars3Operator(4, 4, np.zeros(4), rp, ci, ov, e, e, np.zeros(0))
    x3 = np.array([3e-10, 3e-10, 0.9, 0.9])
    y3 = op.matvec(torch.from_numpy(x3).cuda()).cpu().numpy()
    mm = P.SssMatrix(4, rp, ci, ov, np.zeros(4))
    y3_ref = oracle.spmv_serial(mm.row_ptr, mm.col_ind, mm.off_diags, mm.diags, x3)
    assert rel_err(y3, y3_ref) <= TOL, (y3, y3_ref)


@pytest.mark.parametrize("flags", [0, 8, 16])
def test_locality_order(flags, oracle):
    """The plan's internal locality order (PARS3_PLAN_LOCALITY = 8 forces the
    attempt, NO_LOCALITY = 16 forbids it, 0 = auto): every entry point
    (overwrite, accumulate, fused dot with w = y and w = x) against the
    oracle, in the caller's labels."""
    import torch
    from paper_2407_17651_b200 import generators as G
    from paper_2407_17651_b200.device import operator_for_sss
    cases = [G.random_band(60000, 1024, 16, 0.01, seed_struct=11, seed_perm=12, seed_val=13),
             G.rmat(12, 16, seed_struct=3, seed_perm=4, seed_val=5),
             G.stencil27(14, seed_val=6, alpha=0.5)]
    for g in cases:
        m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
        m = P.permute_sss(m0, P.rcm_order(P.pattern_from_sss(m0)))
        x = G.make_x(m.n, 9)
        y_ref = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
        op = operator_for_sss(m, options=(0, 0, 0, -1, 0, flags, 0))
        st = op.stats()
        if flags == 16:
            assert st["locality_order"] == 0
        if flags == 8 and g.name.startswith("random_band"):
            assert st["locality_order"] == 1, st   # the far entries scramble RCM's layering
        xd = torch.from_numpy(x).cuda()
        y = op.matvec(xd)
        assert rel_err(y.cpu().numpy(), y_ref) <= TOL, (g.name, st)
        y2 = torch.full((m.n,), 0.25, dtype=torch.float64, device="cuda")
        op.matvec(xd, y2, accumulate=True)
        assert rel_err(y2.cpu().numpy() - 0.25, y_ref) <= TOL, (g.name, st)
        y3, dot = op.matvec_dot(xd, None)
        yh = y3.cpu().numpy()
        assert rel_err(yh, y_ref) <= TOL
        assert abs(float(dot.item()) - float(yh @ yh)) <= 1e-12 * float(yh @ yh)
        _, dot2 = op.matvec_dot(xd, xd)
        assert abs(float(dot2.item()) - float(x @ yh)) <= 1e-12 * float(np.abs(x) @ np.abs(yh))
        # grid form: tiles + k_conv + k_finish; + perm in/out with a locality
        # order; row-major form: full CSR + span fix-up + dot (one kernel)
        # (one more for the far part: the long-range entries kept out of the tiles)
        expect = 5 + (1 if st["far_entries"] else 0) if st["locality_order"] else 3 if st["direct"] else 3
        assert op.kernel_count(True) == expect, st
        if flags == 8 and g.name.startswith("random_band"):
            # the far part (k_far_grid / k_far_red): window-mode tiles for the band,
            # bitwise repeatable, IEEE results through the redo as well
            assert st["far_entries"] > 0 and st["list_tiles"] * 10 <= st["tiles"], st
            yb = [op.matvec(xd).cpu().numpy().tobytes() for _ in range(5)]
            assert all(b == yb[0] for b in yb)
            xi = x.copy()
            xi[m.n // 3] = np.inf
            xi[m.n // 2] = 1e300
            ref_i = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, xi)
            got_i = op.matvec(torch.from_numpy(xi).cuda()).cpu().numpy()
            fin = np.isfinite(ref_i)
            assert np.array_equal(np.isnan(got_i), np.isnan(ref_i))
            assert np.array_equal(got_i[~fin & ~np.isnan(ref_i)], ref_i[~fin & ~np.isnan(ref_i)])
            assert rel_err(got_i[fin], ref_i[fin]) <= TOL
            assert op.status() & 1  # that product was redone in fp64
            assert rel_err(op.matvec(xd).cpu().numpy(), y_ref) <= TOL


@pytest.mark.parametrize("flags", [0, 32, 64])
def test_direct_mode(flags, oracle):
    """Direct mode (PARS3_PLAN_DIRECT = 32 forces it, NO_DIRECT = 64 forbids
    it, 0 = auto): the row-major entries with global gathers and reductions,
    every entry point, against the oracle; the shifted diagonal (constant and
    not) included."""
    import torch
    from paper_2407_17651_b200 import generators as G
    from paper_2407_17651_b200.device import operator_for_sss
    cases = [G.rmat(13, 16, seed_struct=7, seed_perm=8, seed_val=9),
             G.random_band(30001, 700, 9, 0.03, seed_struct=1, seed_perm=2, seed_val=3),
             G.stencil27(12, seed_val=6, alpha=0.5), G.grid5(30, seed_perm=7, seed_val=8)]
    for g in cases:
        m = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
        diags = [m.diags, np.linspace(-1.0, 2.0, m.n)]
        for d in diags:
            mm = P.SssMatrix._trusted(m.n, m.row_ptr, m.col_ind, m.off_diags, d)
            x = G.make_x(m.n, 9)
            y_ref = oracle.spmv_serial(mm.row_ptr, mm.col_ind, mm.off_diags, mm.diags, x)
            op = operator_for_sss(mm, options=(0, 0, 0, -1, 0, flags, 0))
            st = op.stats()
            if flags == 32:
                assert st["direct"] == 1 and st["tiles"] == 0, st
            if flags == 64:
                assert st["direct"] == 0
            xd = torch.from_numpy(x).cuda()
            y = op.matvec(xd)
            assert rel_err(y.cpu().numpy(), y_ref) <= TOL, (g.name, st)
            y2 = torch.full((m.n,), -1.5, dtype=torch.float64, device="cuda")
            op.matvec(xd, y2, accumulate=True)
            assert rel_err(y2.cpu().numpy() + 1.5, y_ref) <= TOL, (g.name, st)
            y3, dot = op.matvec_dot(xd, None)
            yh = y3.cpu().numpy()
            assert abs(float(dot.item()) - float(yh @ yh)) <= 1e-12 * float(yh @ yh)
            assert op.status() & 1 == 0  # no product redone
            if st["direct"]:
                assert op.kernel_count(True) == 3  # k_csr, the span fix-up, the dot


def test_product_axpy(oracle):
    """pars3_plan_product_axpy: out = A x + a p + b q and <out, out> (device
    scalars a, b), fused into the finish pass of grid-form plans, one more
    pass for the other forms; the fp64 redo applies it as well."""
    import torch
    from paper_2407_17651_b200 import generators as G
    from paper_2407_17651_b200.device import operator_for_sss
    cases = [(G.stencil27(24, seed_val=6, alpha=0.5), (0, 0, 0, -1, 0, 64, 0)),      # grid form (fused)
             (G.stencil27(20, seed_val=7, alpha=0.5), (0, 0, 0, -1, 0, 32, 0)),      # row-major form
             (G.random_band(30000, 600, 12, 0.01, seed_struct=1, seed_perm=2, seed_val=3), (0, 0, 0, -1, 0, 8, 0))]
    rng = np.random.default_rng(4)
    for g, opts in cases:
        m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
        m = P.permute_sss(m0, P.rcm_order(P.pattern_from_sss(m0)))
        op = operator_for_sss(m, options=opts)
        x, p, q = (rng.uniform(-1, 1, m.n) for _ in range(3))
        coef = torch.tensor([-0.5, 1.75], dtype=torch.float64, device="cuda")
        y_ref = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
        want = y_ref - 0.5 * p + 1.75 * q
        xd, pd, qd = (torch.from_numpy(a).cuda() for a in (x, p, q))
        out = torch.empty_like(xd)
        dot = torch.zeros(1, dtype=torch.float64, device="cuda")
        for strict in (False, True):
            op.matvec_axpy(xd, out, pd, coef[0:1], qd, coef[1:2], dot=dot, strict=strict)
            got = out.cpu().numpy()
            assert rel_err(got, want) <= TOL, (g.name, op.stats())
            assert abs(float(dot.item()) - float(got @ got)) <= 1e-12 * float(got @ got)
        op.matvec_axpy(xd, out, pd, coef[0:1], qd, coef[1:2])      # without the dot
        assert rel_err(out.cpu().numpy(), want) <= TOL
        # the redo (a non-finite x): IEEE result, the update applied once
        xi = x.copy()
        xi[m.n // 2] = np.inf
        ref_i = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, xi) - 0.5 * p + 1.75 * q
        op.matvec_axpy(torch.from_numpy(xi).cuda(), out, pd, coef[0:1], qd, coef[1:2], dot=dot)
        got_i = out.cpu().numpy()
        fin = np.isfinite(ref_i)
        assert np.array_equal(np.isfinite(got_i), fin)
        assert rel_err(got_i[fin], ref_i[fin]) <= TOL
        with pytest.raises(ValueError):
            op.matvec_axpy(xd, out, out, coef[0:1], qd, coef[1:2])   # out aliases p
