"""Bitwise repeatability of the product (the reference's guarantee:
parallel.py:107-108 -- fixed summation order -- and its repeated-run test,
tests/test_parallel.py:81-88), at the BASELINE configs' full sizes.

The grid form accumulates every tile's delivery as an exact integer on one
product-wide fixed-point grid, so y does not depend on the order in which
tiles arrive; the fused <y, y> is summed in a fixed order.  Each product is
repeated ten times and compared byte for byte, and checked against the
oracle's serial product once."""

import numpy as np
import pytest

import paper_2407_17651_b200 as P
from conftest import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _repeat(op, xd, reps=10):
    ys, dots = [], []
    for _ in range(reps):
        y, d = op.matvec_dot(xd, None)
        ys.append(y.cpu().numpy().copy())
        dots.append(d.cpu().numpy().copy())
    return ys, dots


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4", "c5"])
def test_repeated_products_bitwise(cfg, oracle):
    import torch

    import bench
    m, s, bw, beta, x = bench.build_problem(cfg)
    plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, 1))
    op = P.prepare(s, plan)
    xd = torch.from_numpy(x).cuda()
    ys, dots = _repeat(op, xd)
    for k in range(1, len(ys)):
        assert np.array_equal(ys[0], ys[k]), (cfg, k, op.stats())
        assert np.array_equal(dots[0], dots[k]), (cfg, k)
    assert op.status() & 1 == 0, "no product may have needed the fp64 redo"
    y_ref = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
    assert rel_err(ys[0], y_ref) <= 1e-12


def test_repeated_products_small_plans(oracle):
    """Window, list, locality and three-word plans at small sizes."""
    import torch
    from paper_2407_17651_b200 import generators as G
    from paper_2407_17651_b200.device import operator_for_sss
    cases = [G.grid5(100, seed_perm=1, seed_val=2), G.stencil27(24, seed_val=6, alpha=0.5),
             G.random_band(60000, 1024, 16, 0.01, seed_struct=11, seed_perm=12, seed_val=13),
             G.rmat(12, 16, seed_struct=3, seed_perm=4, seed_val=5)]
    for g in cases:
        m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
        m = P.permute_sss(m0, P.rcm_order(P.pattern_from_sss(m0)))
        x = G.make_x(m.n, 9)
        op = operator_for_sss(m)
        ys, dots = _repeat(op, torch.from_numpy(x).cuda(), reps=5)
        for k in range(1, len(ys)):
            assert np.array_equal(ys[0], ys[k]), (g.name, op.stats())
            assert np.array_equal(dots[0], dots[k]), g.name
        y_ref = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
        assert rel_err(ys[0], y_ref) <= 1e-12, g.name


def test_scale_bound_follows_x(oracle):
    """The grid's scale comes from the previous product's max |x|: a product
    whose x grows past it is redone in fp64 (still exact), and the next one
    is back on the grid and repeatable."""
    import torch
    from paper_2407_17651_b200 import generators as G
    from paper_2407_17651_b200.device import operator_for_sss
    g = G.stencil27(20, seed_val=6, alpha=0.5)
    m = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    op = operator_for_sss(m)
    x = G.make_x(m.n, 3)
    for factor, redo in ((1.0, False), (1e6, True), (1e6, False), (1e-9, None), (1e-9, False)):
        xs = x * factor
        y = op.matvec(torch.from_numpy(xs).cuda()).cpu().numpy()
        y_ref = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, xs)
        assert np.max(np.abs(y - y_ref)) <= 1e-12 * np.max(np.abs(y_ref)), factor
        st = op.status()
        if redo is not None:
            assert bool(st & 1) == redo, (factor, st)


def test_strict_products_are_pure(oracle):
    """PARS3_PRODUCT_STRICT: the grid scale comes from this x, so A x is a
    pure function of x bit for bit, whatever product ran before (the
    adaptive default is bitwise repeatable for repeated x); the one-call
    entry points (numpy, host tensors) are strict."""
    import torch
    from paper_2407_17651_b200 import generators as G
    from paper_2407_17651_b200.device import operator_for_sss
    g = G.random_band(20000, 500, 8, 0.02, seed_struct=1, seed_perm=2, seed_val=3)
    m = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    op = operator_for_sss(m, options=(0, 0, 0, -1, 0, 16, 0))  # tiles, no locality order
    x1 = torch.from_numpy(G.make_x(m.n, 1)).cuda()
    decay = torch.from_numpy(np.exp(-np.linspace(0, 40, m.n))).cuda()  # scales spanning 2^-58 .. 1
    ya = op.matvec(x1, strict=True).clone()
    for other in (x1 * 1e5, x1 * decay, x1 * 3e-7):
        op.matvec(other)
        yb = op.matvec(x1, strict=True)
        assert torch.equal(ya, yb)
    # the one-call entry point (its own cached plan): strict as well
    y_np = P.spmv_serial(m, x1.cpu().numpy())
    P.spmv_serial(m, (x1 * 1e5).cpu().numpy())
    assert np.array_equal(y_np, P.spmv_serial(m, x1.cpu().numpy()))
    y_ref = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x1.cpu().numpy())
    assert rel_err(y_np, y_ref) <= 1e-12
