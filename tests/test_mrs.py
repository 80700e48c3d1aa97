"""MRS driver (shifted skew-symmetric minimal residual) on the GPU against a
numpy restatement of the same recurrence built on the oracle's serial SpMV."""

import math

import numpy as np
import pytest

import paper_2407_17651_b200 as P
from conftest import rel_err

pytestmark = pytest.mark.gpu


def mrs_reference(spmv, b, alpha, maxiter):
    """The same skew-Lanczos + Givens recurrence in numpy (test oracle)."""
    n = b.size
    x = np.zeros(n)
    beta = float(np.linalg.norm(b))
    v, w = b / beta, np.zeros(n)
    dm1, dm2 = np.zeros(n), np.zeros(n)
    gamma, c1, s1, c2, s2, phi = 0.0, 1.0, 0.0, 1.0, 0.0, beta
    res = [beta]
    for _ in range(maxiter):
        u = spmv(v) - alpha * v + gamma * w
        g = float(np.linalg.norm(u))
        h1 = -gamma
        r0, h1p = s2 * h1, c2 * h1
        r1 = c1 * h1p + s1 * alpha
        h2p = -s1 * h1p + c1 * alpha
        r2 = math.hypot(h2p, g)
        c, s = h2p / r2, g / r2
        tau, phi = c * phi, -s * phi
        d = (v - r0 * dm2 - r1 * dm1) / r2
        x = x + tau * d
        w, v = v, u / g
        dm2, dm1 = dm1, d
        gamma, c2, s2, c1, s1 = g, c1, s1, c, s
        res.append(abs(phi))
    return x, res


@pytest.fixture(scope="module")
def problem():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2407_17651_b200 import generators as G
    g = G.stencil27(20, seed_val=5, alpha=0.5)
    m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    m = P.permute_sss(m0, P.rcm_order(P.pattern_from_sss(m0)))
    s = P.split_bands(m, P.default_beta(m.n, P.compute_bandwidth(m)))
    plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, 1))
    b = G.make_x(m.n, 77)
    return m, s, plan, b


def test_mrs_matches_reference_recurrence(problem, oracle):
    m, s, plan, b = problem
    op = P.prepare(s, plan)
    out = P.mrs_solve(op, b, alpha=0.5, tol=0.0, maxiter=40)
    spmv = lambda v: oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, v)
    x_ref, res_ref = mrs_reference(spmv, b, 0.5, 40)
    assert out.iterations == 40
    np.testing.assert_allclose(out.residuals, res_ref, rtol=1e-8, atol=1e-14)
    assert rel_err(out.x.cpu().numpy(), x_ref) <= 1e-10


def test_mrs_converges_and_residual_is_true(problem, oracle):
    m, s, plan, b = problem
    op = P.prepare(s, plan)
    out = P.mrs_solve(op, b, alpha=0.5, tol=1e-10, maxiter=500)
    assert out.converged
    x = out.x.cpu().numpy()
    r = b - oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
    assert np.linalg.norm(r) <= 1e-9 * np.linalg.norm(b)
    # the recurrence's residual estimate tracks the true residual
    assert abs(np.linalg.norm(r) - out.residuals[-1]) <= 1e-9 * np.linalg.norm(b)
    # minimal residual: monotone non-increasing
    assert all(a >= b_ - 1e-12 for a, b_ in zip(out.residuals, out.residuals[1:]))
