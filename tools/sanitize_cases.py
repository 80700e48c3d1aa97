"""Small products through every kernel form, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Forms: the grid tile kernel + k_finish (window and list tiles, 2- and
3-word accumulators), the fp64 redo (non-finite x), the RED form (y += A x),
a locality-order plan, the row-major full-CSR form with warp-crossing rows,
the atomic baseline, the GPU RCM / relabel / split chain (c1), and MRS."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_17651_b200 as P  # noqa: E402
from paper_2407_17651_b200 import generators as G  # noqa: E402
from paper_2407_17651_b200.device import operator_for_sss  # noqa: E402
from oracle import oracle as O  # noqa: E402


def check(name, y, m, x):
    y_ref = O.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
    err = O.rel_err(np.asarray(y), y_ref)
    print(f"{name}: rel_err {err:.2e}", flush=True)
    assert err <= 1e-12, name


def rcm(g):
    m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    return P.permute_sss(m0, P.rcm_order(P.pattern_from_sss(m0)))


def main():
    torch.cuda.set_device(0)
    cases = [("grid5_windows", G.grid5(40, seed_perm=1, seed_val=2), ()),
             ("stencil27_2word", G.stencil27(10, seed_val=6, alpha=0.5), ()),
             ("rmat_3word", G.rmat(9, 16, seed_struct=3, seed_perm=4, seed_val=5), (0, 0, 0, -1, 0, 64, 0)),
             ("band_locality", G.random_band(6000, 300, 8, 0.02, seed_struct=1, seed_perm=2, seed_val=3),
              (0, 0, 0, -1, 0, 8, 0)),
             ("rmat_rowmajor", G.rmat(10, 16, seed_struct=7, seed_perm=8, seed_val=9), (0, 0, 0, -1, 0, 32, 0)),
             ("tiny_tiles_list", G.random_band(3000, 900, 6, 0.05, seed_struct=4, seed_perm=5, seed_val=6),
              (64, 128, 4, 0, 0, 64, 0))]
    for name, g, opts in cases:
        m = rcm(g)
        x = G.make_x(m.n, 9)
        op = operator_for_sss(m, options=opts or None)
        xd = torch.from_numpy(x).cuda()
        y, dot = op.matvec_dot(xd, None)
        check(name + " " + str({k: v for k, v in op.stats().items() if k in ("grid_form", "direct",
                                                                              "locality_order", "accum_words")}),
              y.cpu().numpy(), m, x)
        y2 = torch.zeros(m.n, dtype=torch.float64, device="cuda")
        op.matvec(xd, y2, accumulate=True)
        check(name + " accumulate", y2.cpu().numpy(), m, x)
        xb = x.copy()
        xb[3] = np.inf
        yb = op.matvec(torch.from_numpy(xb).cuda()).cpu().numpy()
        with np.errstate(all="ignore"):
            yr = O.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, xb)
        assert np.array_equal(np.isnan(yb), np.isnan(yr)) and np.array_equal(np.isinf(yb), np.isinf(yr)), name
        print(f"{name} non-finite x: IEEE pattern ok (status {op.status()})", flush=True)
    m = rcm(G.grid5(30, seed_perm=3, seed_val=4))
    x = G.make_x(m.n, 2)
    check("atomic", P.spmv_atomic(m, x, 4), m, x)
    from paper_2407_17651_b200.pipeline import prepare_gpu
    g = G.make_config("c1")
    m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    perm, m, s, bw = prepare_gpu(m0)
    assert np.array_equal(perm.forward, P.rcm_order(P.pattern_from_sss(m0)).forward)
    print("prepare_gpu c1: labels == host chain", flush=True)
    a = G.stencil27(8, seed_val=1, alpha=0.5)
    ma = P.SssMatrix._trusted(a.n, a.row_ptr, a.col_ind, a.off_diags, a.diags)
    res = P.mrs_solve(operator_for_sss(ma), G.make_x(ma.n, 4), 0.5, tol=1e-10, maxiter=60)
    print(f"mrs: {res.iterations} iterations, converged {res.converged}", flush=True)
    print("SANITIZE CASES DONE", flush=True)


if __name__ == "__main__":
    main()
