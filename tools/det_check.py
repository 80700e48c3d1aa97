"""Quick GPU check of the product forms: parity against the oracle, bitwise
repeatability over repeated products, the fused dot, status flags, and the
step time (y = A x + <y, y>) per config.

    python tools/det_check.py [c2 c3 c4 c5 small]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_17651_b200 as P  # noqa: E402
from paper_2407_17651_b200 import generators as G  # noqa: E402
from paper_2407_17651_b200.device import operator_for_sss  # noqa: E402
from oracle import oracle as O  # noqa: E402


def small_cases():
    return [G.grid5(100, seed_perm=1, seed_val=2), G.stencil27(24, seed_val=6, alpha=0.5),
            G.random_band(60000, 1024, 16, 0.01, seed_struct=11, seed_perm=12, seed_val=13),
            G.rmat(12, 16, seed_struct=3, seed_perm=4, seed_val=5)]


def check(name, m, x, reps=10, op=None):
    y_ref = O.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
    if op is None:
        op = operator_for_sss(m)
    xd = torch.from_numpy(x).cuda()
    ys = []
    dots = []
    for _ in range(reps):
        y, d = op.matvec_dot(xd, None)
        ys.append(y.cpu().numpy().copy())
        dots.append(float(d.item()))
    st = op.status()
    err = O.rel_err(ys[0], y_ref)
    same = all(np.array_equal(ys[0], yy) for yy in ys[1:]) and len(set(dots)) == 1
    yh = ys[0]
    derr = abs(dots[0] - float(yh @ yh)) / max(1e-300, float(yh @ yh))
    # timing of the step
    y = torch.empty_like(xd)
    dot = torch.empty(1, dtype=torch.float64, device="cuda")
    for _ in range(3):
        op.matvec_dot(xd, y, y, dot)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    k = 20
    e0.record()
    for _ in range(k):
        op.matvec_dot(xd, y, y, dot)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    s = op.stats()
    print(f"{name}: n={m.n} m={m.nnz_offdiag} rel_err={err:.2e} repeat_bitwise={same} dot_rel={derr:.1e} "
          f"status={st} step={ms:.4f} ms grid={s['grid_form']} words={s['accum_words']} "
          f"direct={s['direct']} loc={s['locality_order']} hbits={s['grid_hbits']} cmax={s['grid_cmax']}",
          flush=True)
    return err, same


def main():
    which = sys.argv[1:] or ["small"]
    for w in which:
        if w == "small":
            for g in small_cases():
                m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
                m = P.permute_sss(m0, P.rcm_order(P.pattern_from_sss(m0)))
                check(g.name, m, G.make_x(m.n, 9))
        else:
            import bench
            t = time.time()
            m, s, bw, beta, x = bench.build_problem(w)
            plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, 1))
            op = P.prepare(s, plan)
            print(f"{w}: built in {time.time() - t:.1f}s", flush=True)
            check(w, m, x, reps=5, op=op)


if __name__ == "__main__":
    main()
