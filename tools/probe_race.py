"""Repeated launches in a forced mode; report wrong rows (debug helper)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2407_17651_b200 as P
from paper_2407_17651_b200 import generators as G
from paper_2407_17651_b200.device import operator_for_sss
from oracle import oracle as O
k, mode, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
fill = sys.argv[4] if len(sys.argv) > 4 else "nan"
tile_rows = int(sys.argv[5]) if len(sys.argv) > 5 else 0
g = G.stencil27(k, seed_val=1, alpha=0.5)
m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
m = P.permute_sss(m0, P.rcm_order(P.pattern_from_sss(m0)))
op = operator_for_sss(m, options=(tile_rows, 0, 0, -1, mode))
print(k, mode, op.stats(), flush=True)
x = G.make_x(m.n, 1); xd = torch.from_numpy(x).cuda()
yr = O.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
y = torch.empty(m.n, dtype=torch.float64, device="cuda")
for r in range(reps):
    y.fill_(float(fill))
    op.matvec(xd, y); torch.cuda.synchronize()
    yh = y.cpu().numpy()
    bad = np.flatnonzero(~(np.abs(yh - yr) <= 1e-12 * max(1, np.abs(yr).max())))
    print("launch", r, "bad rows", bad.size, bad[:10], (bad[-5:] if bad.size else ""), flush=True)
