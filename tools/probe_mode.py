"""Run stencil27(k) through the tile kernel in a forced mode (debug helper)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2407_17651_b200 as P
from paper_2407_17651_b200 import generators as G
from paper_2407_17651_b200.device import operator_for_sss
from oracle import oracle as O
k, mode = int(sys.argv[1]), int(sys.argv[2])
g = G.stencil27(k, seed_val=1, alpha=0.5)
m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
m = P.permute_sss(m0, P.rcm_order(P.pattern_from_sss(m0)))
op = operator_for_sss(m, options=(0, 0, 0, -1, mode))
print(k, mode, op.stats(), flush=True)
x = G.make_x(m.n, 1); xd = torch.from_numpy(x).cuda()
yr = O.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
for r in range(reps):
    y = op.matvec(xd); torch.cuda.synchronize()
    print("launch", r, "rel err", O.rel_err(y.cpu().numpy(), yr), flush=True)
