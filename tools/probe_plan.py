"""Time plan build + one product for a config (debug helper for the GPU box)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2407_17651_b200 as P
from paper_2407_17651_b200 import generators as G
from paper_2407_17651_b200.device import operator_for_sss
from oracle import oracle as O
cfg = sys.argv[1]
t = time.time(); g = G.make_config(cfg) if cfg.startswith('c') else G.rmat(int(cfg[4:]), 16, seed_struct=3, seed_perm=4, seed_val=5); print("gen", time.time()-t, flush=True)
m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
t = time.time(); m = P.permute_sss(m0, P.rcm_order(P.pattern_from_sss(m0))); print("rcm", time.time()-t, flush=True)
t = time.time(); op = operator_for_sss(m); print("plan", time.time()-t, op.stats(), flush=True)
x = G.make_x(m.n, 1); xd = torch.from_numpy(x).cuda()
t = time.time(); y = op.matvec(xd); torch.cuda.synchronize(); print("first spmv", time.time()-t, flush=True)
ev0, ev1 = torch.cuda.Event(True), torch.cuda.Event(True)
ev0.record()
for _ in range(20): op.matvec(xd, y)
ev1.record(); torch.cuda.synchronize(); print("spmv ms", ev0.elapsed_time(ev1)/20, flush=True)
yr = O.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x); print("rel err", O.rel_err(y.cpu().numpy(), yr))
