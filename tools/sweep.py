"""Plan-option sweep on one config: build the problem once, time the tile
kernel for several pars3_plan_options tuples (tile_rows, local_slots,
seg_max, gap, mode).  Usage: python tools/sweep.py c5 "0,0,0,-1,1" "0,0,0,-1,2" ..."""
import os
import sys
import time

sys.path.insert(0, '.')
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2407_17651_b200 as P  # noqa: E402
from paper_2407_17651_b200.device import Pars3Operator  # noqa: E402

cfg = sys.argv[1]
def parse(a):
    """[ENV=V[;ENV=V]:]tile_rows,local_slots,seg_max,gap,mode"""
    env = {}
    if ":" in a:
        e, a = a.split(":", 1)
        env = dict(kv.split("=") for kv in e.split(";") if kv)
    return env, tuple(int(v) for v in a.split(",")) if a else ()


variants = [parse(a) for a in sys.argv[2:]] or [({}, ())]
m, s, bw, beta, x = bench.build_problem(cfg)
xd = torch.from_numpy(x).cuda()
y = torch.empty_like(xd)
B = bench.algorithmic_bytes(m.n, m.nnz_offdiag)
yref = None
for env, opt in variants:
    os.environ.update(env)
    t = time.time()
    op = Pars3Operator(s.n, s.beta, s.diag, s.mid_ptr, s.mid_col, s.mid_val, s.outer_row,
                       s.outer_col, s.outer_val, options=opt)
    tp = time.time() - t
    for _ in range(3):
        op.matvec(xd, y)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(True), torch.cuda.Event(True)
    reps = 20
    ev0.record()
    for _ in range(reps):
        op.matvec(xd, y)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / reps
    if yref is None:
        yref = y.clone()
    err = float((y - yref).abs().max() / max(1.0, float(yref.abs().max())))
    print(f"{cfg} env={env} opt={opt}: {ms:.4f} ms {B / ms / 1e6:.0f} GB/s  plan {tp:.1f}s  "
          f"dev_vs_first {err:.1e} {op.stats()}", flush=True)
    op.close()
