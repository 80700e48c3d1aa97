"""Time the MRS solver on a BASELINE config (c5: 100 iterations, as the config names):
python tools/mrs_time.py c5 100"""
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2407_17651_b200 as P  # noqa: E402
from paper_2407_17651_b200.mrs import mrs_solve  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
m, s, bw, beta, x = bench.build_problem(cfg)
plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, 1))
op = P.prepare(s, plan)
alpha = float(m.diags[0])
b = torch.from_numpy(np.random.default_rng(7).uniform(-1, 1, m.n)).cuda()
mrs_solve(op, b, alpha, tol=0.0, maxiter=5, check_every=0)
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(True), torch.cuda.Event(True)
ev0.record()
r = mrs_solve(op, b, alpha, tol=0.0, maxiter=iters, check_every=0)
ev1.record()
torch.cuda.synchronize()
ms = ev0.elapsed_time(ev1)
print(f"{cfg}: {iters} MRS iterations {ms:.2f} ms = {ms / iters:.4f} ms per iteration; "
      f"residual {r.residuals[0]:.3e} -> {r.residuals[-1]:.3e}", flush=True)
