"""Build one BASELINE config and run a few products (the command ncu wraps)."""
import sys
import time

sys.path.insert(0, '.')
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2407_17651_b200 as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
m, s, bw, beta, x = bench.build_problem(cfg)
plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, 1))
t = time.time()
op = P.prepare(s, plan)
print("plan", time.time() - t, op.stats(), flush=True)
xd = torch.from_numpy(x).cuda()
y = torch.empty_like(xd)
for _ in range(reps):
    op.matvec(xd, y)
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(True), torch.cuda.Event(True)
ev0.record()
for _ in range(reps):
    op.matvec(xd, y)
ev1.record()
torch.cuda.synchronize()
ms = ev0.elapsed_time(ev1) / reps
B = bench.algorithmic_bytes(m.n, m.nnz_offdiag)
print(f"{cfg}: spmv {ms:.4f} ms  {B / ms / 1e6:.1f} GB/s", flush=True)
import os
if os.environ.get("PARS3_PHASES") == "1":
    import numpy as np
    from paper_2407_17651_b200 import _lib
    ph = np.zeros(6, dtype=np.int64)
    _lib.check(_lib.load().pars3_plan_phases(op._handle, _lib.ptr(ph)))
    tot = ph.sum()
    print("phase cycles share (claim, windows, stream, store+fence, wait, flush):",
          [round(v / tot, 3) for v in ph], "per-CTA per-launch us:",
          round(tot / op.stats()["grid"] / (2 * reps) / 1.9e3, 1), flush=True)
