"""Time the lock-free atomic comparison kernel (spmv_atomic) against the
tile kernel on one config.  Usage: python tools/atomic_time.py c3"""
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2407_17651_b200 as P  # noqa: E402

cfg = sys.argv[1]
m, s, bw, beta, x = bench.build_problem(cfg)
xd = torch.from_numpy(x).cuda()
y = torch.empty_like(xd)
B = bench.algorithmic_bytes(m.n, m.nnz_offdiag)


def timeit(f, reps=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ta = timeit(lambda: P.spmv_atomic(m, xd, out=y))
ya = y.clone()
op = P.prepare(s)
tt = timeit(lambda: op.matvec(xd, y))
err = float((y - ya).abs().max() / max(1.0, float(ya.abs().max())))
print(f"{cfg}: atomic {ta:.4f} ms {B / ta / 1e6:.0f} GB/s | tiles {tt:.4f} ms {B / tt / 1e6:.0f} GB/s "
      f"| diff {err:.1e}", flush=True)
