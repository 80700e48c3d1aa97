"""Build one BASELINE config once, then time the product under several
environment settings (the plan reads its tuning knobs at creation):

    python tools/exp_env.py c5 "" "PARS3_CONV_REV=1" "PARS3_YACC_KEEP_MB=48,PARS3_CONV_REV=1"

Prints, per setting, the SpMV + <y, y> step and the per-phase times."""
import os
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2407_17651_b200 as P  # noqa: E402
from paper_2407_17651_b200 import _lib  # noqa: E402

cfg = sys.argv[1]
settings = sys.argv[2:] or [""]
reps = int(os.environ.get("REPS", "30"))
m, s, bw, beta, x = bench.build_problem(cfg)
plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, 1))
xd = torch.from_numpy(x).cuda()
B = bench.algorithmic_bytes(m.n, m.nnz_offdiag)
ref = None
for st in settings:
    kv = dict(t.split("=", 1) for t in st.split(",") if t)
    for k, v in kv.items():
        os.environ[k] = v
    if "L2_SETASIDE_MB" in kv:  # cudaLimitPersistingL2CacheSize
        from cuda.bindings import runtime as rt
        print("set-aside", rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize,
                                                 int(kv["L2_SETASIDE_MB"]) << 20),
              rt.cudaDeviceGetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize))
    op = P.prepare(s, plan)
    y = torch.empty_like(xd)
    dot = torch.empty(1, dtype=torch.float64, device="cuda")
    for _ in range(5):
        op.matvec_dot(xd, y, y, dot)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(True), torch.cuda.Event(True)
    ev0.record()
    for _ in range(reps):
        op.matvec_dot(xd, y, y, dot)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / reps
    ph = np.zeros(4, dtype=np.float64)
    _lib.check(_lib.load().pars3_plan_profile(op._handle, _lib.ptr(xd), _lib.ptr(y), 1, reps, _lib.ptr(ph), None))
    yh = y.cpu().numpy()
    if ref is None:
        ref = yh
    err = float(np.max(np.abs(yh - ref)) / max(1.0, float(np.max(np.abs(ref)))))
    print(f"{cfg} [{st}]: step {ms:.4f} ms {B / ms / 1e6:.0f} GB/s  phases main {ph[0]:.4f} finish {ph[1]:.4f} "
          f"rest {ph[2]:.4f} total {ph[3]:.4f}  diff-vs-first {err:.1e}", flush=True)
    op.close()
    del op
    getattr(s, "_device", {}).clear()  # (prepare caches the operator on the split)
    for k in kv:
        del os.environ[k]
