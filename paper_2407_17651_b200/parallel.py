"""PARS3 product entry points (reference parallel.py), on the GPU.

``spmv_pars3(s, plan, x, p=None)`` keeps the reference signature and error
behaviour (parallel.py:123-183): ValueError when the plan does not belong
to the split (n or beta differ) or ``p`` differs from ``plan.p``, ValueError
on a wrong-length x.  The product runs through libpars3's device plan; the
result equals the reference's within the 1e-12 contract (SPEC.md D14).

``spmv_atomic(m, x, t=1)`` is the paper's lock-free comparison kernel
(parallel.py:416-447) as a native CUDA kernel with fp64 L2 reductions.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .formats import SssMatrix, as_vector
from .split import BandSplit, PartitionPlan

__all__ = ["spmv_pars3", "spmv_atomic", "prepare"]


def _check_pair(s: BandSplit, plan: PartitionPlan, p) -> int:
    if plan.n != s.n or plan.beta != s.beta:
        raise ValueError(f"plan (n={plan.n}, beta={plan.beta}) does not match "
                         f"split (n={s.n}, beta={s.beta})")
    if p is None:
        return plan.p
    if p != plan.p:
        raise ValueError(f"worker count {p} does not match the plan's {plan.p}")
    return plan.p


def prepare(s: BandSplit, plan: PartitionPlan | None = None, device=None):
    """Upload the split and build the device plan (cached on ``s``)."""
    from .device import operator_for_split
    p = plan.p if plan is not None else 1
    bs = plan.block_start if plan is not None else None
    return operator_for_split(s, p=p, block_start=bs, device=device)


def spmv_pars3(s: BandSplit, plan: PartitionPlan, x, p: int | None = None, out=None,
               non_blocking=False):
    """Staged 3-way product y = A x (GPU).  numpy in -> numpy out; CUDA
    tensor in -> CUDA tensor out (optionally into ``out``); pinned host
    tensor in -> host tensor out, with ``non_blocking`` pipelining the copies
    of consecutive calls (result ready after torch.cuda.synchronize())."""
    _check_pair(s, plan, p)
    if not hasattr(x, "data_ptr"):
        x = as_vector(x, s.n)
    from .serial import _run
    return _run(prepare(s, plan), x, s.n, out, non_blocking)


def spmv_atomic(m: SssMatrix, x, t: int = 1, out=None):
    """Lock-free product with atomic mirror updates (parallel.py:430-447).
    ``t`` is validated like the reference; the GPU decides the parallelism.
    Reproducible within rounding only."""
    if t < 1:
        raise ValueError(f"worker count must be at least 1, got {t}")
    from .device import require_cuda, sss_device
    torch = require_cuda()
    op = sss_device(m)
    numpy_in = not isinstance(x, torch.Tensor)
    if numpy_in:
        xv = as_vector(x, m.n)
        if m.n == 0:
            return np.zeros(0)
        xd = torch.from_numpy(xv).to(op.device)
    else:
        if x.dim() != 1 or x.shape[0] != m.n:
            raise ValueError(f"x must be a vector of length {m.n}, got shape {tuple(x.shape)}")
        xd = x.to(device=op.device, dtype=torch.float64).contiguous()
    y = out if out is not None else torch.empty(m.n, dtype=torch.float64, device=op.device)
    _lib.check(_lib.load().pars3_sss_spmv_atomic(
        m.n, _lib.ptr(op.row_ptr), _lib.ptr(op.col_ind), _lib.ptr(op.off_diags),
        _lib.ptr(op.diags), _lib.ptr(xd), _lib.ptr(y), _lib.stream_ptr()), "spmv_atomic")
    return y.cpu().numpy() if numpy_in else y
