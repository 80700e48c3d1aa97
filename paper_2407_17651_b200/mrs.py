"""MRS: minimal residual solver for shifted skew-symmetric systems (A = alpha*I + S).

The reference stops at the product (SPEC.md:16 lists the solvers as out of
scope; PAPER.md:49 motivates PARS3 by MRS).  This driver is the iteration the
north star names: each step is one PARS3 product plus one inner product.

Skew Lanczos on S (S v_j = g_{j+1} v_{j+1} - g_j v_{j-1}, the tridiagonal is
skew because v^T S v = 0), so A V_j = V_{j+1} H_j with H's column j equal to
(-g_j, alpha, g_{j+1}); the least-squares problem min ||beta e_1 - H y|| is
solved by Givens rotations exactly as in MINRES, with the solution updated
through three-term direction vectors.  The product computes A v (with the
alpha diagonal), so the Lanczos vector is u = A v_j - alpha v_j + g_j v_{j-1}.

Per iteration on the GPU, with no host round trip: the product (y = A v_j,
the grid-form PARS3 kernels), one fused pass for u and its share of
||u||^2, the fixed-order norm, the Givens rotation (one device thread: the
recurrence scalars live in a device state), and one fused pass for the
direction, x and v_{j+1}.  The host only swaps buffer handles; it reads the
state every ``check_every`` iterations to stop early.  Distributed (one
rank per GPU, rows sharded by partition_rows): each rank runs the same loop
on its block with its distributed operator, and the norm is one 8-byte
all-reduce per iteration on the device (NCCL), the rotation replicated.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import ctypes

import numpy as np

from . import _lib

__all__ = ["MrsResult", "mrs_solve", "mrs_solve_distributed", "RankOperator"]


@dataclass
class MrsResult:
    x: object                 # solution (CUDA tensor)
    iterations: int
    residuals: list = field(default_factory=list)  # |phi_{j+1}| = ||b - A x_j|| per step
    converged: bool = False


def mrs_solve(op, b, alpha: float, tol: float = 1e-10, maxiter: int = 100, stream=None,
              check_every: int = 10, group=None) -> MrsResult:
    """Solve (alpha I + S) x = b with the PARS3 operator ``op`` (whose matrix
    must be alpha*I + S) from x_0 = 0.  Stops when ||r_j|| <= tol * ||b|| or
    after ``maxiter`` iterations.  ``group``: a torch.distributed process
    group when ``op`` is one rank's distributed operator and ``b`` that
    rank's rows (the norms are then all-reduced on the device)."""
    import torch
    L = _lib.load()
    n = op.n
    dev = op.device
    t = torch.float64
    b = torch.as_tensor(b, dtype=t).to(dev).contiguous()
    st = _lib.stream_ptr(stream)
    size, parts = ctypes.c_int32(), ctypes.c_int32()
    _lib.check(L.pars3_mrs_state_size(ctypes.byref(size), ctypes.byref(parts)))
    state = torch.zeros(size.value, dtype=t, device=dev)
    part = torch.zeros(parts.value, dtype=t, device=dev)
    resid = torch.zeros(maxiter + 1, dtype=t, device=dev)

    def allreduce(view):
        if group is not None:
            import torch.distributed as dist
            dist.all_reduce(view, group=group)

    bb = torch.dot(b, b).reshape(1)
    allreduce(bb)
    beta_t = torch.sqrt(bb)
    # state: c1 = c2 = 1, phi = beta, beta, tol, alpha (device ops, no sync)
    state[1] = 1.0
    state[3] = 1.0
    state[5:7] = beta_t.expand(2)
    state[14] = float(tol)
    state[15] = float(alpha)
    state[18] = -float(alpha)  # (the fused product's coefficient of v)
    resid[0:1] = beta_t
    x = torch.zeros(n, dtype=t, device=dev)
    v = b / torch.where(beta_t > 0, beta_t, torch.ones_like(beta_t))  # v_j
    w = torch.zeros(n, dtype=t, device=dev)   # v_{j-1}, then u
    dm1 = torch.zeros(n, dtype=t, device=dev)  # d_{j-1}
    dm2 = torch.zeros(n, dtype=t, device=dev)  # d_{j-2}, then d_j
    y = torch.empty(n, dtype=t, device=dev)   # A v_j; with the fused product: the free buffer u lands in
    # the product fused with the Lanczos update (pars3_plan_product_axpy): u = A v - alpha v +
    # gamma w and ||u||^2 in the product's finish pass, no y written and read back
    fused = group is None and hasattr(op, "matvec_axpy")
    # the update pass leaves the bound of v_{j+1} in the plan's slot, so the strict product skips its pass over v
    slot = op.xbound_slot() if fused and hasattr(op, "xbound_slot") else 0
    import os
    if os.environ.get("PARS3_MRS_NO_XBOUND") == "1":  # A/B knob
        slot = 0
    if os.environ.get("PARS3_MRS_NO_FUSE") == "1":
        fused, slot = False, 0
    res = MrsResult(x=x, iterations=0)
    if float(beta_t.item()) == 0.0:
        res.residuals, res.converged = [0.0], True
        return res
    j = 0
    for j in range(1, maxiter + 1):
        if fused:
            # u (in y's buffer) = A v - alpha v + gamma w, state[7] = ||u||^2; strict: a pure function of v
            op.matvec_axpy(v, y, v, state[18:19], w, state[0:1], dot=state[7:8], stream=stream, strict=True,
                           xbound=bool(slot) and j > 1)
            u = y
        else:
            op.matvec(v, y, stream=stream, strict=True)  # each product a pure function of v
            _lib.check(L.pars3_mrs_lanczos_dev(n, _lib.ptr(y), _lib.ptr(v), _lib.ptr(w), _lib.ptr(state),
                                               _lib.ptr(part), st), "mrs_lanczos")
            allreduce(state[7:8])  # the step's inner product, summed over ranks
            u = w
        _lib.check(L.pars3_mrs_rotate_dev(_lib.ptr(state), _lib.ptr(resid), j, st), "mrs_rotate")
        _lib.check(L.pars3_mrs_update_dev2(n, _lib.ptr(u), _lib.ptr(v), _lib.ptr(dm2), _lib.ptr(dm1),
                                           _lib.ptr(x), _lib.ptr(state), slot or None, st), "mrs_update")
        # rotate the buffers: v_{j+1} <- u, v_j -> w's slot (fused: old w becomes the free buffer); d_j <- dm2
        if fused:
            v, w, y = y, v, w
        else:
            v, w = w, v
        dm1, dm2 = dm2, dm1
        if check_every and j % check_every == 0 and float(state[16].item()) != 0.0:
            break
    flags = state[13:18].cpu().numpy()  # done, tol, alpha, pending, converged iteration
    res.converged = bool(flags[3] != 0.0)
    res.iterations = int(flags[4]) if res.converged else j
    res.residuals = [float(r) for r in resid[:res.iterations + 1].cpu().numpy()]
    res.x = x
    return res


class RankOperator:
    """A distributed operator (PeerPars3 / DistributedPars3: one rank's rows)
    seen through the single-GPU interface mrs_solve drives: ``n`` rows,
    ``device``, ``matvec(v, y)``."""

    def __init__(self, dop):
        self.dop = dop
        self.n = int(dop.shard.hi - dop.shard.lo)
        self.device = dop.device

    def matvec(self, v, y, stream=None, strict=True):
        y.copy_(self.dop.matvec(v))
        return y


def mrs_solve_distributed(dop, b_own, alpha: float, group=None, tol: float = 1e-10, maxiter: int = 100,
                          check_every: int = 10) -> MrsResult:
    """MRS over ranks (one per GPU): each rank iterates on its row block
    (``b_own`` = b[lo:hi]) with its distributed operator; the only exchange
    besides the products is one 8-byte all-reduce per iteration (the norm),
    on the device.  ``x`` of the result is this rank's block."""
    return mrs_solve(RankOperator(dop), b_own, alpha, tol=tol, maxiter=maxiter, check_every=check_every,
                     group=group if group is not None else _default_group())


def _default_group():
    import torch.distributed as dist
    return dist.group.WORLD
