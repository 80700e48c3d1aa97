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

Per iteration on the GPU: the tile kernel (y = A v_j), one fused pass for u
and ||u||^2, one fused pass for v_{j+1}, the direction and x; the rotation
scalars are a few flops on the host (one 8-byte read per iteration).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

from . import _lib

__all__ = ["MrsResult", "mrs_solve"]


@dataclass
class MrsResult:
    x: object                 # solution (CUDA tensor)
    iterations: int
    residuals: list = field(default_factory=list)  # |phi_{j+1}| = ||b - A x_j|| per step
    converged: bool = False


def mrs_solve(op, b, alpha: float, tol: float = 1e-10, maxiter: int = 100, stream=None) -> MrsResult:
    """Solve (alpha I + S) x = b with the PARS3 operator ``op`` (whose matrix
    must be alpha*I + S) from x_0 = 0.  Stops when ||r_j|| <= tol * ||b|| or
    after ``maxiter`` iterations."""
    import torch
    L = _lib.load()
    n = op.n
    dev = op.device
    t = torch.float64
    b = torch.as_tensor(b, dtype=t).to(dev).contiguous()
    st = _lib.stream_ptr(stream)
    x = torch.zeros(n, dtype=t, device=dev)
    beta = float(torch.linalg.vector_norm(b).item())
    res = MrsResult(x=x, iterations=0, residuals=[beta], converged=beta == 0.0)
    if beta == 0.0:
        return res
    v = b / beta                       # v_j
    w = torch.zeros(n, dtype=t, device=dev)   # v_{j-1}, then u
    dm1 = torch.zeros(n, dtype=t, device=dev)  # d_{j-1}
    dm2 = torch.zeros(n, dtype=t, device=dev)  # d_{j-2}, then d_j
    y = torch.empty(n, dtype=t, device=dev)
    norm2 = torch.zeros(1, dtype=t, device=dev)
    gamma = 0.0                        # g_j
    c1, s1, c2, s2 = 1.0, 0.0, 1.0, 0.0  # rotations G_{j-1}, G_{j-2}
    phi = beta
    for j in range(1, maxiter + 1):
        op.matvec(v, y, stream=stream)
        _lib.check(L.pars3_mrs_lanczos(n, _lib.ptr(y), _lib.ptr(v), _lib.ptr(w), float(alpha),
                                       float(gamma), _lib.ptr(norm2), st), "mrs_lanczos")
        gnext = math.sqrt(float(norm2.item()))  # the step's inner product
        # column j of H: (-g_j, alpha, g_{j+1}); previous rotations, then a new one
        h1 = -gamma
        r0 = s2 * h1
        h1p = c2 * h1
        r1 = c1 * h1p + s1 * alpha
        h2p = -s1 * h1p + c1 * alpha
        r2 = math.hypot(h2p, gnext)
        c, s = (h2p / r2, gnext / r2) if r2 > 0 else (1.0, 0.0)
        tau = c * phi
        phi = -s * phi
        inv_g = 1.0 / gnext if gnext > 0 else 0.0
        _lib.check(L.pars3_mrs_update(n, _lib.ptr(w), inv_g, _lib.ptr(v), _lib.ptr(dm2),
                                      _lib.ptr(dm1), r0, r1, 1.0 / r2, tau, _lib.ptr(x), st),
                   "mrs_update")
        # rotate the buffers: v_{j+1} <- w, v_j -> w's slot; d_j <- dm2
        v, w = w, v
        dm1, dm2 = dm2, dm1
        gamma = gnext
        c2, s2, c1, s1 = c1, s1, c, s
        res.iterations = j
        res.residuals.append(abs(phi))
        if abs(phi) <= tol * beta or gnext == 0.0:
            res.converged = True
            break
    res.x = x
    return res
