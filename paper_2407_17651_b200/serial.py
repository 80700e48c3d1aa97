"""Skyline product and operation accounting (reference serial.py).

``spmv_serial(m, x)`` keeps the reference name and contract (serial.py:64-73:
y = A x over an SssMatrix) but runs on the GPU through the same native plan
as ``spmv_pars3``; it matches the reference's serial result within the
1e-12 contract (SPEC.md D14), not bitwise, since the summation order is the
GPU's.  ``count_ops`` (serial.py:28-47) defines the work budget
(reads m + n, multiply-adds 2m + n) that the GFLOP/s figures use.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .formats import CooMatrix, SssMatrix, as_vector

__all__ = ["OpCounter", "count_ops", "spmv_serial", "spmv_dense"]


@dataclass(frozen=True)
class OpCounter:
    element_reads: int = 0
    multiply_adds: int = 0

    def __add__(self, other: "OpCounter") -> "OpCounter":
        return OpCounter(self.element_reads + other.element_reads,
                         self.multiply_adds + other.multiply_adds)


def count_ops(m: SssMatrix) -> OpCounter:
    """m + n element reads and 2m + n multiply-adds per product."""
    return OpCounter(element_reads=m.nnz_offdiag + m.n, multiply_adds=2 * m.nnz_offdiag + m.n)


def _run(op, x, n, out=None, non_blocking=False, strict=True):
    """Dispatch on the input's home: CUDA tensor -> CUDA result; host torch
    tensor (pinned for async copies) -> host tensor (into ``out`` if given),
    through the operator's copy pipeline (``non_blocking``: consecutive calls
    overlap their copies; the result is ready after torch.cuda.synchronize());
    anything else -> numpy.  These one-call entry points are strict: the
    product is a pure function of x, bit for bit (pars3_plan_product)."""
    from .device import require_cuda
    torch = require_cuda()
    if isinstance(x, torch.Tensor):
        if x.dim() != 1 or x.shape[0] != n:
            raise ValueError(f"x must be a vector of length {n}, got shape {tuple(x.shape)}")
        if not x.is_cuda:
            if x.dtype != torch.float64:
                x = x.to(torch.float64)
            return op.matvec_host(x.contiguous(), out, non_blocking=non_blocking, strict=strict)
        xd = x.to(device=op.device, dtype=torch.float64).contiguous()
        return op.matvec(xd, out, strict=strict)
    xv = as_vector(x, n)
    if n == 0:
        return np.zeros(0)
    xd = torch.from_numpy(xv).to(op.device)
    return op.matvec(xd, strict=strict).cpu().numpy()


def spmv_serial(m: SssMatrix, x, out=None, non_blocking=False):
    """y = A x for a skyline matrix (GPU).  numpy in -> numpy out; a CUDA
    tensor in -> a CUDA tensor out; a host tensor in -> a host tensor out."""
    from .device import operator_for_sss
    if not hasattr(x, "data_ptr"):
        as_vector(x, m.n)
    return _run(operator_for_sss(m), x, m.n, out, non_blocking)


def spmv_dense(m, x) -> np.ndarray:
    """Dense product for demos/small checks (host; not part of the product path)."""
    if isinstance(m, SssMatrix):
        from .formats import sss_to_coo
        m = sss_to_coo(m)
    if not isinstance(m, CooMatrix):
        raise TypeError(f"expected CooMatrix or SssMatrix, got {type(m).__name__}")
    return m.to_dense() @ as_vector(x, m.n)
