"""Instrumented protocol models of the products (reference serial.py:76-100,
parallel.py:186-413): ``spmv_serial_instrumented`` and
``spmv_pars3_instrumented`` with their record types ``AccumulationMessage``,
``WorkerContext`` and ``Pars3Trace``.

These are INSPECTION tools, not product paths: they replay the reference's
staged protocol on the host with full bookkeeping -- who owns which rows,
which halo each worker received, every accumulation message with its slot,
the stage order, and operation tallies -- for tiny inputs in tests, demos and
debugging.  ``spmv_pars3`` / ``spmv_serial`` never call them (those run on
the GPU and raise without one).

The arithmetic follows the reference's per-element update order, so ``y``
is bit-identical to the reference's CPU kernels (``_pars3``,
``_spmv_sss``), which is what the reference's twins promise.  Each stage is
expressed as one ordered stream of (target, value) updates applied with
``np.add.at`` (unbuffered, applied in array order), which is the same
sequence of floating-point additions as the reference's loops.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .formats import SssMatrix, as_vector
from .serial import OpCounter
from .split import BandSplit, PartitionPlan

__all__ = ["AccumulationMessage", "WorkerContext", "Pars3Trace", "spmv_pars3_instrumented",
           "spmv_serial_instrumented"]


@dataclass(frozen=True)
class AccumulationMessage:
    """One deferred cross-block update: ``value`` goes into ``y[target_row]``
    on ``target_worker``; it came from element (source_row, source_col) on
    ``source_worker``, and ``slot`` (its conflict-list position) fixes the
    application order (parallel.py:186-203)."""

    target_worker: int
    target_row: int
    value: float
    source_worker: int
    source_row: int
    source_col: int
    slot: int


@dataclass
class WorkerContext:
    """One worker's private state (parallel.py:206-254): it reads x only from
    its block or its delivered halo, writes y only inside its block."""

    worker_id: int
    row_start: int
    row_end: int
    halo_lo: int
    local_diag: np.ndarray
    local_x: np.ndarray | None = None
    halo_x: np.ndarray | None = None
    local_y: np.ndarray | None = None
    outbox: list = field(default_factory=list)
    element_reads: int = 0
    multiply_adds: int = 0
    stages: list = field(default_factory=list)

    def x_at(self, c: int) -> float:
        """x[c] from the block or the halo; AssertionError outside both."""
        if self.row_start <= c < self.row_end:
            return float(self.local_x[c - self.row_start])
        assert self.halo_x is not None, f"worker {self.worker_id} read halo before exchange"
        assert self.halo_lo <= c < self.row_start, (
            f"worker {self.worker_id} read x[{c}] outside block and halo")
        return float(self.halo_x[c - self.halo_lo])

    def y_add(self, i: int, delta: float) -> None:
        """y[i] += delta; AssertionError if i is outside the block."""
        assert self.row_start <= i < self.row_end, (
            f"worker {self.worker_id} wrote y[{i}] outside its block "
            f"[{self.row_start}, {self.row_end})")
        self.local_y[i - self.row_start] += delta

    # vectorised forms used by the replay (same contracts)
    def _gather_x(self, cols: np.ndarray) -> np.ndarray:
        cols = np.asarray(cols, dtype=np.int64)
        own = (cols >= self.row_start) & (cols < self.row_end)
        if not own.all():
            assert self.halo_x is not None, f"worker {self.worker_id} read halo before exchange"
            bad = ~own & ((cols < self.halo_lo) | (cols >= self.row_start))
            assert not bad.any(), (
                f"worker {self.worker_id} read x[{int(cols[bad][0])}] outside block and halo")
        out = np.empty(cols.size)
        out[own] = self.local_x[cols[own] - self.row_start]
        out[~own] = self.halo_x[cols[~own] - self.halo_lo]
        return out

    def _add_stream(self, rows: np.ndarray, vals: np.ndarray) -> None:
        bad = (rows < self.row_start) | (rows >= self.row_end)
        assert not bad.any(), (f"worker {self.worker_id} wrote y[{int(rows[bad][0])}] outside its "
                               f"block [{self.row_start}, {self.row_end})")
        np.add.at(self.local_y, rows - self.row_start, vals)


@dataclass
class Pars3Trace:
    """Everything observable about one replayed staged run (parallel.py:257-282)."""

    y: np.ndarray
    contexts: list
    messages: list
    stage_log: list
    coordinator_reads: int
    coordinator_multiply_adds: int
    outer_count: int

    @property
    def message_count(self) -> int:
        return len(self.messages)

    def total_ops(self) -> OpCounter:
        """Work over all workers plus the coordinator (= 2m + n multiply-adds)."""
        total = OpCounter(self.coordinator_reads, self.coordinator_multiply_adds)
        for ctx in self.contexts:
            total = total + OpCounter(ctx.element_reads, ctx.multiply_adds)
        return total


def _interleave(a_idx, a_val, b_idx, b_val):
    """[a0, b0, a1, b1, ...]: the row update and the mirror update of each
    element, in element order."""
    idx = np.empty(2 * a_idx.size, dtype=np.int64)
    val = np.empty(2 * a_idx.size)
    idx[0::2], idx[1::2] = a_idx, b_idx
    val[0::2], val[1::2] = a_val, b_val
    return idx, val


def spmv_serial_instrumented(m: SssMatrix, x) -> tuple[np.ndarray, OpCounter]:
    """Counted replay of the serial skyline product (serial.py:76-100): per
    row, ``acc = d_i x_i`` plus ``v x_c`` over its entries (in order) while
    each mirror ``-v x_i`` goes straight into ``y[c]``; ``acc`` lands in
    ``y[i]`` after the row.  Returns (y, OpCounter(m + n, 2m + n))."""
    x = as_vector(x, m.n)
    y = np.zeros(m.n)
    for i in range(m.n):
        xi = x[i]
        acc = m.diags[i] * xi
        k0, k1 = int(m.row_ptr[i]), int(m.row_ptr[i + 1])
        cols = m.col_ind[k0:k1]
        vals = m.off_diags[k0:k1]
        for v, xc in zip(vals.tolist(), x[cols].tolist()):
            acc += v * xc
        if k1 > k0:
            np.add.at(y, cols, -vals * xi)
        y[i] += acc
    return y, OpCounter(element_reads=m.nnz_offdiag + m.n, multiply_adds=2 * m.nnz_offdiag + m.n)


def spmv_pars3_instrumented(s: BandSplit, plan: PartitionPlan, x, p: int | None = None) -> Pars3Trace:
    """Replay the staged protocol with full bookkeeping (parallel.py:285-413):
    scatter, halo exchange along the ascending chain, per worker the
    diagonal / safe / conflict sweeps (conflict mirrors become messages),
    message application in slot order, gather, and the coordinator's outer
    pass.  ``trace.y`` is bit-identical to the reference's ``spmv_pars3``."""
    from .parallel import _check_pair
    p = _check_pair(s, plan, p)
    x = as_vector(x, s.n)
    log: list = []
    ctxs = [WorkerContext(w, int(plan.block_start[w]), int(plan.block_start[w + 1]),
                          int(plan.halo_lo[w]), s.diag[plan.block_start[w]:plan.block_start[w + 1]])
            for w in range(p)]
    for c in ctxs:  # 1. scatter
        c.local_x = x[c.row_start:c.row_end].copy()
        c.local_y = np.zeros(c.row_end - c.row_start)
        c.stages.append("scatter")
        log.append((c.worker_id, "scatter"))
    for c in ctxs:  # 2. halo: every earlier worker ships its overlap with [halo_lo, row_start)
        halo = np.empty(c.row_start - c.halo_lo)
        for src in ctxs[:c.worker_id]:
            a, b = max(c.halo_lo, src.row_start), min(c.row_start, src.row_end)
            if a < b:
                assert "scatter" in src.stages
                halo[a - c.halo_lo:b - c.halo_lo] = src.local_x[a - src.row_start:b - src.row_start]
        c.halo_x = halo
        c.stages.append("halo")
        log.append((c.worker_id, "halo"))

    msg_val = np.empty(plan.conflict_count)
    messages: list = []
    mid_ptr, mid_col, mid_val = s.mid_ptr, s.mid_col.astype(np.int64), s.mid_val
    for c in ctxs:
        w, lo, hi = c.worker_id, c.row_start, c.row_end
        rows = np.arange(lo, hi, dtype=np.int64)
        # 3. diagonal
        c._add_stream(rows, c.local_diag * c._gather_x(rows))
        c.element_reads += hi - lo
        c.multiply_adds += hi - lo
        c.stages.append("diag")
        log.append((w, "diag"))
        # 4. safe entries [safe_start, mid_ptr[i+1]): row update then mirror, per element
        starts, ends = plan.safe_start[lo:hi], mid_ptr[lo + 1:hi + 1]
        ks = np.concatenate([np.arange(a, b) for a, b in zip(starts, ends)]) if hi > lo else \
            np.zeros(0, np.int64)
        ri = np.repeat(rows, ends - starts)
        cols, vals = mid_col[ks], mid_val[ks]
        xi = c._gather_x(ri)
        c._add_stream(*_interleave(ri, vals * c._gather_x(cols), cols, -vals * xi))
        c.element_reads += ks.size
        c.multiply_adds += 2 * ks.size
        c.stages.append("safe")
        log.append((w, "safe"))
        # 5. conflict entries [mid_ptr[i], safe_start): local row update, mirror shipped
        starts, ends = mid_ptr[lo:hi], plan.safe_start[lo:hi]
        ks = np.concatenate([np.arange(a, b) for a, b in zip(starts, ends)]) if hi > lo else \
            np.zeros(0, np.int64)
        ri = np.repeat(rows, ends - starts)
        cols, vals = mid_col[ks], mid_val[ks]
        c._add_stream(ri, vals * c._gather_x(cols))
        value = -vals * c._gather_x(ri)
        c0 = int(plan.conflict_ptr[w])
        assert c0 + ks.size == plan.conflict_ptr[w + 1], "conflict slots out of step with plan"
        msg_val[c0:c0 + ks.size] = value
        for q in range(ks.size):
            msg = AccumulationMessage(int(plan.conflict_target[c0 + q]), int(cols[q]),
                                      float(value[q]), w, int(ri[q]), int(cols[q]), c0 + q)
            c.outbox.append(msg)
            messages.append(msg)
        c.element_reads += ks.size
        c.multiply_adds += 2 * ks.size  # the local product plus the shipped one
        c.stages.append("conflict")
        log.append((w, "conflict"))
    for c in ctxs:  # message application, slot order per target
        t = c.worker_id
        slots = plan.apply_order[plan.apply_ptr[t]:plan.apply_ptr[t + 1]]
        assert (plan.conflict_target[slots] == t).all(), "message routed to wrong worker"
        c._add_stream(mid_col[plan.conflict_idx[slots]], msg_val[slots])
        c.stages.append("apply")
        log.append((t, "apply"))
    y = np.concatenate([c.local_y for c in ctxs]) if ctxs else np.zeros(0)
    log.append((0, "gather"))
    oi, oc = s.outer_row.astype(np.int64), s.outer_col.astype(np.int64)
    ov = s.outer_val
    np.add.at(y, *_interleave(oi, ov * x[oc], oc, -(ov * x[oi])))
    log.append((0, "outer"))
    return Pars3Trace(y=y, contexts=ctxs, messages=messages, stage_log=log,
                      coordinator_reads=int(s.outer_count),
                      coordinator_multiply_adds=2 * int(s.outer_count), outer_count=int(s.outer_count))
