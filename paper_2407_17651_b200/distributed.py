"""Row-block sharding of the PARS3 product across ranks (one GPU per rank).

The reference runs its workers as threads over one shared x and y and keeps
the paper's MPI protocol only as a simulation (parallel.py:274-413,
PAPER.md:151, 197).  Here each rank owns the rows ``[lo, hi)`` of the
reference's own partition (``partition_rows(n, p)``, split.py:173-188) -- their
diagonal, middle and outer entries -- and one product is one exchange step:

1. **x halo** (predecessors -> successor): rank w receives
   ``x[halo_lo_w, lo_w)``, the columns below its block that its rows read.
   This is the paper's staged X chain, in the lower-storage direction
   (SPEC.md D16).
2. **local product** over the rank's extended index space
   ``[halo_lo_w, hi_w)``: own rows carry their entries, halo rows none, so
   ``y_ext`` holds the own rows' values and, in its halo part, the mirrors
   ``-a_ic * x_i`` bound for earlier blocks.
3. **accumulation** (successor -> predecessors): the halo part of ``y_ext``
   travels back and the owner adds it -- the reference's accumulation
   messages / ``MPI_Accumulate`` (parallel.py:96-113), as dense segments.

The halo here spans middle and outer entries (the reference's
``PartitionPlan.halo_lo`` covers the middle band only, split.py:341-345,
because its outer pass runs on worker 0).  The reference's
plan arrays are not altered.

Overlap: the rank's rows are split into BOUNDARY rows
(some stored column below ``lo``: they read the x halo and emit partials)
and INTERIOR rows (all columns in the own block).  Each part gets its own
device plan over the same extended index space, both accumulating into one
``y_ext`` (``pars3_plan_spmv_acc``); the interior product is enqueued right
after the halo exchange is started, so it runs while the halo is in flight,
and only the boundary product waits for it.  The interior plan carries the
diagonal; the boundary plan skips rows without entries
(``PARS3_PLAN_SKIP_EMPTY``).  With an RCM band the boundary is the first
~bandwidth rows of the block (c5 at 8 ranks: ~9 %).

Communication uses ``torch.distributed`` point-to-point ops
(``batch_isend_irecv``): NCCL over NVLink with device tensors, or gloo with
host staging for CPU tests.  The local products are GPU tile kernels; tests
may inject another local product (``local_factory``, called per part).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .split import BandSplit, PartitionPlan

__all__ = ["RankShard", "shard_for_rank", "split_shard", "exchange_schedule", "DistributedPars3",
           "PeerPars3", "emulate_ranks"]


@dataclass
class RankShard:
    """Rank w's rows in its extended index space ``[halo_lo, hi)``."""

    rank: int
    lo: int
    hi: int
    halo_lo: int
    # SSS arrays over n_ext = hi - halo_lo rows (halo rows empty)
    row_ptr: np.ndarray
    col_ind: np.ndarray
    off_diags: np.ndarray
    diags: np.ndarray

    @property
    def n_ext(self) -> int:
        return self.hi - self.halo_lo

    @property
    def own_off(self) -> int:
        return self.lo - self.halo_lo


def _rows_entries(s: BandSplit, lo: int, hi: int):
    """Merged (outer then middle) columns/values of rows [lo, hi), per row
    ascending, plus the per-row counts (the merge_splits order, split.py:144-170)."""
    orow = s.outer_row
    o0, o1 = np.searchsorted(orow, [lo, hi])
    ocount = np.bincount(orow[o0:o1] - lo, minlength=hi - lo)
    m0, m1 = int(s.mid_ptr[lo]), int(s.mid_ptr[hi])
    mcount = np.diff(s.mid_ptr[lo:hi + 1])
    rp = np.zeros(hi - lo + 1, dtype=np.int64)
    np.cumsum(ocount + mcount, out=rp[1:])
    col = np.empty(int(rp[-1]), dtype=np.int64)
    val = np.empty(int(rp[-1]), dtype=np.float64)
    optr = np.zeros(hi - lo + 1, dtype=np.int64)
    np.cumsum(ocount, out=optr[1:])
    rows_o = np.repeat(np.arange(hi - lo), ocount)
    dest_o = rp[rows_o] + (np.arange(o1 - o0) - optr[rows_o])
    rows_m = np.repeat(np.arange(hi - lo), mcount)
    dest_m = rp[rows_m] + ocount[rows_m] + (np.arange(m1 - m0) - (s.mid_ptr[lo:hi][rows_m] - m0))
    col[dest_o] = s.outer_col[o0:o1]
    val[dest_o] = s.outer_val[o0:o1]
    col[dest_m] = s.mid_col[m0:m1]
    val[dest_m] = s.mid_val[m0:m1]
    return rp, col, val


def shard_for_rank(s: BandSplit, plan: PartitionPlan, rank: int) -> RankShard:
    lo, hi = int(plan.block_start[rank]), int(plan.block_start[rank + 1])
    rp, col, val = _rows_entries(s, lo, hi)
    halo_lo = int(min(lo, col.min())) if col.size else lo
    own_off = lo - halo_lo
    n_ext = hi - halo_lo
    row_ptr = np.zeros(n_ext + 1, dtype=np.int64)
    row_ptr[own_off:] = rp
    diags = np.zeros(n_ext)
    diags[own_off:] = s.diag[lo:hi]
    return RankShard(rank, lo, hi, halo_lo, row_ptr, (col - halo_lo).astype(np.int32), val, diags)


def split_shard(sh: RankShard):
    """(interior, boundary) parts of a shard over the same extended space:
    boundary rows have a stored column below ``lo`` (the halo), interior rows
    do not.  The interior part keeps the diagonal, the boundary part has a
    zero diagonal; ``boundary`` is None when no row reads the halo."""
    counts = np.diff(sh.row_ptr)
    rows = np.repeat(np.arange(sh.n_ext, dtype=np.int64), counts)
    is_b = np.zeros(sh.n_ext, dtype=bool)
    if sh.col_ind.size:
        halo_rows = np.unique(rows[sh.col_ind < sh.own_off])
        is_b[halo_rows] = True
    if not is_b.any():
        return sh, None

    def part(keep_row, diags):
        keep = keep_row[rows]
        c = np.where(keep_row, counts, 0)
        rp = np.zeros(sh.n_ext + 1, dtype=np.int64)
        np.cumsum(c, out=rp[1:])
        return RankShard(sh.rank, sh.lo, sh.hi, sh.halo_lo, rp, sh.col_ind[keep],
                         sh.off_diags[keep], diags)

    interior = part(~is_b, sh.diags)
    boundary = part(is_b, np.zeros(sh.n_ext))
    return interior, boundary


def exchange_schedule(s: BandSplit, plan: PartitionPlan):
    """Every rank's halo range, and the (src, dst, a, b) segments: rank dst
    needs x[a, b) from owner src (and returns y partials for the same range)."""
    p = plan.p
    halos = []
    for w in range(p):
        lo, hi = int(plan.block_start[w]), int(plan.block_start[w + 1])
        m0, m1 = int(s.mid_ptr[lo]), int(s.mid_ptr[hi])
        cmin = lo
        if m1 > m0:
            cmin = min(cmin, int(s.mid_col[m0:m1].min()))
        o0, o1 = np.searchsorted(s.outer_row, [lo, hi])
        if o1 > o0:
            cmin = min(cmin, int(s.outer_col[o0:o1].min()))
        halos.append(cmin)
    segs = []
    bs = plan.block_start
    for dst in range(p):
        a0, b0 = halos[dst], int(bs[dst])
        for src in range(dst):
            a, b = max(a0, int(bs[src])), min(b0, int(bs[src + 1]))
            if a < b:
                segs.append((src, dst, a, b))
    return halos, segs


class DistributedPars3:
    """One rank's operator: ``y_own = (A x)[lo:hi]`` from ``x_own = x[lo:hi]``.

    ``plan.p`` must equal the world size; rank r owns block r.  With
    ``local_factory`` (tests) each local product is ``local_factory(part)``
    returning a callable ``y_ext = f(x_ext)`` on host arrays; otherwise the
    GPU tile kernel runs it on the rank's device.  ``overlap=False`` runs one
    plan over all the rank's rows after the halo has arrived.
    """

    def __init__(self, s: BandSplit, plan: PartitionPlan, group=None, local_factory=None,
                 device=None, options=None, overlap=True, max_ctas=0):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.group = group
        self.rank = dist.get_rank(group)
        world = dist.get_world_size(group)
        if plan.p != world:
            raise ValueError(f"plan has {plan.p} blocks but the group has {world} ranks")
        if plan.n != s.n or plan.beta != s.beta:
            raise ValueError(f"plan (n={plan.n}, beta={plan.beta}) does not match "
                             f"split (n={s.n}, beta={s.beta})")
        self.shard = shard_for_rank(s, plan, self.rank)
        self.halos, self.segs = exchange_schedule(s, plan)
        assert self.halos[self.rank] == self.shard.halo_lo
        self.staged = dist.get_backend(group) == "gloo"
        sh = self.shard
        self.overlap = bool(overlap)
        parts = split_shard(sh) if overlap else (sh, None)
        self.interior_shard, self.boundary_shard = parts
        if local_factory is not None:
            self._local = [local_factory(p) if p is not None else None for p in parts]
            self.device = torch.device("cpu")
            self._on_host = True
            self.ops = []
        else:
            from ._lib import PLAN_SKIP_EMPTY
            from .device import Pars3Operator
            self.device = torch.device(device) if device is not None else torch.device(
                "cuda", torch.cuda.current_device())
            base = tuple(options or ()) + (0, 0, 0, -1, 0, 0, 0)[len(options or ()):]
            e = np.zeros(0, np.int32)

            def make(p, flags, ctas):
                o = base[:5] + (base[5] | flags, ctas or base[6])
                return Pars3Operator(p.n_ext, max(1, p.n_ext), p.diags, p.row_ptr, p.col_ind,
                                     p.off_diags, e, e, np.zeros(0), device=self.device, options=o)
            # the interior kernel may leave SMs to the concurrent exchange
            self.ops = [make(parts[0], 0, max_ctas)]
            if parts[1] is not None:
                self.ops.append(make(parts[1], PLAN_SKIP_EMPTY, 0))
            self._on_host = False
        self._op = self.ops[0] if self.ops else None  # the dominant (interior) product
        t = torch.float64
        self.x_ext = torch.zeros(sh.n_ext, dtype=t, device=self.device)
        self.y_ext = torch.zeros(sh.n_ext, dtype=t, device=self.device)
        self._inbox = {(dst, a): torch.empty(b - a, dtype=t, device=self.device)
                       for (src, dst, a, b) in self.segs if src == self.rank}

    # -- communication --------------------------------------------------
    def _start(self, ops):
        """Post point-to-point ops; returns what _finish waits on.  NCCL ops
        run on NCCL's stream after the work already enqueued; gloo stages
        device tensors through the host and completes here."""
        if not ops:
            return None
        dist = self.dist
        if self.staged and not self._on_host:
            host_ops, copies = [], []
            for kind, tensor, peer in ops:
                h = tensor.detach().cpu()
                host_ops.append((kind, h, peer))
                copies.append((tensor, h, kind))
            reqs = dist.batch_isend_irecv([dist.P2POp(k, h, peer, self.group)
                                           for k, h, peer in host_ops])
            for r in reqs:
                r.wait()
            for tensor, h, kind in copies:
                if kind is dist.irecv:
                    tensor.copy_(h)
            return None
        return dist.batch_isend_irecv([dist.P2POp(k, tns, peer, self.group)
                                       for k, tns, peer in ops])

    @staticmethod
    def _finish(reqs):
        """Make the current stream wait for the posted ops (once per post)."""
        for r in reqs or ():
            r.wait()

    def _peer(self, r):
        return self.dist.get_global_rank(self.group, r) if self.group is not None else r

    def _local_product(self, k):
        """Local part k (0 interior, 1 boundary) accumulated into y_ext."""
        if self._on_host:
            f = self._local[k]
            if f is not None:
                self.y_ext += self.torch.from_numpy(np.asarray(f(self.x_ext.numpy())))
        elif k < len(self.ops):
            self.ops[k].matvec(self.x_ext, self.y_ext, accumulate=True)

    def matvec(self, x_own):
        """y_own for this rank's block; x_own: length hi - lo (this rank's x)."""
        sh, dist = self.shard, self.dist
        nown = sh.hi - sh.lo
        if x_own.shape[0] != nown:
            raise ValueError(f"x block must have {nown} entries, got {x_own.shape[0]}")
        if x_own.data_ptr() != self.x_ext[sh.own_off:].data_ptr():
            self.x_ext[sh.own_off:] = x_own.to(self.device)
        self.y_ext.zero_()
        # 1. x halo: owners send slices of their block, consumers receive
        ops = []
        for (src, dst, a, b) in self.segs:
            if src == self.rank:
                ops.append((dist.isend, self.x_ext[sh.own_off + (a - sh.lo):
                                                   sh.own_off + (b - sh.lo)].contiguous(),
                            self._peer(dst)))
            elif dst == self.rank:
                ops.append((dist.irecv, self.x_ext[a - sh.halo_lo:b - sh.halo_lo], self._peer(src)))
        reqs = self._start(ops)
        # 2. interior rows while the halo is in flight, then the boundary rows
        #    (without overlap the single product waits for the halo)
        if not self.overlap:
            self._finish(reqs)
            reqs = None
        self._local_product(0)
        self._finish(reqs)
        self._local_product(1)
        # 3. accumulation messages back to the owners, added in source order
        ops = []
        for (src, dst, a, b) in self.segs:
            if dst == self.rank:
                ops.append((dist.isend, self.y_ext[a - sh.halo_lo:b - sh.halo_lo].contiguous(),
                            self._peer(src)))
            elif src == self.rank:
                ops.append((dist.irecv, self._inbox[(dst, a)], self._peer(dst)))
        self._finish(self._start(ops))
        y_own = self.y_ext[sh.own_off:].clone()
        for (src, dst, a, b) in self.segs:
            if src == self.rank:
                y_own[a - sh.lo:b - sh.lo] += self._inbox[(dst, a)]
        return y_own

    def x_view(self):
        """This rank's block of x inside the extended buffer: writing x here
        (e.g. the next iterate of a solver) skips matvec's copy."""
        return self.x_ext[self.shard.own_off:]


class _IpcVector:
    """A float64 device vector in its own cudaMalloc block, exportable to
    other processes (CUDA IPC), viewed as a torch tensor."""

    def __init__(self, n, device):
        import ctypes

        import torch

        from . import _lib
        self._L = _lib.load()
        self.n = int(n)
        p = ctypes.c_void_p()
        with torch.cuda.device(device):
            _lib.check(self._L.pars3_ipc_alloc(8 * max(1, self.n), ctypes.byref(p)), "ipc_alloc")
        self.ptr = p.value
        self.device = device
        self.__cuda_array_interface__ = {"shape": (self.n,), "typestr": "<f8",
                                         "data": (self.ptr, False), "version": 3}
        self.tensor = torch.as_tensor(self, device=device)

    def handle(self) -> bytes:
        import ctypes

        from . import _lib
        buf = (ctypes.c_uint8 * 64)()
        _lib.check(self._L.pars3_ipc_handle(ctypes.c_void_p(self.ptr), buf), "ipc_handle")
        return bytes(buf)

    def close(self):
        if getattr(self, "ptr", None):
            self.tensor = None
            self._L.pars3_ipc_free(ctypes_vp(self.ptr))
            self.ptr = None


def ctypes_vp(v):
    import ctypes
    return ctypes.c_void_p(v)


class PeerPars3:
    """One rank's operator in PEER mode: ``y_own = (A x)[lo:hi]`` with the
    exchange inside the kernel.

    Every rank exports (CUDA IPC) its x block and an inbox for its rows.
    Its single plan covers the extended range [halo_lo, hi); windows are cut
    at block boundaries, and the kernel reads an earlier rank's x straight
    from that rank's buffer and reduces the mirror sums of its rows straight
    into that rank's inbox (``pars3_plan_set_peers``), over NVLink between
    GPUs.  A step is: write x, zero y, barrier (every x written, every inbox
    drained), product, barrier (every reduction landed), y += inbox, drain.
    The barriers are one-element all-reduces on the current stream (NCCL:
    device-side, no host sync) or host barriers (gloo tests)."""

    def __init__(self, s: BandSplit, plan: PartitionPlan, group=None, device=None, options=None):
        import ctypes

        import torch
        import torch.distributed as dist

        from . import _lib
        from .device import Pars3Operator
        self.torch, self.dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        world = dist.get_world_size(group)
        if plan.p != world:
            raise ValueError(f"plan has {plan.p} blocks but the group has {world} ranks")
        if world > 8:
            raise ValueError("peer mode supports up to 8 ranks (one NVLink domain)")
        if plan.n != s.n or plan.beta != s.beta:
            raise ValueError(f"plan (n={plan.n}, beta={plan.beta}) does not match "
                             f"split (n={s.n}, beta={s.beta})")
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.staged = dist.get_backend(group) == "gloo"
        sh = self.shard = shard_for_rank(s, plan, self.rank)
        nown = sh.hi - sh.lo
        # x block and inbox in ONE allocation with one IPC handle: small
        # cudaMallocs share a VA chunk, and a peer's mapping of one handle
        # covers only that allocation
        self._shared = _IpcVector(2 * nown, self.device)
        self._x = self._shared.tensor[:nown]
        self._in = self._shared.tensor[nown:]
        self._shared.tensor.zero_()
        # the kernel accumulates the own rows into y_acc (zero between
        # products); the step epilogue writes y_own = y_acc + inbox
        self.y_acc = torch.zeros(nown, dtype=torch.float64, device=self.device)
        self.y_own = torch.zeros(nown, dtype=torch.float64, device=self.device)
        torch.cuda.synchronize(self.device)
        handles = [None] * world
        dist.all_gather_object(handles, (self._shared.handle(), nown), group=group)
        L = _lib.load()
        self._opened = []
        xp, ip = [], []
        for r, (h, nr) in enumerate(handles):
            if r == self.rank:
                base = self._shared.ptr
            else:
                q = ctypes.c_void_p()
                buf = (ctypes.c_uint8 * 64).from_buffer_copy(h)
                with torch.cuda.device(self.device):
                    _lib.check(L.pars3_ipc_open(buf, ctypes.byref(q)), "ipc_open")
                self._opened.append(q.value)
                base = q.value
            xp.append(base)
            ip.append(base + 8 * int(nr))
        # local cut points: every block boundary inside [halo_lo, hi)
        bs = np.asarray(plan.block_start, dtype=np.int64)
        cuts = [0] + [int(b - sh.halo_lo) for b in bs[1:-1] if sh.halo_lo < b < sh.hi] + [sh.n_ext]
        base = tuple(options or ()) + (0, 0, 0, -1, 0, 0, 0)[len(options or ()):]
        o = base[:5] + (base[5] | _lib.PLAN_CUT_BLOCKS, base[6])
        e = np.zeros(0, np.int32)
        self._op = Pars3Operator(sh.n_ext, max(1, sh.n_ext), sh.diags, sh.row_ptr, sh.col_ind,
                                 sh.off_diags, e, e, np.zeros(0), p=len(cuts) - 1,
                                 block_start=np.asarray(cuts, dtype=np.int64), device=self.device,
                                 options=o)
        self.ops = [self._op]
        xa = (ctypes.c_uint64 * world)(*xp)
        ia = (ctypes.c_uint64 * world)(*ip)
        bsa = np.ascontiguousarray(bs)
        _lib.check(L.pars3_plan_set_peers(self._op._handle, world, self.rank, sh.halo_lo,
                                          _lib.ptr(bsa), xa, ia), "plan_set_peers")
        # the kernel addresses x / y by local index: own block at own_off
        self._x_local = self._shared.ptr - 8 * sh.own_off
        self._y_local = self.y_acc.data_ptr() - 8 * sh.own_off
        self._one = torch.zeros(1, dtype=torch.float64, device=self.device)

    def x_view(self):
        """This rank's x block in the shared buffer (write x here to skip a copy)."""
        return self._x

    def _barrier(self):
        if self.staged:
            self.torch.cuda.synchronize(self.device)
            self.dist.barrier(group=self.group)
        else:
            self.dist.all_reduce(self._one, group=self.group)

    def matvec(self, x_own, dot=None):
        """y_own = (A x)[lo:hi]; with ``dot`` (a 1-element device tensor) also
        its local <y_own, y_own>, from the same epilogue pass."""
        from . import _lib
        sh = self.shard
        nown = sh.hi - sh.lo
        if x_own.shape[0] != nown:
            raise ValueError(f"x block must have {nown} entries, got {x_own.shape[0]}")
        xb = self._x
        if x_own.data_ptr() != xb.data_ptr():
            xb.copy_(x_own)
        self._barrier()  # every rank's x is written and its inbox drained
        L = self._op._L
        _lib.check(L.pars3_plan_spmv_acc(self._op._handle, self._x_local, self._y_local,
                                         _lib.stream_ptr()), "pars3_plan_spmv")
        self._barrier()  # every mirror reduction into an inbox has landed
        _lib.check(L.pars3_peer_finish(nown, _lib.ptr(self.y_acc), _lib.ptr(self._in),
                                       _lib.ptr(self.y_own), _lib.ptr(dot) if dot is not None else None,
                                       _lib.stream_ptr()), "pars3_peer_finish")
        return self.y_own

    def local_product(self):
        """The rank's kernel alone (no barriers; y accumulates): for timing."""
        from . import _lib
        _lib.check(self._op._L.pars3_plan_spmv_acc(self._op._handle, self._x_local, self._y_local,
                                                   _lib.stream_ptr()), "pars3_plan_spmv")

    def close(self):
        from . import _lib
        L = _lib.load()
        self.torch.cuda.synchronize(self.device)
        for q in self._opened:
            L.pars3_ipc_close(ctypes_vp(q))
        self._opened = []
        self._op.close()


def emulate_ranks(s: BandSplit, plan: PartitionPlan, x, make_local, overlap=False):
    """Run the p-rank protocol sequentially in one process: the same shards,
    schedule and data movement as DistributedPars3, with the exchanges as
    direct copies.  ``make_local(shard, boundary)`` returns ``y_ext =
    f(x_ext)`` (for the GPU path: a tile-kernel operator on the rank's
    extended space); with ``overlap`` each rank's product is the sum of its
    interior and boundary parts (split_shard).  Returns y as a torch tensor
    on ``x``'s device."""
    import torch
    p = plan.p
    shards = [shard_for_rank(s, plan, w) for w in range(p)]
    halos, segs = exchange_schedule(s, plan)
    def make(sh):
        if not overlap:
            return make_local(sh, False)
        inner, bnd = split_shard(sh)
        fi = make_local(inner, False)
        if bnd is None:
            return fi
        fb = make_local(bnd, True)
        return lambda xe: fi(xe) + fb(xe)

    local = [make(sh) for sh in shards]
    x = torch.as_tensor(x, dtype=torch.float64)
    x_ext = []
    for sh in shards:
        xe = torch.zeros(sh.n_ext, dtype=torch.float64, device=x.device)
        xe[sh.own_off:] = x[sh.lo:sh.hi]
        x_ext.append(xe)
    for (src, dst, a, b) in segs:  # 1. x halo
        sd, ss = shards[dst], shards[src]
        x_ext[dst][a - sd.halo_lo:b - sd.halo_lo] = x_ext[src][ss.own_off + (a - ss.lo):
                                                               ss.own_off + (b - ss.lo)]
    y_ext = [local[w](x_ext[w]) for w in range(p)]  # 2. local products
    y = torch.cat([y_ext[w][shards[w].own_off:] for w in range(p)])
    for (src, dst, a, b) in segs:  # 3. accumulation, in the same order as the ranks
        sd = shards[dst]
        y[a:b] += y_ext[dst][a - sd.halo_lo:b - sd.halo_lo]
    return y
