"""The whole preprocessing chain on the GPU.

``prepare_gpu(m0, beta=None)`` is

    perm = rcm_order(pattern_from_sss(m0))
    m = permute_sss(m0, perm)
    bw = compute_bandwidth(m); beta = beta or default_beta(m.n, bw)
    s = split_bands(m, beta)

with every stage on the device (csrc/rcm.cu, csrc/prep_gpu.cu): the
skyline arrays are uploaded once, and only the results come back.  The
returned objects are the host-chain's bit for bit (tests/test_gpu_rcm.py
checks both chains, and the reference's SHA-256s for c2-c5).
``classify_conflicts_gpu`` / ``prepare_gpu(..., boundaries=...)`` run the
conflict classification (split.py:303-361) on the device too, on the
device-resident split.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .formats import SssMatrix
from .reorder import Permutation, _upload
from .split import BandSplit, default_beta

__all__ = ["prepare_gpu", "classify_conflicts_gpu"]

_CHUNK = 64 << 20  # first-touch slice per thread task


def _download(tensors, torch):
    """Device tensors -> fresh numpy arrays through page-locked DMA.

    ``.cpu()`` into pageable memory runs at ~2.2 GB/s on the B200 box: the
    driver stages through its own pinned buffer and every destination page
    faults in on one thread.  Here the destinations are first touched by a
    thread pool (numpy releases the GIL for the fill), page-locked in place
    with ``cudaHostRegister``, filled by one async copy each on the current
    stream, and unregistered (tools/prep_time.py measures each step).  If
    registration is refused the copy falls back to ``.cpu()``; the bytes are
    the same either way."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    outs = [np.empty(t.numel(), dtype=torch.empty(0, dtype=t.dtype).numpy().dtype)
            for t in tensors]
    jobs = [(o, i, min(i + _CHUNK // o.itemsize, o.size))
            for o in outs for i in range(0, o.size, max(1, _CHUNK // o.itemsize))]
    workers = max(1, min(16, len(os.sched_getaffinity(0))))
    with ThreadPoolExecutor(workers) as ex:
        list(ex.map(lambda j: j[0][j[1]:j[2]].fill(0), jobs))
    rt = torch.cuda.cudart()
    done = []
    try:
        for o, t in zip(outs, tensors):
            if o.nbytes == 0:
                continue
            if int(rt.cudaHostRegister(o.ctypes.data, o.nbytes, 0)) != 0:
                torch.from_numpy(o).copy_(t.reshape(-1))
                continue
            done.append(o)
            torch.from_numpy(o).copy_(t.reshape(-1), non_blocking=True)
        torch.cuda.current_stream().synchronize()
    finally:
        for o in done:
            rt.cudaHostUnregister(o.ctypes.data)
    return outs


def _classify_device(L, torch, dev, n, beta, mp, mc, boundaries, st):
    """PartitionPlan of a device-resident split (mp, mc: device tensors)."""
    from .split import PartitionPlan, StructuralError
    bs = np.array(boundaries, dtype=np.int64).ravel()
    p = bs.size - 1
    if p < 1 or bs[0] != 0 or bs[-1] != n:
        raise StructuralError("block_start must run from 0 to n over p blocks")
    sizes = np.diff(bs)
    if np.any(sizes < 1):
        raise StructuralError("every block must own at least one row")
    if sizes.max() - sizes.min() > 1:
        raise StructuralError("block sizes must differ by at most one row")
    k = _lib._c_i64()
    ro = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    ss = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    head = (n, _lib.ptr(mp), _lib.ptr(mc), p, _lib.ptr(bs), ctypes.byref(k), _lib.ptr(ro), _lib.ptr(ss))
    _lib.check(L.pars3_classify_conflicts_device(*head, None, None, None, None, None, None, st),
               "classify_conflicts_gpu")
    kk = int(k.value)
    ci = torch.empty(max(kk, 1), dtype=torch.int64, device=dev)
    ct = torch.empty(max(kk, 1), dtype=torch.int64, device=dev)
    ao = torch.empty(max(kk, 1), dtype=torch.int64, device=dev)
    cp = np.empty(p + 1, np.int64)
    ap = np.empty(p + 1, np.int64)
    hl = np.empty(p, np.int64)
    _lib.check(L.pars3_classify_conflicts_device(*head, _lib.ptr(ci), _lib.ptr(cp), _lib.ptr(ct),
                                                 _lib.ptr(ao), _lib.ptr(ap), _lib.ptr(hl), st),
               "classify_conflicts_gpu")
    h = _download((ro[:n], ss[:n], ci[:kk], ct[:kk], ao[:kk]), torch)
    return PartitionPlan(n=n, p=p, beta=int(beta), block_start=bs, row_owner=h[0], safe_start=h[1],
                         conflict_idx=h[2], conflict_ptr=cp, conflict_target=h[3], apply_order=h[4],
                         apply_ptr=ap, halo_lo=hl)


def classify_conflicts_gpu(s, boundaries, device="cuda"):
    """``classify_conflicts`` (split.py:303-361) computed on the GPU: the same
    PartitionPlan and ConflictReport as the host function, bit for bit."""
    from .device import require_cuda
    from .split import conflict_report
    torch = require_cuda()
    dev = torch.device(device)
    L = _lib.load()
    with torch.cuda.device(dev):
        mp = _upload(s.mid_ptr, np.int64, dev)
        mc = _upload(s.mid_col, np.int32, dev) if s.mid_col.size else torch.zeros(1, dtype=torch.int32, device=dev)
        plan = _classify_device(L, torch, dev, s.n, s.beta, mp, mc, boundaries, _lib.stream_ptr())
    return plan, conflict_report(s, plan)


def prepare_gpu(m0: SssMatrix, beta: int | None = None, device="cuda", boundaries=None, keep_device=False):
    """(perm, m, s, bandwidth) of the host chain, computed on the GPU.  With
    ``boundaries`` (a block partition, e.g. ``partition_rows(n, p)``) the
    conflict classification runs on the device-resident split as well and
    the result is (perm, m, s, bandwidth, plan).  ``keep_device``: the split's
    device copies stay attached to ``s`` until its first device plan is built
    (``prepare`` / ``spmv_pars3``), which then skips the upload of the split
    (pars3_plan_create_resident)."""
    from .device import require_cuda
    torch = require_cuda()
    dev = torch.device(device)
    L = _lib.load()
    n, nnz = m0.n, m0.nnz_offdiag
    with torch.cuda.device(dev):
        st = _lib.stream_ptr()
        rp = _upload(m0.row_ptr, np.int64, dev)
        ci = _upload(m0.col_ind, np.int32, dev)
        od = _upload(m0.off_diags, np.float64, dev)
        dg = _upload(m0.diags, np.float64, dev)
        fw = torch.empty(n, dtype=torch.int64, device=dev)
        _lib.check(L.pars3_rcm_order_lower_device(n, _lib.ptr(rp), _lib.ptr(ci), int(nnz),
                                                  _lib.ptr(fw), st), "prepare_gpu: rcm")
        rp2 = torch.empty(n + 1, dtype=torch.int64, device=dev)
        ci2 = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        od2 = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
        dg2 = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        _lib.check(L.pars3_permute_lower_device(n, _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(od),
                                                _lib.ptr(dg), _lib.ptr(fw), _lib.ptr(rp2),
                                                _lib.ptr(ci2), _lib.ptr(od2), _lib.ptr(dg2), st),
                   "prepare_gpu: permute")
        del rp, ci, od, dg
        bw = _lib._c_i64()
        _lib.check(L.pars3_bandwidth_device(n, _lib.ptr(rp2), _lib.ptr(ci2), ctypes.byref(bw), st),
                   "prepare_gpu: bandwidth")
        bw = int(bw.value)
        if beta is None:
            beta = default_beta(n, bw)
        mp = torch.empty(n + 1, dtype=torch.int64, device=dev)
        op = torch.empty(n + 1, dtype=torch.int64, device=dev)
        counts = np.zeros(2, dtype=np.int64)
        args = (n, _lib.ptr(rp2), _lib.ptr(ci2), _lib.ptr(od2), int(beta), _lib.ptr(mp), _lib.ptr(op))
        _lib.check(L.pars3_split_device(*args, None, None, None, None, None, _lib.ptr(counts), st),
                   "prepare_gpu: split")
        nm, no = int(counts[0]), int(counts[1])
        mc = torch.empty(max(nm, 1), dtype=torch.int32, device=dev)
        mv = torch.empty(max(nm, 1), dtype=torch.float64, device=dev)
        orow = torch.empty(max(no, 1), dtype=torch.int32, device=dev)
        ocol = torch.empty(max(no, 1), dtype=torch.int32, device=dev)
        oval = torch.empty(max(no, 1), dtype=torch.float64, device=dev)
        _lib.check(L.pars3_split_device(*args, _lib.ptr(mc), _lib.ptr(mv), _lib.ptr(orow),
                                        _lib.ptr(ocol), _lib.ptr(oval), _lib.ptr(counts), st),
                   "prepare_gpu: split")
        names, ts = zip(*(("fw", fw), ("rp", rp2), ("ci", ci2[:nnz]), ("od", od2[:nnz]),
                          ("dg", dg2[:n]), ("mp", mp), ("mc", mc[:nm]), ("mv", mv[:nm]),
                          ("orow", orow[:no]), ("ocol", ocol[:no]), ("oval", oval[:no])))
        plan = None
        if boundaries is not None:
            plan = _classify_device(L, torch, dev, n, beta, mp, mc, boundaries, st)
        h = dict(zip(names, _download(ts, torch)))
    perm = Permutation(h["fw"])
    m = SssMatrix._trusted(n, h["rp"], h["ci"], h["od"], h["dg"])
    s = BandSplit(n, int(beta), h["dg"], h["mp"], h["mc"], h["mv"], h["orow"], h["ocol"], h["oval"])
    if keep_device:
        from .device import _cache
        _cache(s)["resident_split"] = dict(mid_ptr=mp, mid_col=mc, mid_val=mv, outer_row=orow,
                                           outer_col=ocol, outer_val=oval)
    if boundaries is not None:
        return perm, m, s, bw, plan
    return perm, m, s, bw
