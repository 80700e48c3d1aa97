"""Peer-mode multi-rank product (PeerPars3): two and three processes share
the one GPU through CUDA IPC (the same code maps a peer GPU's buffers over
NVLink on a multi-GPU box).  Each rank's kernel reads earlier ranks' x and
reduces their rows' mirror sums into their inboxes directly; the barriers
are host-side (gloo), so no kernel ever waits on another process's kernel.
The gathered y must equal the oracle's serial product (1e-12)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, name, beta, out):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2407_17651_b200 as P
        from oracle import oracle as O
        from paper_2407_17651_b200 import generators as G
        from paper_2407_17651_b200.distributed import PeerPars3
        g = {"stencil": lambda: G.stencil27(24, seed_val=4, alpha=0.5),
             "band": lambda: G.random_band(30000, 400, 8, 0.02, seed_struct=1, seed_perm=2,
                                           seed_val=3),
             "rmat": lambda: G.rmat(13, 8, seed_struct=5, seed_perm=6, seed_val=7)}[name]()
        m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
        m = P.permute_sss(m0, P.rcm_order(P.pattern_from_sss(m0)))
        s = P.split_bands(m, beta)
        plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, world))
        op = PeerPars3(s, plan)
        x = G.make_x(m.n, 9)
        lo, hi = int(plan.block_start[rank]), int(plan.block_start[rank + 1])
        xb = torch.from_numpy(x[lo:hi].copy()).cuda()
        y1 = op.matvec(xb).clone()
        op.x_view().copy_(xb)          # the zero-copy entry: x written in place
        y2 = op.matvec(op.x_view()).clone()
        d = torch.zeros(1, dtype=torch.float64, device="cuda")
        y3 = op.matvec(xb, dot=d)  # the fused epilogue's local <y, y>
        torch.cuda.synchronize()
        assert abs(float(d) - float(y3 @ y3)) <= 1e-12 * max(1.0, float(y3 @ y3))
        assert torch.equal(y3, y1) or float((y3 - y1).abs().max()) <= 1e-13
        sizes = np.diff(plan.block_start)
        width = int(sizes.max())
        for yk in (y1, y2):
            pad = torch.zeros(width, dtype=torch.float64)
            pad[:hi - lo] = yk.cpu()
            parts = [torch.zeros(width, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(parts, pad)
            if rank == 0:
                y = torch.cat([parts[r][:int(sizes[r])] for r in range(world)]).numpy()
                ref = O.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
                out.put(float(np.max(np.abs(y - ref)) / max(1.0, float(np.max(np.abs(ref))))))
        op.close()
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name,beta", [("stencil", 50), ("band", 30), ("rmat", 8)])
def test_peer_mode_matches_serial(world, name, beta):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, beta, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    for _ in range(2):
        err = out.get(timeout=5)
        assert err <= 1e-12, err


@pytest.mark.parametrize("p", [2, 3, 8])
def test_peer_kernels_emulated_in_one_process(p, oracle):
    """The peer-mode kernels of p ranks run one after another in one process
    (their x blocks and inboxes are ordinary device buffers), including
    windows cut at odd block boundaries and list-mode tiles."""
    import ctypes

    import torch

    import paper_2407_17651_b200 as P
    from paper_2407_17651_b200 import _lib
    from paper_2407_17651_b200 import generators as G
    from paper_2407_17651_b200.device import Pars3Operator
    from paper_2407_17651_b200.distributed import shard_for_rank
    L = _lib.load()
    for g, beta in ((G.stencil27(24, seed_val=4, alpha=0.5), 50),
                    (G.rmat(12, 8, seed_struct=3, seed_perm=4, seed_val=5), 8)):
        m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
        m = P.permute_sss(m0, P.rcm_order(P.pattern_from_sss(m0)))
        s = P.split_bands(m, beta)
        plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, p))
        x = G.make_x(m.n, 9)
        bs = np.asarray(plan.block_start, dtype=np.int64)
        # each rank's x block is its own allocation with nothing mapped before it
        xb = [torch.from_numpy(x[bs[r]:bs[r + 1]].copy()).cuda() for r in range(p)]
        inbox = [torch.zeros(int(bs[r + 1] - bs[r]), dtype=torch.float64, device="cuda")
                 for r in range(p)]
        ys = [torch.zeros_like(inbox[r]) for r in range(p)]
        xa = (ctypes.c_uint64 * p)(*[t.data_ptr() for t in xb])
        ia = (ctypes.c_uint64 * p)(*[t.data_ptr() for t in inbox])
        for w in range(p):
            sh = shard_for_rank(s, plan, w)
            cuts = [0] + [int(b - sh.halo_lo) for b in bs[1:-1] if sh.halo_lo < b < sh.hi] + [sh.n_ext]
            e = np.zeros(0, np.int32)
            op = Pars3Operator(sh.n_ext, max(1, sh.n_ext), sh.diags, sh.row_ptr, sh.col_ind,
                               sh.off_diags, e, e, np.zeros(0), p=len(cuts) - 1,
                               block_start=np.asarray(cuts, np.int64),
                               options=(0, 0, 0, -1, 0, _lib.PLAN_CUT_BLOCKS, 0))
            _lib.check(L.pars3_plan_set_peers(op._handle, p, w, sh.halo_lo, _lib.ptr(bs), xa, ia))
            _lib.check(L.pars3_plan_spmv_acc(op._handle, xb[w].data_ptr() - 8 * sh.own_off,
                                             ys[w].data_ptr() - 8 * sh.own_off, _lib.stream_ptr()))
            torch.cuda.synchronize()
            op.close()
        y = torch.cat([ys[r] + inbox[r] for r in range(p)]).cpu().numpy()
        ref = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
        assert float(np.max(np.abs(y - ref)) / max(1.0, float(np.max(np.abs(ref))))) <= 1e-12, (g.name, p)


def test_set_peers_validation(lib_built):
    import ctypes

    import torch

    from paper_2407_17651_b200 import _lib
    from paper_2407_17651_b200.device import Pars3Operator
    e = np.zeros(0, np.int32)
    op = Pars3Operator(4, 4, np.zeros(4), np.zeros(5, np.int64), e, np.zeros(0), e, e, np.zeros(0))
    L = _lib.load()
    a = (ctypes.c_uint64 * 2)(1, 2)
    bs = np.array([0, 2, 4], dtype=np.int64)
    assert L.pars3_plan_set_peers(op._handle, 9, 0, 0, _lib.ptr(bs), a, a) == _lib.PARS3_ERR_ARG
    assert L.pars3_plan_set_peers(op._handle, 2, 2, 0, _lib.ptr(bs), a, a) == _lib.PARS3_ERR_ARG
    assert L.pars3_plan_set_peers(op._handle, 2, 1, 3, _lib.ptr(bs), a, a) == _lib.PARS3_ERR_ARG
    assert L.pars3_plan_set_peers(op._handle, 0, 0, 0, None, None, None) == _lib.PARS3_OK
    torch.cuda.synchronize()
