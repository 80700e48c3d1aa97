"""The multi-rank protocol on CPU: world sizes 2 and 3 over gloo.

Each rank holds the reference's block of rows (partition_rows), exchanges
the x halo and the mirror partials with torch.distributed point-to-point ops,
and the gathered blocks must equal the serial product (1e-12).  The local
product is injected as the oracle's serial kernel on the rank's extended
index space (the GPU tile kernel is exercised by the -m gpu emulation test),
so what runs here is the product's own sharding, schedule and exchange.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _case(name):
    import sys
    sys.path.insert(0, ROOT)
    import paper_2407_17651_b200 as P
    from paper_2407_17651_b200 import generators as G
    g = {"band": lambda: G.random_band(3000, 120, 6, 0.02, seed_struct=1, seed_perm=2, seed_val=3),
         "stencil": lambda: G.stencil27(12, seed_val=4, alpha=0.5),
         "rmat": lambda: G.rmat(11, 8, seed_struct=5, seed_perm=6, seed_val=7)}[name]()
    m0 = P.SssMatrix(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    m = P.permute_sss(m0, P.rcm_order(P.pattern_from_sss(m0)))
    return m


def _worker(rank, world, port, name, beta, overlap, out):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2407_17651_b200 as P
        from oracle import oracle as O
        from paper_2407_17651_b200.distributed import DistributedPars3
        m = _case(name)
        s = P.split_bands(m, beta)
        plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, world))

        def local(sh):
            return lambda xe: O.spmv_serial(sh.row_ptr, sh.col_ind, sh.off_diags, sh.diags, xe)

        op = DistributedPars3(s, plan, local_factory=local, overlap=overlap)
        x = np.random.default_rng(9).uniform(-1, 1, m.n)
        lo, hi = int(plan.block_start[rank]), int(plan.block_start[rank + 1])
        y_own = op.matvec(torch.from_numpy(x[lo:hi].copy()))
        y_own2 = op.matvec(torch.from_numpy(x[lo:hi].copy()))  # reusable buffers
        assert torch.equal(y_own, y_own2)
        sizes = np.diff(plan.block_start)
        width = int(sizes.max())
        padded = torch.zeros(width, dtype=torch.float64)
        padded[:y_own.shape[0]] = y_own
        parts = [torch.zeros(width, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, padded)
        if rank == 0:
            y = torch.cat([parts[r][:int(sizes[r])] for r in range(world)]).numpy()
            ref = O.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
            out.put(float(np.max(np.abs(y - ref)) / max(1.0, float(np.max(np.abs(ref))))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,overlap", [(2, True), (3, True), (2, False)])
@pytest.mark.parametrize("name,beta", [("band", 8), ("band", 4000), ("stencil", 20), ("rmat", 8)])
def test_gloo_protocol_matches_serial(world, overlap, name, beta):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, beta, overlap, out))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    err = out.get(timeout=5)
    assert err <= 1e-12, err


def test_schedule_and_shards_cover_the_matrix():
    import paper_2407_17651_b200 as P
    from paper_2407_17651_b200.distributed import exchange_schedule, shard_for_rank
    m = _case("rmat")
    s = P.split_bands(m, 8)
    for p in (1, 2, 5):
        plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, p))
        halos, segs = exchange_schedule(s, plan)
        total = 0
        for w in range(p):
            sh = shard_for_rank(s, plan, w)
            assert sh.halo_lo == halos[w] <= sh.lo
            assert sh.row_ptr[sh.own_off] == 0 and sh.row_ptr[-1] == sh.col_ind.size
            total += sh.col_ind.size
            # every halo column range is covered by segments from earlier ranks
            need = sh.lo - sh.halo_lo
            got = sum(b - a for (src, dst, a, b) in segs if dst == w)
            assert got == need and all(src < dst for (src, dst, a, b) in segs)
        assert total == m.nnz_offdiag


def test_split_shard_partitions_rows():
    """Interior and boundary parts cover the shard's entries exactly once;
    boundary rows are exactly the rows reading the halo; the diagonal stays
    with the interior part."""
    import paper_2407_17651_b200 as P
    from paper_2407_17651_b200.distributed import shard_for_rank, split_shard
    m = _case("stencil")
    s = P.split_bands(m, 20)
    plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, 3))
    for w in range(3):
        sh = shard_for_rank(s, plan, w)
        inner, bnd = split_shard(sh)
        if w == 0:
            assert bnd is None and inner is sh
            continue
        assert inner.col_ind.size + bnd.col_ind.size == sh.col_ind.size
        assert np.array_equal(inner.diags, sh.diags) and not bnd.diags.any()
        assert (inner.col_ind >= sh.own_off).all()
        for r in range(sh.n_ext):
            cols = sh.col_ind[sh.row_ptr[r]:sh.row_ptr[r + 1]]
            b = bnd.col_ind[bnd.row_ptr[r]:bnd.row_ptr[r + 1]]
            i = inner.col_ind[inner.row_ptr[r]:inner.row_ptr[r + 1]]
            if cols.size and cols.min() < sh.own_off:
                assert np.array_equal(b, cols) and i.size == 0
            else:
                assert np.array_equal(i, cols) and b.size == 0
