"""Small-config product timing (c2: 1000 back-to-back SpMVs, L2-resident):
plain launches vs one CUDA graph of 100 products, for several tile sizes.
Usage: python tools/small_config.py c2 [tile_rows ...]"""
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2407_17651_b200.device import Pars3Operator  # noqa: E402

cfg = sys.argv[1]
tiles = [int(t) for t in sys.argv[2:]] or [0]
m, s, bw, beta, x = bench.build_problem(cfg)
xd = torch.from_numpy(x).cuda()
y = torch.empty_like(xd)
B = bench.algorithmic_bytes(m.n, m.nnz_offdiag)
for tr in tiles:
    op = Pars3Operator(s.n, s.beta, s.diag, s.mid_ptr, s.mid_col, s.mid_val, s.outer_row,
                       s.outer_col, s.outer_val, options=(tr,))
    for _ in range(10):
        op.matvec(xd, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(1000):
        op.matvec(xd, y)
    e1.record()
    torch.cuda.synchronize()
    plain = e0.elapsed_time(e1) / 1000
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        op.matvec(xd, y)
        with torch.cuda.graph(g, stream=st):
            for _ in range(100):
                op.matvec(xd, y)
    torch.cuda.current_stream().wait_stream(st)
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    graphed = e0.elapsed_time(e1) / 1000
    print(f"{cfg} tile_rows={tr or 1024}: plain {plain * 1e3:.1f} us ({B / plain / 1e6:.0f} GB/s)  "
          f"graph {graphed * 1e3:.1f} us ({B / graphed / 1e6:.0f} GB/s)  {op.stats()}", flush=True)
