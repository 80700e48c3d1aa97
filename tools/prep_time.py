import sys, time, os
# Transfer-path timings for the GPU preprocessing chain (pageable, pinned,
# registered numpy, and pipeline._download); run under gpurun: python tools/prep_time.py c5
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2407_17651_b200 as P
from paper_2407_17651_b200 import generators as G
from paper_2407_17651_b200.reorder import _upload
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
g = G.make_config(cfg)
m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
from paper_2407_17651_b200.pipeline import prepare_gpu
torch.cuda.init(); torch.empty(1, device="cuda")
for rep in range(2):
    torch.cuda.synchronize(); t = time.time(); prepare_gpu(m0); torch.cuda.synchronize()
    print(f"prepare_gpu total {time.time()-t:.3f}s", flush=True)
dev = torch.device("cuda")
arrs = [(m0.row_ptr, np.int64), (m0.col_ind, np.int32), (m0.off_diags, np.float64), (m0.diags, np.float64)]
torch.cuda.synchronize(); t = time.time()
ds = [_upload(a, dt, dev) for a, dt in arrs]; torch.cuda.synchronize()
tot = sum(d.numel() * d.element_size() for d in ds)
print(f"upload pageable {time.time()-t:.3f}s {tot/1e9:.2f} GB", flush=True)
t = time.time(); h = [d.cpu().numpy() for d in ds]; print(f"download pageable .cpu() {time.time()-t:.3f}s", flush=True)
del h
t = time.time()
hs = [torch.empty(d.shape, dtype=d.dtype, pin_memory=True) for d in ds]
t1 = time.time()
for hh, d in zip(hs, ds): hh.copy_(d, non_blocking=True)
torch.cuda.synchronize(); t2 = time.time()
print(f"download pinned alloc {t1-t:.3f}s copy {t2-t1:.3f}s", flush=True)
t = time.time()
for a, dt in arrs:
    a = np.ascontiguousarray(a, dtype=dt)
    hp = torch.empty(a.shape, dtype=torch.from_numpy(a[:1]).dtype, pin_memory=True)
    hp.numpy()[:] = a
    hp.to(dev, non_blocking=True)
torch.cuda.synchronize(); print(f"upload via pinned staging (alloc+memcpy+copy) {time.time()-t:.3f}s", flush=True)
# registered numpy destination
cud = torch.cuda.cudart()
t = time.time()
out = [np.empty(d.numel(), dtype=torch.empty(0, dtype=d.dtype).numpy().dtype) for d in ds]
t0 = time.time()
for o in out:
    r = cud.cudaHostRegister(o.ctypes.data, o.nbytes, 0)
t1 = time.time()
for o, d in zip(out, ds):
    torch.from_numpy(o).copy_(d, non_blocking=True)
torch.cuda.synchronize(); t2 = time.time()
for o in out: cud.cudaHostUnregister(o.ctypes.data)
t3 = time.time()
print(f"download registered numpy: register {t1-t0:.3f}s copy {t2-t1:.3f}s unregister {t3-t2:.3f}s", flush=True)
from paper_2407_17651_b200.pipeline import _download
for rep in range(2):
    t = time.time(); hh = _download(ds, torch); print(f"_download (threaded first touch + register) {time.time()-t:.3f}s", flush=True)
    assert all(np.array_equal(a, np.ascontiguousarray(b, dtype=a.dtype)) for a, (b, _) in zip(hh, arrs))
    del hh
