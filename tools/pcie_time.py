"""PCIe bound of the e2e step: pinned host<->device copies of one c5 vector
(134 MB) alone and both directions at once (the e2e step moves x in and y out
every step, bench.py).  Run under gpurun: python tools/pcie_time.py"""
import torch

n = 16777216
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True).uniform_()
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.randn(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)


B = n * 8
for name, fn in (("h2d", lambda: d_in.copy_(h_in, non_blocking=True)),
                 ("d2h", lambda: h_out.copy_(d_out, non_blocking=True)),
                 ("h2d+d2h concurrent", both)):
    ms = timed(fn)
    k = 2 if "+" in name else 1
    print(f"{name:20s} {ms:.3f} ms  {k * B / ms / 1e6:.1f} GB/s ({B / ms / 1e6:.1f} GB/s per direction)")
