"""PCIe copy time of one 134 MB vector (c5's x or y) split over k streams."""
import torch
n = 16777216
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for direction in ("d2h", "h2d", "both"):
    for k in (1, 2, 4):
        streams = [torch.cuda.Stream() for _ in range(k)]
        h2 = torch.empty(n, dtype=torch.float64).pin_memory()
        d2 = torch.empty(n, dtype=torch.float64, device="cuda")
        def go():
            step = n // k
            for i, s in enumerate(streams):
                with torch.cuda.stream(s):
                    sl = slice(i * step, n if i == k - 1 else (i + 1) * step)
                    if direction in ("d2h", "both"):
                        h[sl].copy_(d[sl], non_blocking=True)
                    if direction in ("h2d", "both"):
                        d2[sl].copy_(h2[sl], non_blocking=True)
        for _ in range(3):
            go()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for s in streams:
            s.wait_event(e0)
        for _ in range(10):
            go()
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"{direction} {k} streams: {ms:.3f} ms  {n * 8 / ms / 1e6:.1f} GB/s per direction")
