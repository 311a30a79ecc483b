"""Pinned host -> device copy bandwidth on 1, 2 and 4 streams (6 GB of float32):
the ceiling of bench.py's e2e uploads.  python profiles/h2d_bw.py"""
import torch, time
n = 2 * 1024**3 // 4 * 3  # 6 GB of f32... keep host memory moderate
host = torch.empty(n, dtype=torch.float32, pin_memory=True)
dev = torch.empty(n, dtype=torch.float32, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    best = 0
    for rep in range(4):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        step = n // ns
        for i, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                lo = i * step; hi = n if i == ns - 1 else lo + step
                dev[lo:hi].copy_(host[lo:hi], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record(); torch.cuda.synchronize()
        bw = n * 4 / (e0.elapsed_time(e1) * 1e-3) / 1e9
        best = max(best, bw)
    print("streams", ns, round(best, 1), "GB/s")
