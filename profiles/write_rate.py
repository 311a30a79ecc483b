"""HBM write-only vs copy bandwidth on this B200 (torch fill_ / copy_ kernels).

usage: python profiles/write_rate.py   (prints GB/s; no libaccel involved)
"""
import torch

n = 13 * 2**30 // 4
x = torch.empty(n, device="cuda")
y = torch.empty(n // 2, device="cuda")
z = torch.empty(n // 2, device="cuda")


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


t = timed(lambda: x.fill_(1.0))
print(f"write-only fill_ 13 GiB: {t:.3f} ms  {n * 4 / t / 1e6:.0f} GB/s")
t = timed(lambda: y.copy_(z))
print(f"copy 6.5 GiB -> 6.5 GiB: {t:.3f} ms  {n * 4 / t / 1e6:.0f} GB/s (read+write)")
