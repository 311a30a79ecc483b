import os, subprocess, sys
if len(sys.argv) == 1:
    for env in [{}, {"ACCEL_TC_FLUSH": "4096"}, {"ACCEL_TC_SR": "16"}, {"ACCEL_TC_SR": "32"}, {"ACCEL_TC_SR": "64"}]:
        subprocess.run([sys.executable, __file__, str(env)], env=dict(os.environ, **env))
    sys.exit()
import torch
from paper_2603_18464_b200 import ops
F = 1600000
res = []
for n, k in [(64, 64), (256, 64), (64, 195)]:
    dy = torch.randn(F, n, device="cuda"); x = ops.pitched(torch.randn(F, k, device="cuda"))
    out = torch.empty(n, k, device="cuda")
    ops.tc_wgrad(dy, x, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ops.tc_wgrad(dy, x, out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    res.append(f"({n},{k}) {ms:.3f}ms {4*F*(n+k)/ms/1e6:.0f}GB/s")
print(sys.argv[1], " | ".join(res), flush=True)
