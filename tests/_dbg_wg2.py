import sys, torch
from paper_2603_18464_b200 import ops
F = int(sys.argv[1])
for n, k in [(64, 64), (256, 64), (64, 195)]:
    dy = torch.randn(F, n, device="cuda"); x = ops.pitched(torch.randn(F, k, device="cuda"))
    out = torch.empty(n, k, device="cuda")
    ops.tc_wgrad(dy, x, out)
    torch.cuda.synchronize()
    ref = dy.double().t() @ x.double()
    print(n, k, float((out.double() - ref).abs().max() / ref.abs().max()), flush=True)
