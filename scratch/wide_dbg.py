import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2603_18464_b200 import ops
torch.manual_seed(0)
def err(got, want):
    return float((got.double()-want).abs().max() / want.abs().max())
for F, O, D in ((528, 320, 512), (528, 4096, 4096), (300, 195, 512)):
    x = ops.alloc_pitched(F, O, 'cuda'); x.copy_(torch.randn(F, O, device='cuda'))
    w0 = torch.randn(D, O, device='cuda') * 0.05; b0 = torch.randn(D, device='cuda')
    h1 = ops.tc_linear(x, w0, bias=b0, tanh=True)
    print(F,O,D,'fwd tanh', err(h1, torch.tanh(x.double() @ w0.double().t() + b0.double())))
    wv = torch.randn(32, D, device='cuda')
    zm = ops.tc_linear(h1, wv)
    print('  N=32 splitK', err(zm, h1.double() @ wv.double().t()))
    wh = torch.randn(256, D, device='cuda')
    h2w = ops.tc_linear(h1, wh)
    print('  N=256', err(h2w, h1.double() @ wh.double().t()))
    g = torch.randn(F, 256, device='cuda')
    dz2, part, n = ops.tc_matmul_nn_dtanh(g, wh, h1, torch.empty(F, D, device='cuda'), lambda n: torch.empty(n, D, device='cuda'))
    want = (g.double() @ wh.double()) * (1 - h1.double()**2)
    print('  nn dtanh', err(dz2, want), err(part.double().sum(0), want.sum(0)))
    for (n_, k_, dy, xx) in ((256, D, g, h1), (D, O, dz2, x), (32, D, torch.randn(F,32,device='cuda'), h1)):
        out = torch.empty(n_, k_, device='cuda')
        ops.tc_wgrad(dy, xx, out)
        print('  wgrad', n_, k_, err(out, dy.double().t() @ xx.double()))
