"""Time the trainer step's dense products: tcgen05 3xTF32 kernel vs cuBLAS fp32.

    python profiles/gemm_bench.py [F]

Shapes are the cfg2 step's (D=64, O=195, A=256, value MLP 64) over F frame
rows.  Prints one line per product: ms (tc), ms (cuBLAS sgemm), GB/s of the
tc kernel against its algorithmic bytes, rel err of each vs fp64.
"""

import sys

import torch

from paper_2603_18464_b200 import ops


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def rel(a, b):
    return float((a.double() - b).abs().max() / b.abs().max())


def main():
    F = int(sys.argv[1]) if len(sys.argv) > 1 else 1_600_000
    torch.backends.cuda.matmul.allow_tf32 = False
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    def rn(*s):
        t = torch.randn(*s, generator=g, device=dev)
        if len(s) == 2 and s[0] > 4096 and s[1] % 4:  # frame rows: pitched storage
            t2 = ops.alloc_pitched(s[0], s[1], dev)
            t2.copy_(t)
            return t2
        return t
    D, O, A, H = 64, 195, 256, 64
    rows = []
    # row transforms: y[F, n] = x[F, k] W[n, k]^T
    for name, k, n in [("h1=frames.W0^T", O, D), ("h2=h1.W1^T", D, D), ("H2W=h2.Wh^T", D, A),
                       ("zm=U.W0v^T", D, H)]:
        x, w = rn(F, k), rn(n, k) * 0.1
        out = torch.empty(F, n, device=dev)
        t_tc = timeit(lambda: ops.tc_linear(x, w, out))
        t_cb = timeit(lambda: torch.mm(x, w.t(), out=out))
        ops.tc_linear(x, w, out)
        e_tc = rel(out, x.double() @ w.double().t())
        byt = 4 * F * (k + n)
        rows.append((name, t_tc, t_cb, byt / t_tc / 1e6, e_tc))
    # backward data: dx[F, k] = dy[F, n] W[n, k]
    for name, n, k in [("dh2=G.Wh", A, D), ("dh1=dz2.W1", D, D), ("dU=dzm.W0v", H, D)]:
        dy, w = rn(F, n), rn(n, k) * 0.1
        out = torch.empty(F, k, device=dev)
        t_tc = timeit(lambda: ops.tc_matmul_nn(dy, w, out))
        t_cb = timeit(lambda: torch.mm(dy, w, out=out))
        ops.tc_matmul_nn(dy, w, out)
        e_tc = rel(out, dy.double() @ w.double())
        rows.append((name, t_tc, t_cb, 4 * F * (n + k) / t_tc / 1e6, e_tc))
    # weight grads: dW[n, k] = dy[F, n]^T x[F, k]
    for name, n, k in [("dWh=G^T.h2", A, D), ("dW1=dz2^T.h1", D, D), ("dW0=dh1^T.frames", D, O),
                       ("dW0v=dzm^T.U", H, D)]:
        dy, x = rn(F, n), rn(F, k)
        out = torch.empty(n, k, device=dev)
        t_tc = timeit(lambda: ops.tc_wgrad(dy, x, out))
        t_cb = timeit(lambda: torch.mm(dy.t(), x, out=out))
        ops.tc_wgrad(dy, x, out)
        e_tc = rel(out, dy.double().t() @ x.double())
        rows.append((name, t_tc, t_cb, 4 * F * (n + k) / t_tc / 1e6, e_tc))
    print(f"F={F}")
    print(f"{'product':20s} {'tc ms':>8s} {'sgemm ms':>9s} {'tc GB/s':>8s} {'tc rel err':>10s}")
    for r in rows:
        print(f"{r[0]:20s} {r[1]:8.3f} {r[2]:9.3f} {r[3]:8.0f} {r[4]:10.2e}")
    print(f"{'total':20s} {sum(r[1] for r in rows):8.3f} {sum(r[2] for r in rows):9.3f}")


if __name__ == "__main__":
    main()
