"""tcgen05 3xTF32 GEMM vs a float64 torch reference (fp32-level accuracy)."""

from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu


def rel_err(x, ref):
    return float((x.double() - ref).abs().max() / ref.abs().max().clamp_min(1e-30))


@pytest.mark.parametrize("M,K,N", [(1, 8, 16), (300, 64, 256), (1000, 195, 64), (4097, 64, 64),
                                   (513, 64, 32), (128, 256, 64), (777, 96, 195)])
def test_tc_linear_matches_fp64(M, K, N):
    from paper_2603_18464_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(M + K + N)
    x = torch.randn(M, K, device="cuda", generator=g)
    w = torch.randn(N, K, device="cuda", generator=g)
    b = torch.randn(N, device="cuda", generator=g)
    ref = x.double() @ w.double().t()
    y = ops.tc_linear(x, w)
    assert rel_err(y, ref) < 4e-6
    yb = ops.tc_linear(x, w, bias=b, tanh=True)
    pre = ref + b.double()  # tanh is 1-Lipschitz: bound by the pre-activation scale
    assert float((yb.double() - torch.tanh(pre)).abs().max()) < 4e-6 * float(pre.abs().max())
    acc = torch.randn(M, N, device="cuda", generator=g)
    ya = ops.tc_linear(x, w, out=acc.clone(), accumulate=True)
    assert rel_err(ya, ref + acc.double()) < 4e-6


@pytest.mark.parametrize("M,K,N", [(1000, 256, 64), (4096, 32, 256)])
def test_tc_matmul_nn(M, K, N):
    from paper_2603_18464_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(M, K, device="cuda", generator=g)
    w = torch.randn(K, N, device="cuda", generator=g)
    assert rel_err(ops.tc_matmul_nn(x, w), x.double() @ w.double()) < 4e-6


@pytest.mark.parametrize("F,n,k,slices", [(5000, 64, 64, None), (100000, 256, 64, None),
                                          (70000, 64, 195, None), (3000, 32, 64, 3)])
def test_tc_wgrad_matches_fp64(F, n, k, slices):
    from paper_2603_18464_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(F)
    dy = torch.randn(F, n, device="cuda", generator=g)
    x = torch.randn(F, k, device="cuda", generator=g)
    out = torch.empty(n, k, device="cuda")
    ops.tc_wgrad(dy, x, out, kslices=slices)
    ref = dy.double().t() @ x.double()
    assert rel_err(out, ref) < 1.2e-5
    out2 = torch.empty_like(out)
    ops.tc_wgrad(dy, x, out2, kslices=slices)
    assert torch.equal(out, out2)  # deterministic


@pytest.mark.gpu
@pytest.mark.parametrize("M,K,N", [(5000, 256, 64), (3001, 64, 64), (700, 64, 32), (1, 256, 64),
                                   (777, 200, 64), (130, 256, 32)])
def test_tc_dtanh_fused_epilogue(M, K, N):
    """(x.w) * (1 - h^2) and its column sums in the GEMM epilogue (dpre = dh (1 - h^2))."""
    from paper_2603_18464_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(M)
    x = torch.randn(M, K, device="cuda", generator=g)
    w = torch.randn(K, N, device="cuda", generator=g) * 0.1
    h = torch.tanh(torch.randn(M, N, device="cuda", generator=g))
    out = torch.empty(M, N, device="cuda")
    parts = {}
    y, part, n = ops.tc_matmul_nn_dtanh(x, w, h, out, lambda k: parts.setdefault(
        "p", torch.empty(k, N, device="cuda")))
    ref = (x.double() @ w.double()) * (1 - h.double() ** 2)
    assert rel_err(y, ref) < 4e-6
    colsum = part[:n].double().sum(0)
    assert float((colsum - ref.sum(0)).abs().max()) < 1e-4 * float(ref.abs().sum(0).max())


@pytest.mark.parametrize("a_trans,b_trans", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_small_gemm_all_layouts(a_trans, b_trans):
    """accel_small_gemm (the <= 264-row products around the factorized head)."""
    import torch

    from paper_2603_18464_b200 import ops
    M, N, K = 257, 70, 264
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(N, K, device="cuda")
    a = A.t().contiguous() if a_trans else A
    b = B.t().contiguous() if b_trans else B
    out = torch.empty(M, N, device="cuda")
    ops.small_gemm(a, b, out, bool(a_trans), bool(b_trans))
    assert rel_err(out, A.double() @ B.double().t()) < 1e-6


@pytest.mark.parametrize("M,N,K", [(7, 256, 4096), (257, 256, 4096), (7, 4096, 256), (3, 5, 9000)])
def test_small_gemm_split_k(M, N, K):
    """Long reductions over few output tiles run as k slices summed in order:
    accurate, and bitwise reproducible run to run."""
    import torch

    from paper_2603_18464_b200 import _lib, ops
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(N, K, device="cuda")
    out, out2 = torch.empty(M, N, device="cuda"), torch.empty(M, N, device="cuda")
    ops.small_gemm(A, B, out, False, False)
    ops.small_gemm(A, B, out2, False, False)
    assert torch.equal(out, out2)
    assert rel_err(out, A.double() @ B.double().t()) < 1e-6
    if M * N <= 2048:
        assert _lib.lib().accel_small_gemm_ws_floats(M, N, K) > 0  # the split path ran


@pytest.mark.parametrize("M,K,N", [(1, 64, 64), (129, 195, 64), (1000, 64, 256), (4099, 256, 64)])
def test_row_gemms_write_only_their_outputs(M, K, N):
    """Row transform (TMA-store and dtanh epilogues) and weight gradient at
    ragged sizes: pitched outputs with canaries around them stay untouched."""
    from paper_2603_18464_b200 import ops
    CAN = 4242.0
    g = torch.Generator(device="cuda").manual_seed(M + N)
    x = torch.randn(M, K, device="cuda", generator=g) * 0.1
    w = torch.randn(N, K, device="cuda", generator=g)
    buf = torch.full((M + 3, N + 8), CAN, device="cuda")
    out = buf[1:M + 1, 4:N + 4]
    ops.tc_linear(x, w, out=out)
    torch.cuda.synchronize()
    mask = torch.ones_like(buf, dtype=torch.bool)
    mask[1:M + 1, 4:N + 4] = False
    assert bool((buf[mask] == CAN).all())
    assert rel_err(out, x.double() @ w.double().t()) < 4e-6
    # dtanh: (x . w2) (1 - h^2) with column-sum parts
    w2 = torch.randn(K, N, device="cuda", generator=g)
    h = torch.tanh(torch.randn(M, N, device="cuda", generator=g))
    buf.fill_(CAN)
    parts = {}

    def part_fn(n):
        parts["buf"] = torch.full((n + 2, N), CAN, device="cuda")
        parts["n"] = n
        return parts["buf"][:n]
    y, part, n = ops.tc_matmul_nn_dtanh(x, w2, h, out, part_fn)
    torch.cuda.synchronize()
    assert bool((buf[mask] == CAN).all())
    assert bool((parts["buf"][parts["n"]:] == CAN).all())
    want = (x.double() @ w2.double()) * (1 - h.double() ** 2)
    assert rel_err(out, want) < 4e-6
    assert float((part.double().sum(0) - want.sum(0)).abs().max()) < 1e-5 * float(want.abs().sum(0).max())
    # weight gradient into a pitched [N, K] block
    dy = torch.randn(M, N, device="cuda", generator=g)
    gbuf = torch.full((N + 2, K + 8), CAN, device="cuda")
    gout = gbuf[1:N + 1, 4:K + 4]
    ops.tc_wgrad(dy, x, gout)
    torch.cuda.synchronize()
    gmask = torch.ones_like(gbuf, dtype=torch.bool)
    gmask[1:N + 1, 4:K + 4] = False
    assert bool((gbuf[gmask] == CAN).all())
    assert rel_err(gout, dy.double().t() @ x.double()) < 4e-6
