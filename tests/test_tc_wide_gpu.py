"""Wide tensor-core GEMM (csrc/tc_wide.cu, cfg4 widths) against float64.

Every operand layout (A / B K-major or MN-major), every epilogue (store, bias
+ tanh, tanh derivative with column sums, split-K slices), ragged tiles (M,
N, K not multiples of the tile), narrow N (BN = 32).  Accuracy target: the
3xTF32 class.  The tensor core's fp32 accumulate truncates, a drift of about
n_mma * 2^-25 relative (2e-5 at K = 4096; cuBLAS's TF32 GEMMs share it):
|err| <= 4e-5 of max |C| (the trainer's gradient tolerance is 1e-4).
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL = 4e-5


def _mats(M, N, K, a_mn, b_mn, seed=0):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = torch.randn(M, K, device="cuda", generator=g)
    B = torch.randn(N, K, device="cuda", generator=g)
    a = A.t().contiguous() if a_mn else A
    b = B.t().contiguous() if b_mn else B
    return A, B, a, b


def _err(got, want):
    got, want = got.double().cpu().numpy(), want.cpu().numpy()
    return float(np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-30))


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1), (1, 0)])
@pytest.mark.parametrize("M,N,K", [(300, 320, 300), (128, 256, 16), (1000, 4096, 40),
                                   (257, 32, 4100), (64, 512, 1029)])
def test_store_matches_float64(a_mn, b_mn, M, N, K):
    import torch

    from paper_2603_18464_b200 import ops
    A, B, a, b = _mats(M, N, K, a_mn, b_mn, seed=M + N + K)
    out = torch.full((M, N), float("nan"), device="cuda")
    ops.wide_gemm(a, b, out, a_mn=bool(a_mn), b_mn=bool(b_mn))
    want = A.double() @ B.double().t()
    assert _err(out, want) < TOL


def test_accumulation_chunks_bound_the_drift():
    """Chunked accumulation (accel_tc_wide_set_chunk): fresh accumulators per
    1024 k, summed rounding to nearest by the epilogue."""
    import torch

    from paper_2603_18464_b200 import _lib, ops
    M, N, K = 256, 256, 8192
    A, B, a, b = _mats(M, N, K, 0, 0, seed=9)
    want = A.double() @ B.double().t()
    errs = {}
    try:
        for chunk in (0, 64):
            _lib.lib().accel_tc_wide_set_chunk(chunk)
            out = torch.empty(M, N, device="cuda")
            ops.wide_gemm(a, b, out, a_mn=False, b_mn=False)
            errs[chunk] = _err(out, want)
    finally:
        _lib.lib().accel_tc_wide_set_chunk(0)
    assert errs[64] < errs[0] and errs[64] < TOL


@pytest.mark.parametrize("multicast", [0, 1, 2])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(1000, 512, 300), (384, 4096, 64), (8256, 256, 48)])
def test_cluster_multicast_matches_single_cta(multicast, a_mn, b_mn, M, N, K):
    """2-CTA clusters -- 1-SM MMAs with the B tile multicast (1) or 2-SM UMMA
    pairs, cta_group::2 (2) -- odd m-tile counts included, == the one-CTA
    kernel == float64."""
    import torch

    from paper_2603_18464_b200 import _lib, ops
    A, B, a, b = _mats(M, N, K, a_mn, b_mn, seed=K)
    outs = []
    try:
        for mc in (0, multicast):
            _lib.lib().accel_tc_wide_set_multicast(mc)
            out = torch.full((M, N), float("nan"), device="cuda")
            ops.wide_gemm(a, b, out, a_mn=bool(a_mn), b_mn=bool(b_mn))
            outs.append(out)
    finally:
        _lib.lib().accel_tc_wide_set_multicast(2)
    assert _err(outs[1], A.double() @ B.double().t()) < TOL
    assert torch.equal(outs[0], outs[1])  # same accumulation order either way


@pytest.mark.parametrize("ks", [2, 5])
def test_split_k_slices_sum_to_product(ks):
    import torch

    from paper_2603_18464_b200 import ops
    M, N, K = 256, 300, 2000
    A, B, a, b = _mats(M, N, K, 1, 1, seed=ks)
    part = torch.full((ks, M, N), float("nan"), device="cuda")
    ops.wide_gemm(a, b, part, a_mn=True, b_mn=True, epi=3, kslices=ks)
    want = A.double() @ B.double().t()
    assert _err(part.double().sum(0), want) < TOL
    out = torch.empty(M, N, device="cuda")
    ops.reduce_segments([(part, out, ks, M * N, M * N)])
    assert _err(out, want) < TOL


def test_bias_tanh_and_dtanh_epilogues():
    import torch

    from paper_2603_18464_b200 import ops
    M, N, K = 700, 512, 600
    A, B, a, b = _mats(M, N, K, 0, 0, seed=3)
    A = A * 0.05
    a = A
    bias = torch.randn(N, device="cuda")
    out = torch.empty(M, N, device="cuda")
    ops.wide_gemm(a, b, out, a_mn=False, b_mn=False, epi=1, bias=bias)
    pre = A.double() @ B.double().t() + bias.double()
    # tanh' <= 1: the GEMM's error (<= TOL of max |pre|) bounds the output's
    assert float((out.double() - torch.tanh(pre)).abs().max()) < TOL * float(pre.abs().max())
    # dtanh: Y = (A . W) (1 - H^2), W stored [K, N] (MN-major B), column sums per 128-row tile
    W = torch.randn(K, N, device="cuda")
    H = torch.tanh(torch.randn(M, N, device="cuda"))
    y = torch.empty(M, N, device="cuda")
    nt = -(-M // 128)
    part = torch.full((nt, N), float("nan"), device="cuda")
    ops.wide_gemm(A, W, y, a_mn=False, b_mn=True, epi=2, h=H, col_part=part)
    want = (A.double() @ W.double()) * (1 - H.double() ** 2)
    assert _err(y, want) < TOL
    assert _err(part.double().sum(0), want.sum(0)) < TOL
    # public wrappers route wide shapes here
    y2, part2, n2 = ops.tc_matmul_nn_dtanh(A, W, H, torch.empty(M, N, device="cuda"),
                                          lambda n: torch.empty(n, N, device="cuda"))
    assert n2 == nt and _err(y2, want) < TOL


@pytest.mark.parametrize("M", [528, 129, 17])
def test_dtanh_column_sums_stay_inside_col_part(M):
    """An odd number of 128-row tiles: the 2-SM pair's second tile lies past M
    and must not write a column-sum row (col_part has ceil(M / 128) rows)."""
    import torch

    from paper_2603_18464_b200 import ops
    N, K = 512, 256
    A = torch.randn(M, K, device="cuda") * 0.05
    W = torch.randn(K, N, device="cuda")
    H = torch.tanh(torch.randn(M, N, device="cuda"))
    nt = -(-M // 128)
    buf = torch.full((nt + 2, N), float("nan"), device="cuda")
    buf[nt:] = 12345.0  # canary rows right after the parts
    y = torch.empty(M, N, device="cuda")
    ops.wide_gemm(A, W, y, a_mn=False, b_mn=True, epi=2, h=H, col_part=buf[:nt])
    torch.cuda.synchronize()
    assert bool((buf[nt:] == 12345.0).all())
    want = (A.double() @ W.double()) * (1 - H.double() ** 2)
    assert _err(y, want) < TOL
    assert _err(buf[:nt].double().sum(0), want.sum(0)) < TOL


def test_public_wrappers_use_the_wide_kernel():
    import torch

    from paper_2603_18464_b200 import _lib, ops
    M, K, N = 513, 4096, 256
    x = torch.randn(M, K, device="cuda")
    w = torch.randn(N, K, device="cuda")
    n0 = _lib.launch_count()
    y = ops.tc_linear(x, w)
    assert _lib.launch_count() > n0  # libaccel launched it (pairs + GEMM + reduce)
    assert _err(y, x.double() @ w.double().t()) < TOL
    dy = torch.randn(M, 300, device="cuda")
    g = ops.tc_wgrad(dy, x, torch.empty(300, K, device="cuda"))
    assert _err(g, dy.double().t() @ x.double()) < TOL


def test_pairs_hold_the_tf32_split():
    """Per 8-group: bf16(hi) and bf16(lo) with hi = trunc19(x) (the tf32 value
    of the raw word) and lo = x - hi, in either order, along rows or columns."""
    import torch

    from paper_2603_18464_b200 import ops
    x = torch.randn(37, 45, device="cuda") * 3.0
    hi_t = (x.view(torch.int32) & -8192).view(torch.float32)
    lo_t = x - hi_t
    for row_pair in (False, True):
        for lo_first in (False, True):
            p = ops.tf32_pairs(x, row_pair, lo_first).float()
            if row_pair:
                grp = p.view(-1, 2, 8, p.shape[1])
                f, s_ = grp[:, 0].reshape(-1, p.shape[1]), grp[:, 1].reshape(-1, p.shape[1])
                f, s_ = f[:37, :45], s_[:37, :45]
            else:
                grp = p.view(p.shape[0], -1, 2, 8)
                f = grp[:, :, 0].reshape(p.shape[0], -1)[:, :45]
                s_ = grp[:, :, 1].reshape(p.shape[0], -1)[:, :45]
            hi, lo = (s_, f) if lo_first else (f, s_)
            assert float(((hi - hi_t).abs() / hi_t.abs().clamp_min(1e-30)).max()) <= 2 ** -8
            assert float((lo - lo_t).abs().max()) <= float(lo_t.abs().max()) * 2 ** -8


@pytest.mark.parametrize("M,N,K", [(1, 32, 16), (129, 96, 200), (385, 300, 40), (641, 544, 72)])
@pytest.mark.parametrize("epi", [0, 1, 2, 3])
def test_epilogues_write_only_their_outputs(M, N, K, epi):
    """Ragged M / N / K (odd tile counts, so a 2-SM pair's second tile can lie
    past M): every epilogue writes exactly its [M, N] block (pitched output with
    canary rows and columns around it), its column-sum rows and its split-K
    slices -- nothing else."""
    import torch

    from paper_2603_18464_b200 import ops
    CAN = 7777.0
    A, W, a, w = _mats(M, N, K, 0, 1, seed=M * 7 + N)
    A = A * 0.05
    a = A
    want = A.double() @ W.double().t()
    nt = -(-M // 128)
    if epi == 3:
        ks = 3 if K >= 48 else 1
        buf = torch.full((ks * M * N + 1024,), CAN, device="cuda")
        ops.wide_gemm(a, w, buf, a_mn=False, b_mn=True, epi=3, kslices=ks)
        torch.cuda.synchronize()
        assert bool((buf[ks * M * N:] == CAN).all())
        got = buf[:ks * M * N].view(ks, M, N).double().sum(0)
        assert _err(got, want) < TOL
        return
    buf = torch.full((M + 3, N + 12), CAN, device="cuda")
    out = buf[1:M + 1, 4:N + 4]  # pitched, with canaries on every side
    bias = torch.randn(N, device="cuda") if epi == 1 else None
    H = torch.tanh(torch.randn(M, N, device="cuda")) if epi == 2 else None
    part = torch.full((nt + 2, N), CAN, device="cuda") if epi == 2 else None
    ops.wide_gemm(a, w, out, a_mn=False, b_mn=True, epi=epi, bias=bias, h=H,
                  col_part=part[:nt] if part is not None else None)
    torch.cuda.synchronize()
    mask = torch.ones_like(buf, dtype=torch.bool)
    mask[1:M + 1, 4:N + 4] = False
    assert bool((buf[mask] == CAN).all())
    if epi == 0:
        assert _err(out, want) < TOL
    elif epi == 1:
        pre = want + bias.double()
        assert float((out.double() - torch.tanh(pre)).abs().max()) < TOL * float(pre.abs().max())
    else:
        y = want * (1 - H.double() ** 2)
        assert _err(out, y) < TOL
        assert bool((part[nt:] == CAN).all())
        assert _err(part[:nt].double().sum(0), y.sum(0)) < TOL
