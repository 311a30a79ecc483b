"""Value-head attention backward: the fused one-pass kernel
(accel_value_attn_backward) against the two-pass kernels it replaces on the
trainer path (value_attn_grad + value_attn_wgrad) and a float64 restatement
of models.py:292-314 (dalpha_j = du . h_j, de = alpha (dalpha - sum alpha dalpha),
dw_attn = sum_ij de_ij h_ij, db_attn = sum_ij de_ij)."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("D,frames", [(64, True), (32, False), (48, True)])
def test_attn_backward_fused_matches_two_pass(D, frames):
    import torch

    from paper_2603_18464_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(D)
    F, R = 3000, 5001
    h1 = torch.tanh(torch.randn(F, D, device="cuda", generator=g))
    h2 = torch.tanh(torch.randn(F, D, device="cuda", generator=g))
    rows = F if not frames else R
    row_frame = (torch.randint(0, F, (R,), device="cuda", generator=g, dtype=torch.int32)
                 if frames else None)
    dU = torch.randn(rows, D, device="cuda", generator=g)
    alpha = torch.softmax(torch.randn(rows, 2, device="cuda", generator=g), 1)
    grid = ops.warp_grid(rows)
    de1, de2 = torch.empty(rows, 2, device="cuda"), torch.empty(rows, 2, device="cuda")
    b1, b2 = torch.empty(grid, device="cuda"), torch.empty(grid, device="cuda")
    w2 = torch.empty(grid, D, device="cuda")
    ops.value_attn_backward(dU, h1, h2, row_frame, alpha, b2, w2, grid, de=de2)
    ops.value_attn_grad(dU, h1, h2, row_frame, alpha, de1, b1, grid)
    gr = ops.rows_grid(rows)
    w1 = torch.empty(gr, D, device="cuda")
    ops.value_attn_wgrad(de1, h1, h2, row_frame, rows, w1, gr)
    assert torch.equal(de1, de2) and torch.equal(b1, b2)
    # float64 restatement
    idx = row_frame.long() if frames else torch.arange(rows, device="cuda")
    a, c = h1[idx].double(), h2[idx].double()
    d0, d1 = (dU.double() * a).sum(1), (dU.double() * c).sum(1)
    al = alpha.double()
    s = al[:, 0] * d0 + al[:, 1] * d1
    de = torch.stack([al[:, 0] * (d0 - s), al[:, 1] * (d1 - s)], 1)
    torch.testing.assert_close(de2.double(), de, rtol=1e-5, atol=1e-6)
    want_w = (de[:, :1] * a + de[:, 1:] * c).sum(0)
    scale = float(want_w.abs().max())
    assert float((w2.double().sum(0) - want_w).abs().max()) < 1e-5 * max(scale, 1.0)
    assert float((w1.double().sum(0) - want_w).abs().max()) < 1e-5 * max(scale, 1.0)
    assert abs(float(b2.double().sum()) - float(de.sum())) < 1e-4


def test_attn_backward_without_de_rows():
    import torch

    from paper_2603_18464_b200 import errors, ops
    D, F = 64, 777
    h1 = torch.randn(F, D, device="cuda")
    h2 = torch.randn(F, D, device="cuda")
    dU = torch.randn(F, D, device="cuda")
    alpha = torch.softmax(torch.randn(F, 2, device="cuda"), 1)
    grid = ops.warp_grid(F)
    b, w = torch.empty(grid, device="cuda"), torch.empty(grid, D, device="cuda")
    ops.value_attn_backward(dU, h1, h2, None, alpha, b, w, grid)  # fused path: no de needed
    b2, w2 = torch.empty(grid, device="cuda"), torch.empty(grid, D, device="cuda")
    ops.value_attn_backward(dU, h1, h2, None, alpha, b2, w2, grid, de=torch.empty(F, 2, device="cuda"))
    assert torch.equal(b, b2) and torch.equal(w, w2)
    # a width the fused kernel does not cover needs the de rows
    with pytest.raises(errors.DimensionError):
        ops.value_attn_backward(dU[:, :40].contiguous(), h1[:, :40].contiguous(),
                                h2[:, :40].contiguous(), None, alpha, b, w[:, :40].contiguous(), grid)
