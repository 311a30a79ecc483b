"""Blocked-grouping key pass (accel_fold_blocked_pieces) vs a float64 sum:
out[key] = sum over blocks of the pieces of composite key block * nkeys + key,
with and without a heavy key (folded over its own CTAs), at block counts on
both sides of the heavy split (64), and deterministic."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nblocks,heavy", [(1, 2), (3, 2), (43, 2), (70, 2), (70, -1), (5, 0)])
def test_fold_blocked_pieces(nblocks, heavy):
    import torch

    from paper_2603_18464_b200 import _lib
    from paper_2603_18464_b200.ops import _pp

    rng = np.random.default_rng(nblocks * 7 + heavy)
    nkeys, D = 6, 256
    counts = rng.integers(0, 4, size=(nblocks, nkeys))
    if heavy >= 0:
        counts[:, heavy] = rng.integers(100, 160, size=nblocks)
    off = np.zeros(nblocks * nkeys + 1, dtype=np.int64)
    np.cumsum(counts.reshape(-1), out=off[1:])
    P = int(off[-1])
    pieces = rng.normal(size=(max(P, 1), D)).astype(np.float32)
    want = np.zeros((nkeys, D))
    for b in range(nblocks):
        for k in range(nkeys):
            ck = b * nkeys + k
            want[k] += pieces[off[ck]:off[ck + 1]].astype(np.float64).sum(0)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    pb, po = dev(pieces), dev(off)
    ws = torch.empty(int(_lib.lib().accel_fold_workspace_size(nkeys, D)) // 4 + 4,
                     dtype=torch.float32, device="cuda")
    outs = []
    for _ in range(2):
        out = torch.full((nkeys, D), float("nan"), device="cuda")
        _lib.call("accel_fold_blocked_pieces", _pp(pb), _pp(po), nkeys, nblocks, D, heavy,
                  _pp(out), _pp(ws), None)
        torch.cuda.synchronize()
        outs.append(out.cpu().numpy())
    np.testing.assert_allclose(outs[0], want, rtol=1e-5, atol=1e-3)
    np.testing.assert_array_equal(outs[0], outs[1])  # fixed partitions: bitwise repeatable
