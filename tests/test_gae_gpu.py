"""(a) Segmented GAE + pooled normalization on the GPU vs the float64 oracle.

Tolerances (north star): advantages/returns within 1e-5 scaled-relative;
segmentation (frame rows) bit-exact.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import scaled_err
from oracle import c_oracle
from oracle.trainer_ref import gae, pooled_normalize

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _run(lengths, done, gamma=0.99, lam=0.95, seed=0):
    import torch

    from paper_2603_18464_b200 import ops

    rng = np.random.default_rng(seed)
    lens = np.asarray(lengths, dtype=np.int64)
    off = np.zeros(len(lens) + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    n, nt = int(off[-1]), len(lens)
    r = rng.normal(size=n).astype(np.float32)
    v = rng.normal(size=n + nt).astype(np.float32)
    d = np.asarray(done, dtype=np.uint8)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    frame = torch.empty(n, dtype=torch.int32, device="cuda")
    adv, ret, sums = ops.gae_segmented(dev(r), dev(v), dev(off), dev(d), gamma, lam,
                                       frame_of=frame)
    torch.cuda.synchronize()
    return r, v, off, d, adv.cpu().numpy(), ret.cpu().numpy(), sums.cpu().numpy(), \
        frame.cpu().numpy()


def test_gae_matches_oracle_small_ragged():
    rng = np.random.default_rng(1)
    lens = rng.integers(1, 40, size=50)
    done = rng.random(50) < 0.5
    r, v, off, d, adv, ret, sums, frame = _run(lens, done)
    exp_adv, exp_ret = [], []
    for s in range(len(lens)):
        a, b = off[s], off[s + 1]
        ea, er = gae(r[a:b], v[a + s:b + s + 1], bool(d[s]), 0.99, 0.95)
        exp_adv.append(ea)
        exp_ret.append(er)
    exp_adv, exp_ret = np.concatenate(exp_adv), np.concatenate(exp_ret)
    assert scaled_err(adv, exp_adv) < TOL
    assert scaled_err(ret, exp_ret) < TOL
    np.testing.assert_array_equal(frame, np.arange(off[-1]) + np.repeat(np.arange(len(lens)), lens))
    assert sums[2] == off[-1] and sums[3] == 0
    assert abs(sums[0] - exp_adv.sum()) < 1e-4 * max(1.0, np.abs(exp_adv).sum())


@pytest.mark.parametrize("case", ["one_long", "all_ones", "libero_mix", "tile_edges",
                                  "pass_edges", "with_empty", "skewed", "fewer_than_warps"])
def test_gae_matches_c_oracle_edge_cases(case):
    rng = np.random.default_rng(7)
    if case == "one_long":          # one trajectory spanning many tiles (look-back chain)
        lens, done = [50_000], [False]
    elif case == "all_ones":        # every transition is its own trajectory
        lens, done = [1] * 5000, rng.random(5000) < 0.5
    elif case == "tile_edges":      # boundaries exactly on 2048-frame segment strides
        lens, done = [2048, 2047, 1, 4096, 2049, 3], [True, False, True, False, True, False]
    elif case == "pass_edges":      # trajectories around the 3072-frame pass size
        lens = [3071, 3072, 3073, 6143, 6144, 1, 2, 9215, 5, 3070]
        done = [True, False, True, True, False, False, True, False, True, False]
    elif case == "with_empty":      # zero-step trajectories (bootstrap frame only)
        lens = rng.integers(0, 6, size=3000)
        lens[:7] = 0
        lens[-5:] = 0
        done = rng.random(3000) < 0.5
    elif case == "skewed":          # the warp ranges balance steps + a per-trajectory cost:
        lens = [20_000] + [1] * 20_000 + [0] * 300 + [15_000] + [2] * 7000  # long and tiny mixed
        done = rng.random(len(lens)) < 0.5
    elif case == "fewer_than_warps":  # most warps own no trajectory
        lens, done = [5, 700, 3], [True, False, False]
    else:
        from paper_2603_18464_b200.workload import libero_long_lengths
        lens, done = libero_long_lengths(rng, 512)
    r, v, off, d, adv, ret, sums, frame = _run(lens, done, seed=3)
    ea, er = c_oracle.gae_csr(r, v, off, d, 0.99, 0.95)
    assert scaled_err(adv, ea) < TOL
    assert scaled_err(ret, er) < TOL
    assert int(sums[2]) == int(off[-1])


def test_gae_full_cfg2_size_matches_c_oracle():
    """cfg2 upper end: 65,536 LIBERO-Long trajectories (~25M steps)."""
    from paper_2603_18464_b200.workload import libero_long_lengths
    lens, done = libero_long_lengths(np.random.default_rng(11), 65536)
    r, v, off, d, adv, ret, sums, frame = _run(lens, done, gamma=0.995, lam=0.97, seed=5)
    ea, er = c_oracle.gae_csr(r, v, off, d, 0.995, 0.97)
    assert scaled_err(adv, ea) < TOL
    assert scaled_err(ret, er) < TOL
    s, q = c_oracle.sums(ea)
    assert abs(sums[0] - s) <= 1e-6 * max(1.0, abs(s)) + 1e-3
    assert abs(sums[1] - q) <= 1e-5 * q


def test_gae_deterministic():
    a = _run([300, 7, 9000, 1, 40], [True, False, False, True, False], seed=9)
    b = _run([300, 7, 9000, 1, 40], [True, False, False, True, False], seed=9)
    np.testing.assert_array_equal(a[4], b[4])
    np.testing.assert_array_equal(a[6], b[6])


def test_normalize_finalize_and_apply():
    import torch

    from paper_2603_18464_b200 import ops

    rng = np.random.default_rng(2)
    x = rng.normal(loc=1.0, scale=3.0, size=1001)
    xs = x.astype(np.float32)
    sums = torch.tensor([xs.astype(np.float64).sum(), (xs.astype(np.float64) ** 2).sum(),
                         float(xs.size)], dtype=torch.float64, device="cuda")
    stats = ops.normalize_finalize(sums, 1e-8)
    out = ops.normalize_apply(torch.from_numpy(xs).cuda(), stats)
    exp, summ = pooled_normalize(np.array_split(xs.astype(np.float64), 4))
    st = stats.cpu().numpy()
    assert st[3] == 0
    assert abs(st[0] - summ["mean"]) < 1e-12 and abs(st[1] - summ["std"]) < 1e-9
    assert scaled_err(out.cpu().numpy(), np.concatenate(exp)) < TOL
    # domain flags: N == 0 and negative variance
    st0 = ops.normalize_finalize(torch.zeros(3, dtype=torch.float64, device="cuda"), 1e-8)
    assert st0.cpu().numpy()[3] == 1
    bad = torch.tensor([10.0, 1.0, 2.0], dtype=torch.float64, device="cuda")
    assert ops.normalize_finalize(bad, 1e-8).cpu().numpy()[3] == 2


def test_gae_validation_errors():
    import torch

    from paper_2603_18464_b200 import ops
    from paper_2603_18464_b200.errors import DimensionError, DomainError

    z = lambda n, dt: torch.zeros(n, dtype=dt, device="cuda")
    off = torch.tensor([0, 2], dtype=torch.int64, device="cuda")
    with pytest.raises(DomainError):
        ops.gae_segmented(z(2, torch.float32), z(3, torch.float32), off, z(1, torch.uint8),
                          0.0, 0.95)
    with pytest.raises(DimensionError):
        ops.gae_segmented(z(2, torch.float32), z(4, torch.float32), off, z(1, torch.uint8),
                          0.9, 0.95)


@pytest.mark.parametrize("case", ["nan_reward", "inf_value", "huge_finite"])
def test_gae_nonfinite_count(case):
    """sums[3] = number of steps whose advantage or return is not finite (the
    build's check_finite input); finite outputs whose per-lane sums overflow
    count as finite."""
    import torch

    from paper_2603_18464_b200 import ops

    rng = np.random.default_rng(5)
    lens = np.array([300, 17, 544, 545, 1, 90] * 40, dtype=np.int64)
    off = np.zeros(len(lens) + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    n, nt = int(off[-1]), len(lens)
    r = rng.normal(size=n).astype(np.float32)
    v = rng.normal(size=n + nt).astype(np.float32)
    lam = 0.95
    if case == "nan_reward":
        r[[5, 400, 1000, n - 1]] = np.nan
    elif case == "inf_value":
        v[[3, 777, 2000]] = np.inf
    else:  # |A| ~ 1e38 on many consecutive steps: finite, but their sums overflow
        r[:] = 1e38
        v[:] = 0.0
        lam = 0.0
    d = (rng.random(nt) < 0.5).astype(np.uint8)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    adv, ret, sums = ops.gae_segmented(dev(r), dev(v), dev(off), dev(d), 0.99, lam)
    torch.cuda.synchronize()
    adv, ret, sums = adv.cpu().numpy(), ret.cpu().numpy(), sums.cpu().numpy()
    want = int(np.sum(~np.isfinite(adv) | ~np.isfinite(ret)))
    assert int(sums[3]) == want
    if case == "huge_finite":
        assert want == 0 and np.all(np.isfinite(adv))
    else:
        assert want > 0
