"""The drop-in's host pack (trainer.py:365-391 flattening rules): CSR layout,
float32 casts in place, threaded over trajectories, optional page-locked
staging -- equal to a plain concatenation of the reference fields."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2603_18464_b200.workload import pack_trajectories, synthetic_trajectories


def _naive(trajs):
    cat = np.concatenate
    return dict(
        frames=cat([t.observations for t in trajs]).astype(np.float32),
        steps=cat([t.steps for t in trajs]).astype(np.int32),
        values=cat([np.append(t.values, t.bootstrap_value) for t in trajs]).astype(np.float32),
        tokens=cat([t.tokens for t in trajs]).astype(np.int32),
        rewards=cat([t.rewards for t in trajs]).astype(np.float32),
        mu=cat([t.behavior_logits for t in trajs]).astype(np.float32))


def _check(pb, trajs):
    want = _naive(trajs)
    for k, v in want.items():
        np.testing.assert_array_equal(getattr(pb, k), v, err_msg=k)
    lens = [t.t_len for t in trajs]
    np.testing.assert_array_equal(pb.traj_off, np.concatenate([[0], np.cumsum(lens)]))
    np.testing.assert_array_equal(pb.done, [t.done for t in trajs])
    np.testing.assert_array_equal(pb.real, [t.source == "real" for t in trajs])


@pytest.mark.parametrize("threads", [1, 4])
def test_pack_matches_concatenation(threads):
    rng = np.random.default_rng(0)
    lens = rng.integers(1, 700, size=40)  # > 4096 transitions per worker: threaded
    trajs = synthetic_trajectories(rng, lens, rng.random(40) < 0.5, 3, 16, 11, imagined_every=4)
    _check(pack_trajectories(trajs, threads=threads), trajs)


@pytest.mark.gpu
def test_pack_into_pinned_staging_reuses_buffers():
    from paper_2603_18464_b200.workload import PinnedStaging
    rng = np.random.default_rng(1)
    st = PinnedStaging()
    for n in (30, 12, 30):
        lens = rng.integers(1, 400, size=n)
        trajs = synthetic_trajectories(rng, lens, rng.random(n) < 0.5, 7, 32, 9)
        pb = pack_trajectories(trajs, staging=st)
        _check(pb, trajs)
    import torch
    assert torch.from_numpy(pb.mu).is_pinned()


@pytest.mark.parametrize("chunks", [1, 3, 7])
def test_chunked_pack_reports_consecutive_ranges(chunks):
    """chunks > 1 (the drop-in uploads each chunk while the next is packed):
    the same arrays, and on_chunk sees consecutive trajectory ranges covering
    the batch, each already packed when reported."""
    rng = np.random.default_rng(5)
    trajs = synthetic_trajectories(rng, rng.integers(1, 300, size=23), rng.random(23) < 0.5,
                                   3, 16, 9)
    seen = []

    def on_chunk(lo, hi, off, frames, mu):
        a, b = int(off[lo]), int(off[hi])
        want = np.concatenate([t.behavior_logits for t in trajs[lo:hi]]).astype(np.float32)
        np.testing.assert_array_equal(mu[a:b], want)
        wf = np.concatenate([t.observations for t in trajs[lo:hi]]).astype(np.float32)
        np.testing.assert_array_equal(frames[a + lo:b + hi], wf)
        seen.append((lo, hi))

    pb = pack_trajectories(trajs, threads=4, chunks=chunks, on_chunk=on_chunk)
    _check(pb, trajs)
    assert seen[0][0] == 0 and seen[-1][1] == len(trajs)
    assert all(a[1] == b[0] for a, b in zip(seen, seen[1:]))
    assert len(seen) <= chunks
