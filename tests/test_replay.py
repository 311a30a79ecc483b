"""On-device replay buffer (reference buffers.py:44-94).

CPU: the span ring allocator.  GPU: sampling draws the reference's picks
(rng.integers over the FIFO), FIFO eviction at capacity, and a batch built
from device-resident trajectories equals the one built from the host
trajectories (same kernels on the same packed data: bitwise)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2603_18464_b200.replay import SpanRing


def test_span_ring_allocates_wraps_and_evicts_overlaps():
    r = SpanRing(10)
    a, ev = r.alloc(4, "a")
    b, _ = r.alloc(4, "b")
    assert (a, b, ev) == (0, 4, [])
    c, ev = r.alloc(3, "c")  # 8 + 3 > 10: restarts at 0, overlaps a
    assert c == 0 and ev == ["a"]
    d, ev = r.alloc(3, "d")  # [3, 6): overlaps b
    assert d == 3 and ev == ["b"]
    r.release("c")
    e, ev = r.alloc(5, "e")  # [6, 11) > 10: wraps to 0, overlaps d only (c released)
    assert e == 0 and ev == ["d"]
    with pytest.raises(Exception):
        r.alloc(11, "f")


def _trajs(rng, n, K, A, O):
    from paper_2603_18464_b200.workload import synthetic_trajectories
    lens = rng.integers(1, 30, size=n)
    return synthetic_trajectories(rng, lens, rng.random(n) < 0.5, K, A, O)


@pytest.mark.gpu
def test_device_replay_matches_host_build():
    from paper_2603_18464_b200.replay import DeviceReplayBuffer
    from paper_2603_18464_b200.trainer import Trainer, TrainerConfig
    from paper_2603_18464_b200.types import (ModelBundle, PolicyConfig, PolicyModel, ValueConfig,
                                             ValueHead)
    rng = np.random.default_rng(4)
    K, A, O, D = 7, 256, 195, 64
    pc = PolicyConfig(obs_dim=O, hidden_dim=D, chunk_len=K, n_actions=A, vocab_size=A + 8,
                      action_start=4)
    bundle = ModelBundle(PolicyModel.init(rng, pc), ValueHead.init(rng, ValueConfig(D, 40, 32)))
    trajs = _trajs(rng, 14, K, A, O)
    buf = DeviceReplayBuffer("main", capacity=10, obs_dim=O, chunk_len=K, n_actions=A,
                             max_transitions=10 * 30)
    for t in trajs:
        buf.push(t)
    st = buf.stats()
    assert (st.size, st.pushed, st.evicted) == (10, 14, 4)  # FIFO: the first 4 are gone
    live = trajs[4:]
    g1, g2 = np.random.default_rng(9), np.random.default_rng(9)
    picks = buf.sample(6, g1)
    want = [live[i] for i in g2.integers(0, len(live), size=6)]  # the reference's draw
    assert [p.t_len for p in picks] == [t.tokens.shape[0] for t in want]
    tr_dev = Trainer(bundle, TrainerConfig())
    tr_host = Trainer(bundle, TrainerConfig())
    bd = tr_dev.build_train_batch(picks)
    bh = tr_host.build_train_batch(want)
    for k in ("tokens", "steps", "advantages", "value_targets", "behavior_logp", "obs"):
        np.testing.assert_array_equal(getattr(bd, k), getattr(bh, k), err_msg=k)
    assert (bd.n_real, bd.behavior_lag_mean) == (bh.n_real, bh.behavior_lag_mean)
    rd, rh = tr_dev.train_step(bd), tr_host.train_step(bh)
    # parameters are bitwise equal; the loss kernel's float64 statistics are summed
    # in the order its dynamic schedule hands out transitions (last-bit differences)
    assert set(rd) == set(rh)
    for k in rd:
        assert abs(rd[k] - rh[k]) <= 1e-12 * max(1.0, abs(rh[k])), k
    np.testing.assert_array_equal(tr_dev.params.p[tr_dev.params.cur].cpu().numpy(),
                                  tr_host.params.p[tr_host.params.cur].cpu().numpy())
