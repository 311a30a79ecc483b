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


def test_span_ring_matches_linear_scan_allocator():
    """The bisection ring reports exactly the overlaps (oldest first) that a scan
    of every live span does, under random allocs and releases with wraps."""
    class ScanRing:
        def __init__(self, size):
            self.size, self.head, self.live = size, 0, []

        def alloc(self, n, owner):
            start = self.head if self.head + n <= self.size else 0
            end = start + n
            if n == 0:  # an empty span occupies nothing
                self.head = end
                return start, []
            ev = [o for s, ln, o in self.live if s < end and start < s + ln]
            self.live = [x for x in self.live if not (x[0] < end and start < x[0] + x[1])]
            self.live.append((start, n, owner))
            self.head = end
            return start, ev

        def release(self, owner):
            self.live = [x for x in self.live if x[2] is not owner]

    def run(size, seed):
        rng = np.random.default_rng(seed)
        a, b = SpanRing(size), ScanRing(size)
        owners = []
        for step in range(3000):
            if owners and rng.random() < 0.3:
                o = owners.pop(int(rng.integers(len(owners))))
                a.release(o)
                b.release(o)
                continue
            if len(owners) > 2 and rng.random() < 0.05:  # release_many == releases in order
                k = int(rng.integers(1, len(owners)))
                gone, owners = owners[:k], owners[k:]
                a.release_many(gone)
                for o in gone:
                    b.release(o)
                continue
            if rng.random() < 0.2:  # a batch: alloc_many == the same allocs in order
                k = int(rng.integers(1, 6))
                ns = [int(rng.integers(0, size // 4 + 2)) for _ in range(k)]
                os_ = [object() for _ in range(k)]
                seq = [b.alloc(n, o) for n, o in zip(ns, os_)]
                ev_b = [x for _, ev in seq for x in ev]
                if any(x in os_ for x in ev_b):  # the batch overlaps itself
                    with pytest.raises(Exception):
                        a.alloc_many(ns, os_)
                    return
                starts, ev_a = a.alloc_many(ns, os_)
                assert starts == [st for st, _ in seq], (size, step)
                assert set(map(id, ev_a)) == set(map(id, ev_b)), (size, step)
                owners = [x for x in owners if x not in ev_a]
                owners += [o for n, o in zip(ns, os_) if n]
                continue
            o = object()
            n = int(rng.integers(1, size // 3 + 2))
            ra, rb = a.alloc(n, o), b.alloc(n, o)
            assert ra[0] == rb[0] and ra[1] == rb[1], (size, step)
            owners = [x for x in owners if x not in ra[1]] + [o]

    for size in (17, 64, 500):
        for seed in range(4):
            run(size, seed)


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


@pytest.mark.gpu
def test_push_imagined_equals_host_records():
    """Imagination outputs pushed on the device == the same episodes pushed as
    host Trajectory records (imagine_trajectories)."""
    from paper_2603_18464_b200.imagine import Imaginer
    from paper_2603_18464_b200.replay import DeviceReplayBuffer
    from paper_2603_18464_b200.types import (ModelBundle, ObsModel, ObsModelConfig, PolicyConfig,
                                             PolicyModel, RewardModel, ValueConfig, ValueHead)
    from types import SimpleNamespace
    rng = np.random.default_rng(2)
    O, K, A = 51, 2, 7
    pc = PolicyConfig(obs_dim=O, hidden_dim=16, chunk_len=K, n_actions=A)
    b = ModelBundle(PolicyModel.init(rng, pc), ValueHead.init(rng, ValueConfig(16, 30, 8)),
                    ObsModel.init(rng, ObsModelConfig(obs_dim=O, chunk_len=K, hidden_dim=24)),
                    RewardModel.init(rng, O, hidden_dim=12))
    n, H = 24, 6
    starts = np.zeros((n, O))
    for e in range(n):
        for c in range(3):
            starts[e, c * 16 + rng.integers(16)] = 1.0
        starts[e, 48 + e % 3] = 1.0
    im = Imaginer(b, grid=(4, 4))
    u = rng.random((n, H + 1, K))
    out = im.imagine_device(starts, np.arange(n) % 5, H, uniforms=u)
    dev_buf = DeviceReplayBuffer("imagined", 64, O, K, A, max_transitions=64 * H)
    host_buf = DeviceReplayBuffer("imagined", 64, O, K, A, max_transitions=64 * H)
    pushed = dev_buf.push_imagined(out)
    host = im.imagine_trajectories([SimpleNamespace(vec=starts[e], step=e % 5, task_id=0)
                                    for e in range(n)], H, uniforms=u)
    kept = [t for t in host if t is not None]
    for t in kept:
        host_buf.push(t)
    assert pushed == len(kept) == len(dev_buf) == len(host_buf)
    a, _, _ = dev_buf.gather(list(dev_buf._items))
    c, _, _ = host_buf.gather(list(host_buf._items))
    for k in a:
        np.testing.assert_array_equal(a[k].cpu().numpy(), c[k].cpu().numpy(), err_msg=k)


@pytest.mark.gpu
def test_push_imagined_fifo_overflow_equals_host_pushes():
    """Batches larger than the free capacity (and one larger than the capacity
    itself) leave the buffer, its counters and its arena contents as the
    reference's bounded FIFO of one-by-one pushes does."""
    from paper_2603_18464_b200.imagine import Imaginer
    from paper_2603_18464_b200.replay import DeviceReplayBuffer
    from paper_2603_18464_b200.types import (ModelBundle, ObsModel, ObsModelConfig, PolicyConfig,
                                             PolicyModel, RewardModel, ValueConfig, ValueHead)
    from types import SimpleNamespace
    rng = np.random.default_rng(4)
    O, K, A = 51, 2, 7
    pc = PolicyConfig(obs_dim=O, hidden_dim=16, chunk_len=K, n_actions=A)
    b = ModelBundle(PolicyModel.init(rng, pc), ValueHead.init(rng, ValueConfig(16, 30, 8)),
                    ObsModel.init(rng, ObsModelConfig(obs_dim=O, chunk_len=K, hidden_dim=24)),
                    RewardModel.init(rng, O, hidden_dim=12))
    im = Imaginer(b, grid=(4, 4))
    H, cap = 5, 10
    dev_buf = DeviceReplayBuffer("imagined", cap, O, K, A, max_transitions=cap * H)
    host_buf = DeviceReplayBuffer("imagined", cap, O, K, A, max_transitions=cap * H)
    for n in (6, 7, 13, 3):  # the third batch alone exceeds the capacity
        starts = np.zeros((n, O))
        for e in range(n):
            for c in range(3):
                starts[e, c * 16 + rng.integers(16)] = 1.0
            starts[e, 48 + e % 3] = 1.0
        u = rng.random((n, H + 1, K))
        out = im.imagine_device(starts, np.arange(n) % 5, H, uniforms=u)
        dev_buf.push_imagined(out)
        host = im.imagine_trajectories([SimpleNamespace(vec=starts[e], step=e % 5, task_id=0)
                                        for e in range(n)], H, uniforms=u)
        for t in host:
            if t is not None:
                host_buf.push(t)
        assert dev_buf.stats() == host_buf.stats()
        a, _, _ = dev_buf.gather(list(dev_buf._items))
        c, _, _ = host_buf.gather(list(host_buf._items))
        for k in a:
            np.testing.assert_array_equal(a[k].cpu().numpy(), c[k].cpu().numpy(), err_msg=k)
        np.testing.assert_allclose([h.episode_return for h in dev_buf._items],
                                   [h.episode_return for h in host_buf._items], rtol=1e-12,
                                   atol=1e-12)
        assert [(h.t_len, h.done) for h in dev_buf._items] == \
            [(h.t_len, h.done) for h in host_buf._items]


def test_span_ring_plan_does_not_mutate_on_failure():
    """A batch the arena cannot hold raises before any ring state changes
    (push_imagined checks both rings this way before touching its counters)."""
    from paper_2603_18464_b200.errors import DimensionError
    r = SpanRing(10)
    r.alloc(4, "a")
    state = (r.head, list(r._starts), dict(r._spans))
    with pytest.raises(DimensionError):
        r.plan([4, 4, 4])  # 12 slots > 10: the spans would overlap each other
    with pytest.raises(DimensionError):
        r.alloc_many([4, 4, 4], ["x", "y", "z"])
    assert (r.head, list(r._starts), dict(r._spans)) == state
    starts, _, head = r.plan([3, 3])
    assert starts == [4, 7] and head == 10 and r.head == 4


def test_world_model_kind_is_rejected():
    from paper_2603_18464_b200.replay import BufferKindError, DeviceReplayBuffer
    with pytest.raises(BufferKindError):
        DeviceReplayBuffer("world_model", 4, 3, 2, 7, max_transitions=16)


@pytest.mark.gpu
def test_gather_of_evicted_handle_is_a_dropped_batch():
    """A sampled handle evicted before the build gives a None batch (the
    reference Prefetcher drops None batches) instead of an exception or mixed
    data; the trainer's build returns None for it."""
    from paper_2603_18464_b200.replay import DeviceReplayBuffer
    from paper_2603_18464_b200.workload import synthetic_trajectories
    rng = np.random.default_rng(3)
    buf = DeviceReplayBuffer("main", 2, 6, 2, 8, max_transitions=64)
    for t in synthetic_trajectories(rng, [3, 4], [True, False], 2, 8, 6):
        buf.push(t)
    picks = buf.sample(2, np.random.default_rng(0))
    assert buf.gather(picks) is not None
    for t in synthetic_trajectories(rng, [5, 2], [False, True], 2, 8, 6):
        buf.push(t)  # FIFO: both sampled handles leave
    assert buf.gather(picks) is None


@pytest.mark.gpu
def test_push_imagined_too_large_for_arena_changes_nothing():
    import torch
    from paper_2603_18464_b200.errors import DimensionError
    from paper_2603_18464_b200.replay import DeviceReplayBuffer
    O, K, A, H, n = 5, 2, 3, 4, 6
    buf = DeviceReplayBuffer("imagined", 8, O, K, A, max_transitions=10)
    out = {"status": torch.zeros(n, dtype=torch.int32), "t_len": torch.full((n,), H),
           "done": torch.zeros(n, dtype=torch.bool), "rewards": torch.zeros(n, H),
           "observations": torch.zeros(n, H + 1, O)}
    before = buf.stats()
    with pytest.raises(DimensionError):
        buf.push_imagined(out)  # 24 transitions do not fit a 10-transition arena
    assert buf.stats() == before and len(buf) == 0
