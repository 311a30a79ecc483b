"""On-device replay buffer for the train-batch prefetcher.

Reference: `ReplayBuffer` (buffers.py:44-94) -- a bounded FIFO of immutable
trajectories, uniform sampling with replacement -- feeding `Prefetcher`
(buffers.py:125-186), whose builder packs the sampled trajectories on the host
and (here) uploads them every batch.  `DeviceReplayBuffer` keeps the same API
(`push`, `sample(n, rng)`, `stats`, `len`, kind checks, FIFO eviction at
`capacity` trajectories) but copies each trajectory into HBM once, on push, into
contiguous frame / transition spans of a ring arena.  `sample` draws exactly as
the reference (`rng.integers`) and returns `DeviceTrajectory` handles; the
trainer's `build_train_batch` recognises them and assembles the packed batch
with on-device row gathers (`gather`), so neither the host pack nor the
per-batch host-to-device copy sits on the build path.  The reference
`Prefetcher` runs unchanged on top (it only calls stats / sample / builder).
"""

from __future__ import annotations

import bisect
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .errors import DimensionError

_ACCEPTED_SOURCE = {"main": "real", "world_model": "real", "imagined": "imagined"}


class BufferKindError(ValueError):
    """A trajectory of the wrong source for the buffer (buffers.py:30-31)."""


@dataclass(frozen=True)
class BufferStats:  # buffers.py:34-40
    size: int
    pushed: int
    sampled: int
    evicted: int


class SpanRing:
    """Ring allocator of contiguous spans (host logic, CPU-testable).

    alloc(n) returns the start of n contiguous slots; a span never wraps (it
    restarts at 0 when the tail is too short) and every live span it overlaps
    is reported for eviction (oldest first).  With an arena of at least
    capacity x (longest trajectory + 1) slots no span is ever evicted this way,
    and the buffer's contents (hence its sampling) follow the reference's FIFO
    exactly.  Live spans never overlap, so they are kept sorted by start and an
    alloc / release costs a bisection, not a scan of every live span (a push of
    a 4096-episode imagination batch into an 8192-episode buffer was quadratic)."""

    def __init__(self, size: int) -> None:
        self.size = int(size)
        self.head = 0
        self._starts: list = []   # sorted starts of the live spans
        self._spans: dict = {}    # start -> (length, owner, allocation seq)
        self._where: dict = {}    # id(owner) -> start
        self._seq = 0

    def alloc(self, n: int, owner) -> tuple:
        if n > self.size:
            raise DimensionError(f"span of {n} exceeds the arena ({self.size})")
        start = self.head if self.head + n <= self.size else 0
        end = start + n
        self.head = end
        if n == 0:  # occupies nothing, overlaps nothing
            return start, []
        st = self._starts
        i = bisect.bisect_left(st, start)
        if i > 0 and st[i - 1] + self._spans[st[i - 1]][0] > start:
            i -= 1
        j = i
        while j < len(st) and st[j] < end:
            j += 1
        gone = [self._spans.pop(x) for x in st[i:j]]
        del st[i:j]
        for _, o, _ in gone:
            del self._where[id(o)]
        st.insert(i, start)
        self._spans[start] = (n, owner, self._seq)
        self._where[id(owner)] = start
        self._seq += 1
        return start, [o for _, o, _ in sorted(gone, key=lambda g: g[2])]

    def plan(self, ns) -> tuple:
        """Placement of spans of lengths ns from the current head, without
        changing the ring: (starts, runs, new head).  Raises DimensionError when
        a span exceeds the arena or the new spans would overlap each other (the
        arena is smaller than the batch), so callers can check a batch fits
        before mutating anything."""
        size = self.size
        ns_a = np.asarray(ns, dtype=np.int64).reshape(-1)
        k = len(ns_a)
        if k and int(ns_a.max()) > size:
            raise DimensionError(f"span of {int(ns_a.max())} exceeds the arena ({size})")
        starts_a = np.empty(k, dtype=np.int64)
        runs, head, i = [], self.head, 0
        while i < k:  # one pass per wrap: every span that fits from head on
            ends = head + np.cumsum(ns_a[i:])
            over = np.flatnonzero(ends > size)
            m = int(over[0]) if len(over) else k - i
            if m == 0:  # span i does not fit in the tail: it restarts at 0
                head = 0
                continue
            starts_a[i:i + m] = ends[:m] - ns_a[i:i + m]
            if runs and runs[-1][1] == head:
                runs[-1][1] = int(ends[m - 1])
            else:
                runs.append([head, int(ends[m - 1])])
            head = int(ends[m - 1])
            i += m
        starts = starts_a.tolist()
        for a in range(len(runs)):
            for b in range(a):
                if runs[a][0] < runs[b][1] and runs[b][0] < runs[a][1] \
                        and runs[a][0] < runs[a][1] and runs[b][0] < runs[b][1]:
                    raise DimensionError("the replay arena is smaller than one batch")
        return starts, runs, head

    def alloc_many(self, ns, owners) -> tuple:
        """alloc(n, owner) for every pair in order, as one operation: the starts,
        and every previously live span any of them overlaps (oldest first).  The
        new spans must not overlap each other (DimensionError: the arena is
        smaller than the batch; the ring is then unchanged)."""
        starts, runs, head = self.plan(ns)
        ns_a = np.asarray(ns, dtype=np.int64).reshape(-1)
        st, gone = self._starts, []
        for r0, r1 in runs:
            if r0 == r1:
                continue
            i = bisect.bisect_left(st, r0)
            if i > 0 and st[i - 1] + self._spans[st[i - 1]][0] > r0:
                i -= 1
            j = i
            while j < len(st) and st[j] < r1:
                j += 1
            gone += [self._spans.pop(x) for x in st[i:j]]
            del st[i:j]
        for _, o, _ in gone:
            del self._where[id(o)]
        nz = np.flatnonzero(ns_a).tolist()
        s_nz = [starts[q] for q in nz]
        o_nz = [owners[q] for q in nz]
        seq = self._seq
        self._spans.update(zip(s_nz, zip(ns_a[nz].tolist(), o_nz, range(seq, seq + len(nz)))))
        self._where.update(zip(map(id, o_nz), s_nz))
        st.extend(s_nz)
        st.sort()
        self._seq = seq + len(nz)
        self.head = head
        return starts, [o for _, o, _ in sorted(gone, key=lambda g: g[2])]

    def release_many(self, owners) -> None:
        """release(o) for every o, with one pass over the live spans."""
        gone = set()
        for o in owners:
            x = self._where.pop(id(o), None)
            if x is not None:
                del self._spans[x]
                gone.add(x)
        if gone:
            self._starts = [x for x in self._starts if x not in gone]

    def release(self, owner) -> None:
        x = self._where.pop(id(owner), None)
        if x is None:
            return
        del self._spans[x]
        del self._starts[bisect.bisect_left(self._starts, x)]


def _spans(starts: np.ndarray, lens: np.ndarray) -> np.ndarray:
    """Concatenation of arange(s, s + n) over (starts, lens), vectorized."""
    total = int(lens.sum())
    base = np.repeat(starts - (np.cumsum(lens) - lens), lens)
    return base + np.arange(total, dtype=np.int64)


class DeviceTrajectory:
    """Handle of a trajectory resident in a DeviceReplayBuffer arena (duck-types
    the reference Trajectory's metadata: t_len, done, source, task_id,
    behavior_version, episode_return)."""

    __slots__ = ("buffer", "f0", "t0", "t_len", "done", "source", "task_id", "behavior_version",
                 "episode_return", "alive")

    def __init__(self, buffer, f0, t0, traj) -> None:
        self.buffer = buffer
        self.f0, self.t0 = f0, t0
        self.t_len = int(traj.tokens.shape[0])
        self.done = bool(traj.done)
        self.source = traj.source
        self.task_id = int(getattr(traj, "task_id", 0))
        self.behavior_version = int(getattr(traj, "behavior_version", 0))
        self.episode_return = float(np.sum(traj.rewards))
        self.alive = True

    @classmethod
    def imagined(cls, buffer, t_len: int, done: bool, task_id: int, version: int,
                 episode_return: float):
        """Handle of an imagined episode from its scalars (push_imagined's batch path)."""
        h = cls.__new__(cls)
        h.buffer, h.f0, h.t0 = buffer, 0, 0
        h.t_len, h.done, h.source = t_len, done, "imagined"
        h.task_id, h.behavior_version = task_id, version
        h.episode_return, h.alive = episode_return, True
        return h


class DeviceReplayBuffer:
    """Bounded FIFO of trajectories resident in HBM, uniform sampling."""

    def __init__(self, kind: str, capacity: int, obs_dim: int, chunk_len: int, n_actions: int,
                 max_transitions: int, device=None) -> None:
        if kind not in _ACCEPTED_SOURCE:
            raise BufferKindError(f"unknown buffer kind {kind!r}")
        if kind == "world_model":
            # the world-model sub-steps read observations / tokens of the sampled
            # trajectories on the host (world_model.obs_model_data): that buffer
            # stays a host ReplayBuffer
            raise BufferKindError("the world-model buffer must be a host ReplayBuffer "
                                  "(its sub-steps read trajectory fields on the host)")
        if capacity < 1:
            raise ValueError(f"capacity must be >= 1, got {capacity}")
        self.kind, self.capacity = kind, int(capacity)
        self.O, self.K, self.A = int(obs_dim), int(chunk_len), int(n_actions)
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        cap_t = int(max_transitions)
        cap_f = cap_t + self.capacity  # a bootstrap frame per trajectory
        f32 = torch.float32
        self.frames = ops.alloc_pitched(cap_f, self.O, dev)   # [cap_f, O] view, aligned rows
        self.steps = torch.zeros(cap_f, dtype=torch.int32, device=dev)
        self.values = torch.zeros(cap_f, dtype=f32, device=dev)  # values + bootstrap last
        self.rewards = torch.zeros(cap_t, dtype=f32, device=dev)
        self.tokens = torch.zeros(cap_t, self.K, dtype=torch.int32, device=dev)
        self.mu = torch.zeros(cap_t, self.K * self.A, dtype=f32, device=dev)
        self._fring, self._tring = SpanRing(cap_f), SpanRing(cap_t)
        self._items: list = []
        self._lock = threading.Lock()
        self._ready = None  # event after the last queued arena write
        self._pushed = self._sampled = self._evicted = 0

    # -- reference API ---------------------------------------------------------------
    def push(self, traj) -> None:
        """Append one completed trajectory (one host-to-device copy per field)."""
        expected = _ACCEPTED_SOURCE[self.kind]
        if traj.source != expected:
            raise BufferKindError(
                f"buffer {self.kind!r} accepts source {expected!r}, got {traj.source!r}")
        T = int(traj.tokens.shape[0])
        obs = np.asarray(traj.observations)
        if obs.shape != (T + 1, self.O) or np.asarray(traj.behavior_logits).shape != (T, self.K,
                                                                                        self.A):
            raise DimensionError("trajectory shapes do not match the buffer")
        if T + 1 > self._fring.size or T > self._tring.size:
            raise DimensionError(f"a trajectory of {T} steps exceeds the replay arena")
        with self._lock:
            if len(self._items) >= self.capacity:
                self._evict(self._items[0])
            h = DeviceTrajectory(self, 0, 0, traj)
            f0, ev_f = self._fring.alloc(T + 1, h)
            t0, ev_t = self._tring.alloc(T, h)
            for o in ev_f + ev_t:
                if o.alive:
                    self._evict(o)
            h.f0, h.t0 = f0, t0
            dev = self.device
            t = lambda a, dt: torch.tensor(np.asarray(a), dtype=dt).to(dev)
            self.frames[f0:f0 + T + 1].copy_(t(obs, torch.float32))
            self.steps[f0:f0 + T + 1].copy_(t(traj.steps, torch.int32))
            self.values[f0:f0 + T].copy_(t(traj.values, torch.float32))
            self.values[f0 + T] = float(traj.bootstrap_value)
            self.rewards[t0:t0 + T].copy_(t(traj.rewards, torch.float32))
            self.tokens[t0:t0 + T].copy_(t(traj.tokens, torch.int32))
            self.mu[t0:t0 + T].copy_(t(np.asarray(traj.behavior_logits).reshape(T, -1),
                                       torch.float32))
            self._ready = torch.cuda.Event()
            self._ready.record()
            self._items.append(h)
            self._pushed += 1

    def push_imagined(self, out: dict, task_ids=None, version: int = 0) -> int:
        """Push a batch of imagined episodes straight from `Imaginer.imagine_device`
        outputs (device tensors; rollout.py:345-362 builds the same records on the
        host): episodes with status 0 (the reference keeps them) enter in order,
        their spans filled by a handful of on-device row copies.  Returns the
        number pushed."""
        if self.kind != "imagined":
            raise BufferKindError(f"buffer {self.kind!r} does not accept imagined episodes")
        status = out["status"].cpu().numpy()
        t_len = out["t_len"].cpu().numpy()
        done = out["done"].cpu().numpy()
        rew = out["rewards"].double().sum(dim=1).cpu().numpy()
        H1 = out["observations"].shape[1]
        H = H1 - 1
        keep_all = np.flatnonzero(status == 0).tolist()
        n_keep = len(keep_all)
        # the reference's bounded FIFO: the oldest leave first; episodes of this
        # batch beyond the capacity would leave at once, so they never enter
        keep = keep_all[n_keep - self.capacity:] if n_keep > self.capacity else keep_all
        T_l = t_len[keep].astype(np.int64).tolist()
        with self._lock:
            # placement first: a batch the arena cannot hold raises here, before
            # any counter, eviction or ring state changes
            self._fring.plan([T + 1 for T in T_l])
            self._tring.plan(T_l)
            self._pushed += n_keep
            self._evicted += n_keep - len(keep)
            n_over = len(self._items) + len(keep) - self.capacity
            if n_over > 0:
                old = self._items[:n_over]
                for h in old:
                    h.alive = False
                self._fring.release_many(old)
                self._tring.release_many(old)
                del self._items[:n_over]
                self._evicted += n_over
            tid = (np.asarray(task_ids)[keep].astype(np.int64).tolist() if task_ids is not None
                   else [0] * len(keep))
            mk, v = DeviceTrajectory.imagined, int(version)
            # the episode return is the sum of one float64 (rollout.py:345-362 stores it)
            hs = [mk(self, T, d, t, v, r) for T, d, t, r in
                  zip(T_l, done[keep].astype(bool).tolist(), tid, rew[keep].tolist())]
            f0s, ev_f = self._fring.alloc_many([T + 1 for T in T_l], hs)
            t0s, ev_t = self._tring.alloc_many(T_l, hs)
            for o in ev_f + ev_t:
                if o.alive:
                    self._evict(o)
            for h, f0, t0 in zip(hs, f0s, t0s):
                h.f0, h.t0 = f0, t0
            if keep:
                # the arena rows are queued BEFORE the handles become visible to
                # sample(); consumers on other streams wait on the event (gather)
                self._copy_imagined(out, keep, t_len, f0s, t0s, H1)
                self._ready = torch.cuda.Event()
                self._ready.record()
            self._items.extend(hs)
        return n_keep

    def _copy_imagined(self, out, keep, t_len, f0s, t0s, H1) -> None:
        H = H1 - 1
        dev = self.device
        ke = np.asarray(keep, dtype=np.int64)
        T = t_len[ke].astype(np.int64)
        f0a, t0a = np.asarray(f0s, dtype=np.int64), np.asarray(t0s, dtype=np.int64)
        ix = lambda a: torch.from_numpy(a).to(dev)
        sf, df = ix(_spans(ke * H1, T + 1)), ix(_spans(f0a, T + 1))
        st, dt = ix(_spans(ke * H, T)), ix(_spans(t0a, T))
        dst_v = _spans(f0a, T)  # values of transitions sit on their frames
        boot_dst, boot_src = (f0a + T).tolist(), keep
        O, K, A = self.O, self.K, self.A
        obs = out["observations"].reshape(-1, O).float()
        self.frames.index_copy_(0, df, obs.index_select(0, sf))
        self.steps.index_copy_(0, df, out["steps"].reshape(-1).index_select(0, sf).int())
        vals = out["values"].reshape(-1).float()
        if st.numel():
            self.values.index_copy_(0, ix(dst_v), vals.index_select(0, st))
        bd = torch.tensor(boot_dst, dtype=torch.int64, device=dev)
        self.values.index_copy_(0, bd, out["bootstrap_value"].float().index_select(
            0, torch.tensor(boot_src, dtype=torch.int64, device=dev)))
        if st.numel():
            self.rewards.index_copy_(0, dt, out["rewards"].reshape(-1).float().index_select(0, st))
            self.tokens.index_copy_(0, dt, out["tokens"].reshape(-1, K).int().index_select(0, st))
            self.mu.index_copy_(0, dt, out["behavior_logits"].reshape(-1, K * A).float()
                                .index_select(0, st))

    def _evict(self, h) -> None:
        h.alive = False
        self._items.remove(h)
        self._fring.release(h)
        self._tring.release(h)
        self._evicted += 1

    def sample(self, n: int, rng: np.random.Generator):
        """n uniform picks with replacement; None signals not-ready (buffers.py:74-86)."""
        if n < 0:
            raise ValueError(f"sample size must be >= 0, got {n}")
        if n == 0:
            return []
        with self._lock:
            if len(self._items) < n:
                return None
            idx = rng.integers(0, len(self._items), size=n)
            picks = [self._items[i] for i in idx]
            self._sampled += n
        return picks

    def __len__(self) -> int:
        with self._lock:
            return len(self._items)

    def stats(self) -> BufferStats:
        with self._lock:
            return BufferStats(len(self._items), self._pushed, self._sampled, self._evicted)

    # -- batch assembly on the device --------------------------------------------------
    def gather(self, handles) -> dict:
        """Packed CSR batch (the layout of trainer.upload) of the sampled handles,
        by on-device row gathers of their arena spans; None (a dropped batch, as
        the reference Prefetcher handles a None from its builder) when a sampled
        trajectory was evicted before the batch was built.  The liveness check
        and the gathers are queued under the buffer lock, so a concurrent push
        cannot overwrite a span between the check and the reads."""
        with self._lock:
            if any(not h.alive for h in handles):
                return None
            if self._ready is not None:  # pushes queued on another stream
                torch.cuda.current_stream().wait_event(self._ready)
            return self._gather_locked(handles)

    def _gather_locked(self, handles):
        dev = self.device
        lens = np.array([h.t_len for h in handles], dtype=np.int64)
        n = len(handles)
        off = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(lens, out=off[1:])
        N = int(off[-1])
        lens_d = torch.from_numpy(lens).to(dev)
        f0 = torch.tensor([h.f0 for h in handles], dtype=torch.int64, device=dev)
        t0 = torch.tensor([h.t0 for h in handles], dtype=torch.int64, device=dev)
        off_d = torch.from_numpy(off).to(dev)
        # frame rows: f0[s] + j for j in [0, T_s]; transition rows: t0[s] + j, j < T_s
        fcount = lens_d + 1
        # output sizes known on the host: no device-to-host sync inside the gathers
        fstart = torch.repeat_interleave(f0 - (off_d[:-1] + torch.arange(n, device=dev)), fcount,
                                         output_size=N + n)
        fidx = fstart + torch.arange(N + n, device=dev)
        tstart = torch.repeat_interleave(t0 - off_d[:-1], lens_d, output_size=N)
        tidx = tstart + torch.arange(N, device=dev)
        frames = ops.alloc_pitched(N + n, self.O, dev)
        full = self.frames.as_strided((self.frames.shape[0], self.frames.stride(0)),
                                      (self.frames.stride(0), 1))  # the pitched rows
        torch.index_select(full, 0, fidx, out=frames.as_strided(
            (N + n, frames.stride(0)), (frames.stride(0), 1)))
        return {
            "traj_off": off_d,
            "frames": frames,
            "steps": self.steps.index_select(0, fidx),
            "values": self.values.index_select(0, fidx),
            "tokens": self.tokens.index_select(0, tidx).reshape(-1),
            "rewards": self.rewards.index_select(0, tidx),
            "mu": self.mu.index_select(0, tidx).reshape(N * self.K, self.A),
            "done": torch.tensor([h.done for h in handles], dtype=torch.uint8, device=dev),
        }, int(sum(h.source == "real" for h in handles)), \
            np.array([h.behavior_version for h in handles], dtype=np.int64)
