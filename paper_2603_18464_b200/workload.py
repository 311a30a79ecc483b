"""Ragged trajectory batches: CSR packing and seeded synthetic workloads.

The packed layout (`PackedBatch`) is the wire format of the drop-in
boundary: the reference's `list[Trajectory]` (rollout.py:31-86) flattened
in trajectory order exactly as `Trainer.build_train_batch` concatenates it
(trainer.py:365-391), plus the T+1-frame arrays that revaluation needs.

  traj_off  i64[n+1]   transition offsets (trajectory s owns [off[s], off[s+1]))
  frames    f32[F, O]  all T+1 observations of every trajectory, F = N + n;
                       frame row of transition t of trajectory s is t + s
  steps     i32[F]     step index of every frame
  values    f32[F]     stored values with the bootstrap value appended
                       (trainer.py:369, used when revalue is off)
  tokens    i32[N, K]
  rewards   f32[N]
  mu        f32[N, K, A] behavior logits
  done      u8[n], real u8[n], behavior_version i64[n]

Synthetic generators follow SURVEY.md §8(d): N(0,1) rewards/values/logits/
observations, U[0, A) tokens; cfg2 lengths are the LIBERO-Long-like mix
(50% successes with T ~ U[1, 520] and done=True, 50% truncations at T=520).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DimensionError
from .types import Trajectory


@dataclass
class PackedBatch:
    traj_off: np.ndarray
    frames: np.ndarray
    steps: np.ndarray
    values: np.ndarray
    tokens: np.ndarray
    rewards: np.ndarray
    mu: np.ndarray
    done: np.ndarray
    real: np.ndarray
    behavior_version: np.ndarray

    @property
    def n_traj(self) -> int:
        return int(self.traj_off.shape[0] - 1)

    @property
    def n_transitions(self) -> int:
        return int(self.traj_off[-1])

    @property
    def n_frames(self) -> int:
        return self.n_transitions + self.n_traj

    @property
    def chunk_len(self) -> int:
        return int(self.tokens.shape[1])

    @property
    def n_actions(self) -> int:
        return int(self.mu.shape[2])

    @property
    def obs_dim(self) -> int:
        return int(self.frames.shape[1])

    def frame_rows(self) -> np.ndarray:
        """Frame row of every transition (t + trajectory index)."""
        lens = np.diff(self.traj_off)
        return (np.arange(self.n_transitions) + np.repeat(np.arange(self.n_traj), lens)).astype(
            np.int64)

    def transition_frame_mask(self) -> np.ndarray:
        mask = np.ones(self.n_frames, dtype=bool)
        mask[self.traj_off[1:] + np.arange(self.n_traj)] = False
        return mask

    def nbytes(self) -> int:
        return sum(a.nbytes for a in (self.traj_off, self.frames, self.steps, self.values,
                                      self.tokens, self.rewards, self.mu, self.done))


class PinnedStaging:
    """Grow-only page-locked host buffers for the packed batch: the pack writes
    float32 straight into them and the upload is one asynchronous DMA per field
    (a pageable source makes every host-to-device copy synchronous and staged)."""

    def __init__(self) -> None:
        self._bufs: dict = {}

    def get(self, name: str, shape, dtype) -> np.ndarray:
        import torch
        n = int(np.prod(shape))
        tdt = {np.float32: torch.float32, np.int32: torch.int32, np.int64: torch.int64,
               np.uint8: torch.uint8}[np.dtype(dtype).type]
        buf = self._bufs.get(name)
        if buf is None or buf.dtype != tdt or buf.numel() < n:
            buf = torch.empty(max(n, 1) + (n >> 3), dtype=tdt, pin_memory=True)
            self._bufs[name] = buf
        return buf[:n].numpy().reshape(shape)


def _pack_rows(trajs, lens, off, frames, steps, values, tokens, rewards, mu, lo, hi) -> None:
    """Trajectories [lo, hi) into their CSR rows (float64 -> float32 casts in place)."""
    for s in range(lo, hi):
        t = trajs[s]
        a, b = int(off[s]), int(off[s + 1])
        fa, fb = a + s, b + s + 1
        np.copyto(frames[fa:fb], np.asarray(t.observations), casting="unsafe")
        np.copyto(steps[fa:fb], np.asarray(t.steps), casting="unsafe")
        np.copyto(values[fa:fb - 1], np.asarray(t.values), casting="unsafe")
        values[fb - 1] = t.bootstrap_value
        np.copyto(tokens[a:b], np.asarray(t.tokens), casting="unsafe")
        np.copyto(rewards[a:b], np.asarray(t.rewards), casting="unsafe")
        np.copyto(mu[a:b], np.asarray(t.behavior_logits), casting="unsafe")


def _pack_threads() -> int:
    """Every host core (the pack is bound by host memory bandwidth; measured on
    the 16-core box: 8 threads 84 GB/s, 16 threads 110 GB/s)."""
    import os
    return max(1, min(32, os.cpu_count() or 8))


def pack_trajectories(trajs, staging: PinnedStaging | None = None,
                      threads: int | None = None, chunks: int = 1,
                      on_chunk=None) -> PackedBatch:
    """Flatten duck-typed trajectories into the CSR wire format (float32).

    Every field is written once, cast in place, into preallocated rows (with
    `staging`: page-locked buffers, so the upload is asynchronous DMA); the
    copies run on a thread pool over trajectories (NumPy releases the GIL).
    chunks > 1: the trajectories are packed in that many consecutive ranges
    (balanced by transitions) and on_chunk(lo, hi, off, frames, mu) is called
    after each, so the caller can start that range's upload while the next one
    is packed."""
    if not trajs:
        raise DimensionError("cannot pack an empty trajectory list")
    k = int(np.asarray(trajs[0].tokens).shape[1])
    a = int(np.asarray(trajs[0].behavior_logits).shape[2])
    o = int(np.asarray(trajs[0].observations).shape[1])
    lens = np.array([int(np.asarray(t.tokens).shape[0]) for t in trajs], dtype=np.int64)
    if np.any(lens < 1):
        raise DimensionError("every trajectory needs at least one decision")
    for t in trajs:
        if (np.asarray(t.tokens).shape[1] != k or np.asarray(t.behavior_logits).shape[2] != a
                or np.asarray(t.observations).shape[1] != o):
            raise DimensionError("trajectories disagree on chunk_len / n_actions / obs_dim")
    n = len(trajs)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    for t in trajs:
        st = np.asarray(t.steps)
        if st.size and (st.min() < np.iinfo(np.int32).min or st.max() > np.iinfo(np.int32).max):
            raise DimensionError("step index outside int32 range")
    N = int(off[-1])
    F = N + n
    if staging is None:
        alloc = lambda name, shape, dt: np.empty(shape, dtype=dt)
    else:
        alloc = staging.get
    frames = alloc("frames", (F, o), np.float32)
    steps = alloc("steps", (F,), np.int32)
    values = alloc("values", (F,), np.float32)
    tokens = alloc("tokens", (N, k), np.int32)
    rewards = alloc("rewards", (N,), np.float32)
    mu = alloc("mu", (N, k, a), np.float32)
    args = (trajs, lens, off, frames, steps, values, tokens, rewards, mu)
    # consecutive chunks of trajectories (balanced by transition count)
    cb = sorted(set([0] + np.searchsorted(off, np.linspace(0, N, max(1, chunks) + 1)[1:-1]).tolist()
                    + [n]))
    ex = None
    try:
        for lo, hi in zip(cb[:-1], cb[1:]):
            n_c = int(off[hi] - off[lo])
            workers = min(threads or _pack_threads(), max(1, n_c // 512), hi - lo)
            if workers <= 1:
                _pack_rows(*args, lo, hi)
            else:
                if ex is None:
                    from concurrent.futures import ThreadPoolExecutor
                    ex = ThreadPoolExecutor(threads or _pack_threads())
                # contiguous trajectory ranges balanced by transition count
                cuts = np.searchsorted(off, np.linspace(off[lo], off[hi], workers + 1)[1:-1]).tolist()
                bounds = [lo] + [min(max(c, lo), hi) for c in cuts] + [hi]
                list(ex.map(lambda i: _pack_rows(*args, bounds[i], bounds[i + 1]),
                            range(workers)))
            if on_chunk is not None:
                on_chunk(lo, hi, off, frames, mu)
    finally:
        if ex is not None:
            ex.shutdown()
    return PackedBatch(
        traj_off=off, frames=frames, steps=steps, values=values, tokens=tokens, rewards=rewards,
        mu=mu,
        done=np.array([bool(t.done) for t in trajs], dtype=np.uint8),
        real=np.array([t.source == "real" for t in trajs], dtype=np.uint8),
        behavior_version=np.array([int(t.behavior_version) for t in trajs], dtype=np.int64),
    )


def libero_long_lengths(rng: np.random.Generator, n: int, horizon: int = 520,
                        pure_uniform: bool = False):
    """(lengths, done) for the cfg2 mix."""
    if pure_uniform:
        lens = rng.integers(1, horizon + 1, size=n)
        return lens.astype(np.int64), rng.random(n) < 0.5
    success = rng.random(n) < 0.5
    lens = np.where(success, rng.integers(1, horizon + 1, size=n), horizon)
    return lens.astype(np.int64), success


def synthetic_trajectories(rng: np.random.Generator, lengths, done, chunk_len: int,
                           n_actions: int, obs_dim: int, n_steps: int | None = None,
                           imagined_every: int = 0, behavior_version: int = 0) -> list:
    """Seeded float64 trajectories (one Generator draw order, trajectory-major)."""
    out = []
    for i, (t_len, d) in enumerate(zip(lengths, done)):
        t_len = int(t_len)
        start = 0 if n_steps is None else int(rng.integers(0, max(1, n_steps - t_len)))
        out.append(Trajectory(
            task_id=i % 3,
            source="imagined" if imagined_every and i % imagined_every == 1 else "real",
            observations=rng.normal(size=(t_len + 1, obs_dim)),
            steps=np.arange(start, start + t_len + 1),
            tokens=rng.integers(0, n_actions, size=(t_len, chunk_len)),
            rewards=rng.normal(size=t_len),
            behavior_logits=rng.normal(size=(t_len, chunk_len, n_actions)),
            values=rng.normal(size=t_len),
            bootstrap_value=float(rng.normal()),
            done=bool(d),
            behavior_version=behavior_version,
        ))
    return out


def synthetic_packed(seed: int, lengths, done, chunk_len: int, n_actions: int, obs_dim: int,
                     max_step: int | None = None) -> PackedBatch:
    """Fast float32 generator straight into the packed layout (bench sizes)."""
    rng = np.random.default_rng(seed)
    lens = np.asarray(lengths, dtype=np.int64)
    n = lens.shape[0]
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    N = int(off[-1])
    F = N + n
    steps = (np.arange(F) - np.repeat(off[:-1] + np.arange(n), lens + 1)).astype(np.int32)
    if max_step is not None:
        steps = np.minimum(steps, max_step).astype(np.int32)
    f32 = np.float32
    return PackedBatch(
        traj_off=off,
        frames=rng.standard_normal((F, obs_dim), dtype=f32),
        steps=steps,
        values=rng.standard_normal(F, dtype=f32),
        tokens=rng.integers(0, n_actions, size=(N, chunk_len), dtype=np.int32),
        rewards=rng.standard_normal(N, dtype=f32),
        mu=rng.standard_normal((N, chunk_len, n_actions), dtype=f32),
        done=np.asarray(done, dtype=np.uint8),
        real=np.ones(n, dtype=np.uint8),
        behavior_version=np.zeros(n, dtype=np.int64),
    )


def unpack_trajectories(pb: PackedBatch) -> list:
    """Inverse of pack_trajectories (float64 views of the packed values)."""
    out = []
    for s in range(pb.n_traj):
        a, b = int(pb.traj_off[s]), int(pb.traj_off[s + 1])
        fa, fb = a + s, b + s + 1
        out.append(Trajectory(
            task_id=0, source="real" if pb.real[s] else "imagined",
            observations=pb.frames[fa:fb].astype(np.float64),
            steps=pb.steps[fa:fb].astype(np.int64),
            tokens=pb.tokens[a:b].astype(np.int64),
            rewards=pb.rewards[a:b].astype(np.float64),
            behavior_logits=pb.mu[a:b].astype(np.float64),
            values=pb.values[fa:fb - 1].astype(np.float64),
            bootstrap_value=float(pb.values[fb - 1]),
            done=bool(pb.done[s]),
            behavior_version=int(pb.behavior_version[s]),
        ))
    return out
