"""The device-resident TrainBatch (reference: buffers.py:97-122).

Everything the optimizer step needs stays in HBM in "frame space": the T+1
observations of every trajectory are kept as one [F, O] matrix (F = N + n),
and `frame_of[i]` maps transition i to its frame row, so revaluation and the
training forward share one observation upload and nothing is re-gathered.
The reference's flat host arrays (`obs`, `steps`, `tokens`, `behavior_logp`,
`advantages`, `value_targets`) are materialized lazily, only if read.
"""

from __future__ import annotations

import numpy as np
import torch

from . import ops
from .errors import DimensionError


class DeviceTrainBatch:
    def __init__(self, *, frames, steps, tokens, frame_of, lp_old, adv, ret, n_actions: int,
                 chunk_len: int, critic_version: int, n_real: int, n_imagined: int,
                 norm_mean: float, norm_std: float, norm_count: int, shard_sizes: tuple,
                 behavior_lag_mean: float, finite: bool = True, prev_group=None,
                 step_group=None, n_steps: int | None = None) -> None:
        self.frames = frames
        self.frame_steps = steps
        self.tokens_dev = tokens
        self.frame_of = frame_of
        self.lp_old = lp_old
        self.adv = adv
        self.ret = ret
        self.n_actions = int(n_actions)
        self.chunk_len = int(chunk_len)
        self.critic_version = critic_version
        self.n_real = n_real
        self.n_imagined = n_imagined
        self.norm_mean = norm_mean
        self.norm_std = norm_std
        self.norm_count = norm_count
        self.shard_sizes = tuple(shard_sizes)
        self.behavior_lag_mean = behavior_lag_mean
        self._finite = bool(finite)
        self.prev_group = prev_group
        self.pk_group = None
        self.step_group = step_group
        self.frame_step_group = None  # e_step grouping over frames (frame-space value path)
        self.n_steps_f = None
        # (param generation, h1, h2) from revaluation; reused by train_step when
        # the parameters have not changed since the batch was built
        self.h_cache = None
        self.n_steps = n_steps
        self._host = {}

    # -- sizes ------------------------------------------------------------------
    @property
    def n_transitions(self) -> int:
        return int(self.frame_of.shape[0])

    @property
    def n_frames(self) -> int:
        return int(self.frames.shape[0])

    @property
    def n_tokens(self) -> int:
        return self.n_transitions * self.chunk_len

    def check_finite(self) -> bool:
        return self._finite

    # -- lazily materialized reference fields (float64 / int64 numpy) ------------
    def _get(self, key, fn):
        if key not in self._host:
            self._host[key] = fn()
        return self._host[key]

    @property
    def obs(self) -> np.ndarray:
        return self._get("obs", lambda: self.frames.index_select(
            0, self.frame_of.long()).double().cpu().numpy())

    @property
    def steps(self) -> np.ndarray:
        return self._get("steps", lambda: self.frame_steps.index_select(
            0, self.frame_of.long()).long().cpu().numpy())

    @property
    def tokens(self) -> np.ndarray:
        return self._get("tokens", lambda: self.tokens_dev.view(-1, self.chunk_len)
                         .long().cpu().numpy())

    @property
    def behavior_logp(self) -> np.ndarray:
        return self._get("lp", lambda: self.lp_old.view(-1, self.chunk_len).double().cpu().numpy())

    @property
    def advantages(self) -> np.ndarray:
        return self._get("adv", lambda: self.adv.double().cpu().numpy())

    @property
    def value_targets(self) -> np.ndarray:
        return self._get("ret", lambda: self.ret.double().cpu().numpy())

    def ensure_groupings(self, n_steps: int, bad_count, factorized: bool = True,
                         frame_space: bool = False, pk_cpb: int = 0) -> None:
        """Stable key sorts for the deterministic scatter-adds (fixed per batch):
        (prev token, chunk position) for the factorized head, prev token for the
        materialized head, step index for the value head's e_step (over
        transitions, or over all frames when the value backward runs in frame
        space).  pk_cpb > 0: the (prev, k) sort is frame-blocked (blocks of
        pk_cpb 4096-token chunks) for the dz-recomputing grouped sums."""
        N, K, A = self.n_transitions, self.chunk_len, self.n_actions
        if factorized and (self.pk_group is None or self.pk_group.cpb != pk_cpb):
            # the scatter also writes the inverse permutation (the loss kernel's
            # scalar positions) when the grouping is frame-blocked
            # key prev * K + k; every transition's token 0 falls in the chunk-start
            # key A * K (1/K of all tokens): the heavy key of the fold
            self.pk_group = ops.Grouping(ops.prev_keys(self.tokens_dev, N, K, A, with_pos=True),
                                         (A + 1) * K, cpb=pk_cpb, rows=pk_cpb > 0,
                                         heavy_key=A * K)
        if not factorized and self.prev_group is None:
            self.prev_group = ops.Grouping(ops.prev_keys(self.tokens_dev, N, K, A), A + 1)
        if frame_space:
            if self.frame_step_group is None or self.n_steps_f != n_steps:
                keys = ops.step_keys(self.frame_steps, None, self.n_frames, n_steps, bad_count)
                self.frame_step_group = ops.Grouping(keys, n_steps)
                self.n_steps_f = n_steps
        elif self.step_group is None or self.n_steps != n_steps:
            keys = ops.step_keys(self.frame_steps, self.frame_of, N, n_steps, bad_count)
            self.step_group = ops.Grouping(keys, n_steps)
            self.n_steps = n_steps

    @classmethod
    def from_host(cls, batch, device) -> "DeviceTrainBatch":
        """Upload a reference-shaped host TrainBatch (buffers.py:97-114)."""
        obs = np.asarray(batch.obs)
        N = obs.shape[0]
        tokens = np.asarray(batch.tokens)
        if tokens.ndim != 2 or tokens.shape[0] != N:
            raise DimensionError(f"tokens shape {tokens.shape} inconsistent with N={N}")
        K = tokens.shape[1]
        lp = np.asarray(batch.behavior_logp)
        if lp.shape != (N, K):
            raise DimensionError(f"behavior_logp shape {lp.shape} != {(N, K)}")
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(device)
        finite = all(np.all(np.isfinite(np.asarray(a))) for a in
                     (obs, lp, batch.advantages, batch.value_targets))
        out = cls(
            frames=ops.upload_pitched(obs.astype(np.float32), device), steps=t(batch.steps, np.int32),
            tokens=t(tokens.reshape(-1), np.int32),
            frame_of=torch.arange(N, dtype=torch.int32, device=device),
            lp_old=t(lp.reshape(-1), np.float32), adv=t(batch.advantages, np.float32),
            ret=t(batch.value_targets, np.float32), n_actions=-1, chunk_len=K,
            critic_version=batch.critic_version, n_real=batch.n_real,
            n_imagined=batch.n_imagined, norm_mean=batch.norm_mean, norm_std=batch.norm_std,
            norm_count=batch.norm_count, shard_sizes=batch.shard_sizes,
            behavior_lag_mean=batch.behavior_lag_mean, finite=finite)
        old = getattr(batch, "old_values", None)  # rollout-time V (value clipping)
        if old is not None:
            out.v_old = t(old, np.float32)
        return out
