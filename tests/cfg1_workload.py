"""Seed-regenerable BASELINE cfg1 inputs (SURVEY.md §8(d) "cfg1").

64 trajectories x 128 steps, done alternating True/False, rewards
Bernoulli(0.02) * N(0, 1), N(0, 1) values / behavior logits / observations,
U[0, 256) tokens, obs 195, K = 7, A = 256.  The inputs are regenerated from
the seed on both sides (the golden maker, which runs the real reference, and
the GPU tests), so only the reference OUTPUTS are committed
(tests/golden/trainer_cfg1_full_*.npz).  Pure NumPy: no reference import.
"""

from __future__ import annotations

import numpy as np

N_TRAJ, T_LEN, K, A, O, D, MLP = 64, 128, 7, 256, 195, 64, 32
N_STEPS = T_LEN + 2  # value step table covers every frame (steps 0..T)


def cfg1_fields(seed: int, step: int, n_traj: int = N_TRAJ, t_len: int = T_LEN,
                version: int = 0) -> list[dict]:
    """Trajectory field dicts (reference `Trajectory` keywords, rollout.py:31-86)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, step, 1]))
    out = []
    for i in range(n_traj):
        r = rng.normal(size=t_len) * (rng.random(t_len) < 0.02)
        out.append(dict(
            task_id=i % 3, source="real",
            observations=rng.normal(size=(t_len + 1, O)),
            steps=np.arange(t_len + 1, dtype=np.int64),
            tokens=rng.integers(0, A, size=(t_len, K)),
            rewards=r,
            behavior_logits=rng.normal(size=(t_len, K, A)),
            values=rng.normal(size=t_len),
            bootstrap_value=float(rng.normal()),
            done=(i % 2 == 0),
            behavior_version=version,
            step_versions=np.full(t_len, version, dtype=np.int64)))
    return out


def cfg1_trajectories(seed: int, step: int, cls=None, **kw) -> list:
    """The same trajectories as objects of `cls` (default: this package's mirror)."""
    if cls is None:
        from paper_2603_18464_b200.types import Trajectory as cls
    fields = cfg1_fields(seed, step, **kw)
    names = set(getattr(cls, "__dataclass_fields__", {}) or fields[0])
    return [cls(**{k: v for k, v in f.items() if k in names}) for f in fields]
