"""Host-side record types mirroring the reference trainer boundary.

These exist so the GPU box (which has no reference checkout) can build
inputs for the drop-in trainer.  The trainer itself is duck-typed: any
object with the same attributes (e.g. the reference's own `Trajectory`
and `ModelBundle`) is accepted.

Mirrors:
  * `Trajectory`          — rollout.py:31-86
  * `ParamSet`            — numerics.py:32-72
  * `PolicyConfig/Model`  — models.py:65-110 (init draw order kept so a
                            seeded init matches the reference bit-for-bit)
  * `ValueConfig/Head`    — models.py:231-256
  * `ObsModelConfig/ObsModel`, `RewardModel` — models.py:321-381
  * `ModelBundle`         — models.py:388-403
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import DimensionError, NonFiniteError


@dataclass
class ParamSet:
    """Named float64 tensors plus a monotone optimizer-step counter."""

    tensors: dict
    version: int = 0

    def __post_init__(self) -> None:
        self.tensors = {k: np.asarray(v, dtype=np.float64) for k, v in self.tensors.items()}

    def copy(self) -> "ParamSet":
        return ParamSet({k: v.copy() for k, v in self.tensors.items()}, self.version)

    def __getitem__(self, name: str) -> np.ndarray:
        return self.tensors[name]

    def names(self) -> list:
        return list(self.tensors)

    def n_params(self) -> int:
        return int(sum(t.size for t in self.tensors.values()))

    def flatten(self) -> np.ndarray:
        return np.concatenate([self.tensors[k].ravel() for k in sorted(self.tensors)])

    def check_finite(self) -> None:
        for name, t in self.tensors.items():
            if not np.all(np.isfinite(t)):
                raise NonFiniteError(f"parameter tensor {name!r} contains non-finite values")


def _init_mlp(rng: np.random.Generator, dims: list, scale: float) -> dict:
    out = {}
    for i in range(len(dims) - 1):
        out[f"w{i}"] = rng.normal(0.0, scale / np.sqrt(dims[i]), size=(dims[i + 1], dims[i]))
        out[f"b{i}"] = np.zeros(dims[i + 1])
    return out


@dataclass(frozen=True)
class PolicyConfig:
    obs_dim: int
    hidden_dim: int = 64
    chunk_len: int = 4
    n_actions: int = 7
    vocab_size: int = 32
    action_start: int = 16
    init_scale: float = 0.1

    def __post_init__(self) -> None:
        if self.action_start + self.n_actions > self.vocab_size:
            raise DimensionError(
                f"action range [{self.action_start}, {self.action_start + self.n_actions}) "
                f"exceeds vocabulary size {self.vocab_size}")


class PolicyModel:
    """Parameter holder for the AR token policy (math lives on the GPU)."""

    def __init__(self, cfg: PolicyConfig, params: ParamSet) -> None:
        self.cfg = cfg
        self.params = params

    @classmethod
    def init(cls, rng: np.random.Generator, cfg: PolicyConfig) -> "PolicyModel":
        d, s = cfg.hidden_dim, cfg.init_scale
        bb = _init_mlp(rng, [cfg.obs_dim, d, d], s)
        full_head = rng.normal(0.0, s / np.sqrt(d), size=(cfg.vocab_size, d))
        lo, hi = cfg.action_start, cfg.action_start + cfg.n_actions
        tensors = {
            "w0": bb["w0"], "b0": bb["b0"], "w1": bb["w1"], "b1": bb["b1"],
            "e_prev": rng.normal(0.0, s, size=(cfg.n_actions + 1, d)),
            "e_pos": rng.normal(0.0, s, size=(cfg.chunk_len, d)),
            "w_head": full_head[lo:hi].copy(), "b_head": np.zeros(cfg.n_actions),
        }
        return cls(cfg, ParamSet(tensors))

    def with_params(self, params: ParamSet) -> "PolicyModel":
        return PolicyModel(self.cfg, params)


@dataclass(frozen=True)
class ValueConfig:
    hidden_dim: int = 64
    n_steps: int = 41
    mlp_hidden: int = 32
    init_scale: float = 0.1


class ValueHead:
    def __init__(self, cfg: ValueConfig, params: ParamSet) -> None:
        self.cfg = cfg
        self.params = params

    @classmethod
    def init(cls, rng: np.random.Generator, cfg: ValueConfig) -> "ValueHead":
        d, m, s = cfg.hidden_dim, cfg.mlp_hidden, cfg.init_scale
        tensors = {
            "w_attn": rng.normal(0.0, s, size=d),
            "b_attn": np.zeros(1),
            "e_step": rng.normal(0.0, s, size=(cfg.n_steps, d)),
            "w0v": rng.normal(0.0, s / np.sqrt(d), size=(m, d)),
            "b0v": np.zeros(m),
            "w1v": rng.normal(0.0, s / np.sqrt(m), size=(1, m)),
            "b1v": np.zeros(1),
        }
        return cls(cfg, ParamSet(tensors))

    def with_params(self, params: ParamSet) -> "ValueHead":
        return ValueHead(self.cfg, params)


@dataclass(frozen=True)
class ObsModelConfig:
    obs_dim: int
    chunk_len: int = 4
    n_actions: int = 7
    hidden_dim: int = 96
    init_scale: float = 0.1

    @property
    def in_dim(self) -> int:
        return self.obs_dim + self.chunk_len * self.n_actions


class ObsModel:
    def __init__(self, cfg: ObsModelConfig, params: ParamSet) -> None:
        self.cfg = cfg
        self.params = params

    @classmethod
    def init(cls, rng: np.random.Generator, cfg: ObsModelConfig) -> "ObsModel":
        return cls(cfg, ParamSet(_init_mlp(rng, [cfg.in_dim, cfg.hidden_dim, cfg.obs_dim],
                                           cfg.init_scale)))

    def with_params(self, params: ParamSet) -> "ObsModel":
        return ObsModel(self.cfg, params)


class RewardModel:
    def __init__(self, obs_dim: int, params: ParamSet, hidden_dim: int = 64) -> None:
        self.obs_dim = obs_dim
        self.hidden_dim = hidden_dim
        self.params = params

    @classmethod
    def init(cls, rng: np.random.Generator, obs_dim: int, hidden_dim: int = 64,
             init_scale: float = 0.1) -> "RewardModel":
        return cls(obs_dim, ParamSet(_init_mlp(rng, [obs_dim, hidden_dim, 1], init_scale)),
                   hidden_dim)

    def with_params(self, params: ParamSet) -> "RewardModel":
        return RewardModel(self.obs_dim, params, self.hidden_dim)


@dataclass
class ModelBundle:
    policy: PolicyModel
    value: ValueHead
    obs_model: ObsModel | None = None
    reward_model: RewardModel | None = None

    def clone(self) -> "ModelBundle":
        def cp(m):
            return None if m is None else m.with_params(m.params.copy())
        return ModelBundle(cp(self.policy), cp(self.value), cp(self.obs_model),
                           cp(self.reward_model))


@dataclass(frozen=True)
class Trajectory:
    """One completed episode; observations/steps cover T+1 frames."""

    task_id: int
    source: str
    observations: np.ndarray
    steps: np.ndarray
    tokens: np.ndarray
    rewards: np.ndarray
    behavior_logits: np.ndarray
    values: np.ndarray
    bootstrap_value: float
    done: bool
    behavior_version: int
    step_versions: np.ndarray = field(default=None)

    def __post_init__(self) -> None:
        if self.source not in ("real", "imagined"):
            raise ValueError(f"source must be real|imagined, got {self.source!r}")
        tokens = np.asarray(self.tokens, dtype=np.int64)
        t_len = tokens.shape[0]
        if t_len < 1:
            raise ValueError("trajectory needs at least one decision")
        versions = (np.full(t_len, self.behavior_version, dtype=np.int64)
                    if self.step_versions is None else np.asarray(self.step_versions, np.int64))
        arrays = {
            "observations": np.asarray(self.observations, dtype=np.float64),
            "steps": np.asarray(self.steps, dtype=np.int64),
            "tokens": tokens,
            "rewards": np.asarray(self.rewards, dtype=np.float64),
            "behavior_logits": np.asarray(self.behavior_logits, dtype=np.float64),
            "values": np.asarray(self.values, dtype=np.float64),
            "step_versions": versions,
        }
        if arrays["observations"].shape[0] != t_len + 1 or arrays["steps"].shape != (t_len + 1,):
            raise ValueError("observations/steps must cover T+1 frames")
        for name in ("rewards", "values", "step_versions"):
            if arrays[name].shape != (t_len,):
                raise ValueError("per-decision arrays must have length T")
        if arrays["behavior_logits"].shape[:2] != (t_len, tokens.shape[1]):
            raise ValueError("behavior logits must be (T, K, n_actions)")
        for name, arr in arrays.items():
            arr.setflags(write=False)
            object.__setattr__(self, name, arr)

    @property
    def t_len(self) -> int:
        return int(self.tokens.shape[0])

    @property
    def episode_return(self) -> float:
        return float(np.sum(self.rewards))
