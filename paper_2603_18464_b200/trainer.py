"""B200 drop-in for the reference trainer hot path (`asyncrl.trainer`).

Same public surface as the reference module (`trainer.py:44-560`):
`GaeConfig`, `LossConfig`, `TrainerConfig`, `compute_gae`,
`shard_statistics`, `ShardStats`, `global_normalize`, `trust_weight`,
`chunk_ratio`, `policy_surrogate`, `entropy_bonus`, `total_loss`,
`behavior_log_probs` and `Trainer` with `build_train_batch`, `train_step`,
`recompute_values`, `run`, `publish_*` and the same attributes, record keys,
metric events and error types.  The math runs in libaccel.so (sm_100a): the
dense products on its tcgen05 3xTF32 GEMM kernels, the rest on its row /
segment kernels; torch provides device memory, streams and three tiny
(<= 257-row) products.  There is no CPU path.

`Trainer.build_train_batch` accepts the reference's `list[Trajectory]` (any
objects with those fields) or an already packed `workload.PackedBatch`, and
returns a `DeviceTrainBatch` (lazy host views of the reference TrainBatch
fields) or None.  `Trainer.train_step` accepts that batch or any
reference-shaped host TrainBatch.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Any, Generator

import numpy as np
import torch

from . import _lib, ops
from .batch import DeviceTrainBatch
from .errors import AccelError, DimensionError, DomainError, NonFiniteError
from .params import AdamStateView, DeviceParams, Dims, FlatLayout, POLICY_NAMES, VALUE_NAMES
from .publish import OBS_MODEL, POLICY, REWARD_MODEL, VersionedWeights
from .replay import DeviceTrajectory
from .world_model import DeviceMlp2, obs_model_data, reward_model_data
from .workload import PackedBatch, PinnedStaging, pack_trajectories

F32, F64, I32 = torch.float32, torch.float64, torch.int32


# ---------------------------------------------------------------------------
# configuration — trainer.py:44-72, :263-286


@dataclass(frozen=True)
class GaeConfig:
    gamma: float = 0.99
    lam: float = 0.95

    def __post_init__(self) -> None:
        if not 0.0 < self.gamma <= 1.0:
            raise DomainError(f"gamma must be in (0, 1], got {self.gamma}")
        if not 0.0 <= self.lam <= 1.0:
            raise DomainError(f"lam must be in [0, 1], got {self.lam}")


@dataclass(frozen=True)
class LossConfig:
    algorithm: str = "trust"
    sigma: float = 0.3
    clip_eps: float = 0.2
    lambda_v: float = 0.5
    lambda_h: float = 0.01
    # PPO value clipping (north star (b)); None = the reference's plain MSE
    # (trainer.py:438-443), which has no clipped variant
    value_clip: float | None = None

    def __post_init__(self) -> None:
        if self.value_clip is not None and not self.value_clip > 0:
            raise DomainError(f"value_clip must be > 0, got {self.value_clip}")
        if self.algorithm not in ("trust", "clip"):
            raise DomainError(f"unknown algorithm {self.algorithm!r}")
        if self.sigma <= 0:
            raise DomainError(f"sigma must be > 0, got {self.sigma}")
        if not 0.0 < self.clip_eps < 1.0:
            raise DomainError(f"clip_eps must be in (0, 1), got {self.clip_eps}")
        if self.lambda_v < 0 or self.lambda_h < 0:
            raise DomainError("loss coefficients must be >= 0")


@dataclass(frozen=True)
class TrainerConfig:
    gae: GaeConfig = GaeConfig()
    loss: LossConfig = LossConfig()
    lr: float = 3e-4
    beta1: float = 0.9
    beta2: float = 0.999
    k_shards: int = 4
    eps_norm: float = 1e-8
    revalue: bool = True
    world_model: bool = False
    t_obs: int = 4
    t_reward: int = 8
    wm_batch_episodes: int = 8
    wm_max_transitions: int = 512
    reward_neg_ratio: int = 4
    poll_interval: float = 0.002
    train_service_time: float = 0.0

    def __post_init__(self) -> None:
        if self.k_shards < 1:
            raise DomainError("k_shards must be >= 1")
        if self.t_obs < 1 or self.t_reward < 1:
            raise DomainError("world-model schedules must be >= 1")


def _algo_id(cfg: LossConfig) -> int:
    return 0 if cfg.algorithm == "trust" else 1


def _device():
    if not torch.cuda.is_available():
        raise AccelError("the B200 trainer needs a CUDA device (there is no CPU path)")
    return torch.device("cuda", torch.cuda.current_device())


def _dev(a, dtype, device):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).to(device, non_blocking=True)


# ---------------------------------------------------------------------------
# module-level functions (reference trainer.py:79-256, :289-293)


def compute_gae(rewards, values, done: bool, cfg: GaeConfig):
    """One trajectory through the segmented GAE kernel (trainer.py:79-101)."""
    r = np.asarray(rewards, dtype=np.float64)
    v = np.asarray(values, dtype=np.float64)
    t_len = r.shape[0]
    if v.shape != (t_len + 1,):
        raise DomainError(f"values must have length T+1={t_len + 1}, got {v.shape}")
    if t_len == 0:
        raise DomainError("empty trajectory")
    dev = _device()
    off = torch.tensor([0, t_len], dtype=torch.int64, device=dev)
    adv, ret, _ = ops.gae_segmented(_dev(r, np.float32, dev), _dev(v, np.float32, dev), off,
                                    torch.tensor([1 if done else 0], dtype=torch.uint8, device=dev),
                                    cfg.gamma, cfg.lam)
    return adv.double().cpu().numpy(), ret.double().cpu().numpy()


@dataclass(frozen=True)
class ShardStats:
    """Per-shard (sum, sum-of-squares, count) — trainer.py:108-125."""

    s: np.ndarray
    q: np.ndarray
    n: np.ndarray

    def __post_init__(self) -> None:
        s, q, n = (np.asarray(a, dtype=np.float64) for a in (self.s, self.q, self.n))
        if not (s.shape == q.shape == n.shape):
            raise DomainError("shard stat arrays must share one shape")
        if np.any(n * q - s * s < -1e-9):
            raise DomainError("inconsistent shard stats: N*Q < S^2")
        object.__setattr__(self, "s", s)
        object.__setattr__(self, "q", q)
        object.__setattr__(self, "n", n)


def _moments(shards) -> np.ndarray:
    dev = _device()
    arrs = [np.asarray(a, dtype=np.float64).ravel() for a in shards]
    sizes = np.array([a.size for a in arrs], dtype=np.int64)
    off = np.zeros(len(arrs) + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    flat = np.concatenate(arrs) if arrs else np.zeros(0)
    out = ops.segment_moments(_dev(flat if flat.size else np.zeros(1), np.float32, dev),
                              _dev(off, np.int64, dev))
    return out.cpu().numpy()


def shard_statistics(shards) -> ShardStats:
    """trainer.py:128-132 on the GPU (segmented float64 moments)."""
    mom = _moments(shards) if len(shards) else np.zeros((0, 3))
    return ShardStats(mom[:, 0], mom[:, 1], mom[:, 2])


def global_normalize(shards, eps: float = 1e-8):
    """Pooled normalization from shard sums — trainer.py:135-158."""
    stats = shard_statistics(list(shards))
    dev = _device()
    sums = torch.tensor([float(np.sum(stats.s)), float(np.sum(stats.q)), float(np.sum(stats.n))],
                        dtype=F64, device=dev)
    st = ops.normalize_finalize(sums, eps).cpu().numpy()
    if st[3] == 1:
        raise DomainError("cannot normalize zero advantages")
    if st[3] == 2:
        raise DomainError(f"negative pooled variance {st[1]}")
    out = []
    st_dev = torch.from_numpy(st).to(dev)
    for a in shards:
        a = np.asarray(a, dtype=np.float64)
        if a.size == 0:
            out.append(np.zeros(0))
            continue
        x = _dev(a, np.float32, dev)
        out.append(ops.normalize_apply(x, st_dev).double().cpu().numpy())
    return out, {"mean": float(st[0]), "std": float(st[1]), "n": int(np.sum(stats.n)),
                 "shard_sizes": tuple(int(k) for k in stats.n)}


def trust_weight(ratio, sigma: float):
    """exp(-log(r)^2 / (2 sigma^2)) — trainer.py:165-175 (float64, on device)."""
    r = np.asarray(ratio, dtype=np.float64)
    if np.any(r <= 0) or not np.all(np.isfinite(r)):
        raise DomainError("trust weight needs finite ratios > 0")
    t = torch.from_numpy(np.atleast_1d(r).copy()).to(_device())
    w = torch.exp(-0.5 * torch.square(torch.log(t) / sigma)).cpu().numpy()
    return float(w[0]) if np.isscalar(ratio) else w.reshape(r.shape)


def chunk_ratio(logp_new, logp_old):
    """Joint chunk ratio exp(sum_k (lp_new - lp_old)) — trainer.py:178-180."""
    a = torch.from_numpy(np.asarray(logp_new, dtype=np.float64).copy()).to(_device())
    b = torch.from_numpy(np.asarray(logp_old, dtype=np.float64).copy()).to(_device())
    return torch.exp((a - b).sum(dim=-1)).cpu().numpy()


def policy_surrogate(logp_new, logp_old, advantages, cfg: LossConfig, trust_weights=None):
    """Token surrogate and its lp gradient — trainer.py:183-239 (float64 on device).

    The trainer itself never calls this: it runs the fused logits-level
    kernel (accel_token_loss).  This function keeps the reference's
    log-prob-level API, including the pinned `trust_weights` override."""
    dev = _device()
    lpn = torch.from_numpy(np.asarray(logp_new, dtype=np.float64).copy()).to(dev)
    lpo = torch.from_numpy(np.asarray(logp_old, dtype=np.float64).copy()).to(dev)
    adv = torch.from_numpy(np.asarray(advantages, dtype=np.float64).copy()).to(dev)
    a_tok = adv[:, None].expand_as(lpn)
    ratios = torch.exp(lpn - lpo)
    inc = torch.isfinite(ratios) & (ratios > 0)
    n_inc = int(inc.sum().item())
    diag: dict[str, Any] = {"excluded_tokens": int(inc.numel() - n_inc), "dropped": False}
    if n_inc == 0:
        diag["dropped"] = True
        return 0.0, np.zeros(lpn.shape), diag
    m = float(n_inc)
    r = torch.where(inc, ratios, torch.ones_like(ratios))
    a = torch.where(inc, a_tok, torch.zeros_like(a_tok))
    if cfg.algorithm == "trust":
        if trust_weights is None:
            w = torch.exp(-0.5 * torch.square(torch.log(r) / cfg.sigma))
        else:
            w = torch.from_numpy(np.broadcast_to(np.asarray(trust_weights, dtype=np.float64),
                                                 tuple(lpn.shape)).copy()).to(dev)
        w = torch.where(inc, w, torch.zeros_like(w))
        loss = -float((w * r * a)[inc].sum().item()) / m
        dlogp = torch.where(inc, -(w * r * a) / m, torch.zeros_like(r))
        diag["trust_weight_mean"] = float(w[inc].mean().item())
        diag["trust_weight_min"] = float(w[inc].min().item())
    else:
        lo, hi = 1.0 - cfg.clip_eps, 1.0 + cfg.clip_eps
        rc = torch.clamp(r, lo, hi)
        loss = -float(torch.minimum(r * a, rc * a)[inc].sum().item()) / m
        dlogp = torch.where((r * a <= rc * a) & inc, -(r * a) / m, torch.zeros_like(r))
        diag["clipped_fraction"] = float(((r < lo) | (r > hi))[inc].double().mean().item())
    diag["ratio_mean"] = float(r[inc].mean().item())
    diag["ratio_max"] = float(r[inc].max().item())
    return loss, dlogp.cpu().numpy(), diag


def entropy_bonus(logits):
    """Mean token entropy and its logits gradient — trainer.py:242-251 (float64, device)."""
    z = torch.from_numpy(np.asarray(logits, dtype=np.float64).copy()).to(_device())
    if z.numel() == 0 or not bool(torch.isfinite(z).all().item()):
        raise DomainError("log_softmax input contains non-finite values")
    lp = torch.log_softmax(z, dim=-1)
    p = torch.exp(lp)
    h_tok = -(p * lp).sum(dim=-1)
    n = float(h_tok.numel())
    return float(h_tok.sum().item()) / n, (-p * (lp + h_tok[..., None]) / n).cpu().numpy()


def total_loss(policy_term: float, value_term: float, entropy: float, cfg: LossConfig) -> float:
    """L = L_policy + lambda_v L_value - lambda_h H — trainer.py:254-256."""
    return policy_term + cfg.lambda_v * value_term - cfg.lambda_h * entropy


def behavior_log_probs(behavior_logits, tokens):
    """(T, K) chosen-token log-probs through accel_token_logp (trainer.py:289-293)."""
    mu = np.asarray(behavior_logits, dtype=np.float64)
    t = np.asarray(tokens, dtype=np.int64)
    if mu.shape[:-1] != t.shape:
        raise DimensionError(f"tokens {t.shape} do not index logits {mu.shape}")
    dev = _device()
    A = mu.shape[-1]
    lp, bad = ops.token_logp(_dev(mu.reshape(-1, A), np.float32, dev),
                             _dev(t.reshape(-1), np.int32, dev))
    bad = bad.sum(dim=0).cpu().numpy()
    if bad[0] > 0:
        raise DomainError("log_softmax input contains non-finite values")
    if bad[1] > 0:
        raise DimensionError("token index outside the action vocabulary")
    return lp.double().cpu().numpy().reshape(t.shape)


# ---------------------------------------------------------------------------
# scratch buffers


class _Scratch:
    """Grow-only named device buffers (shapes change with every batch).

    Guard mode (tests): every buffer handed out is followed by >= 4 KB of a
    byte pattern, re-armed at each get(); check_guards() lists the buffers
    whose tail a kernel wrote past its shape."""

    GUARD_BYTE = 0xA5
    GUARD_BYTES = 4096

    def __init__(self, device) -> None:
        self.device = device
        self._bufs: dict = {}
        self.guard = False
        self._armed: dict = {}

    def get(self, name: str, shape, dtype=F32) -> torch.Tensor:
        n = int(np.prod(shape)) if len(shape) else 1
        buf = self._bufs.get(name)
        pad = -(-self.GUARD_BYTES // torch.empty((), dtype=dtype).element_size()) if self.guard else 0
        if buf is None or buf.dtype != dtype or buf.numel() < n + pad:
            ops.retire(buf)
            buf = torch.empty(max(n, 1) + (n >> 4) + pad, dtype=dtype, device=self.device)
            self._bufs[name] = buf
        if self.guard:
            buf.view(torch.uint8)[n * buf.element_size():].fill_(self.GUARD_BYTE)
            self._armed[name] = n
        return buf[:n].view(*shape) if len(shape) else buf[:1]

    def check_guards(self) -> list:
        bad = []
        for name, n in self._armed.items():
            buf = self._bufs[name]
            tail = buf.view(torch.uint8)[n * buf.element_size():]
            if not bool((tail == self.GUARD_BYTE).all()):
                bad.append(name)
        return bad


def _array_split_sizes(n: int, k: int) -> tuple:
    base, extra = divmod(n, k)
    return tuple(base + 1 if i < extra else base for i in range(k))


# ---------------------------------------------------------------------------
# the trainer


class Trainer:
    """Owns the live models on the device; consumes TrainBatches; publishes.

    Reference: trainer.py:296-560.  `comm` (optional) is a data-parallel
    communicator (`dp.DataParallel`); without it the trainer is one GPU.
    """

    def __init__(self, bundle, cfg: TrainerConfig, service: Any = None, metrics: Any = None,
                 seed: int = 0, comm: Any = None) -> None:
        if cfg.world_model and (getattr(bundle, "obs_model", None) is None
                                or getattr(bundle, "reward_model", None) is None):
            raise DomainError("world_model=True needs a bundle with obs_model and reward_model")
        self.cfg = cfg
        self.service = service
        self.metrics = metrics
        self.comm = comm
        self._dec_idx = None  # data parallel: the build's summed flag entries (device)
        self.device = _device()
        self.rng = np.random.default_rng(np.random.SeedSequence([seed, 7]))
        self._bundle = bundle
        self.dims = Dims.from_models(bundle.policy, bundle.value)
        self.layout = FlatLayout(self.dims, pad_to=4 * (comm.world if comm is not None else 1))
        self.params = DeviceParams(self.layout, self.device,
                                   shard=(comm.rank, comm.world) if comm is not None else None)
        self.params.load(bundle.policy.params.tensors, bundle.value.params.tensors)
        self._policy_version = int(getattr(bundle.policy.params, "version", 0))
        self._value_version = int(getattr(bundle.value.params, "version", 0))
        self._host_stale = False
        self._param_gen = 0  # bumps whenever the device parameters change
        self._last_h = None
        self.adam_policy = AdamStateView(self, 0, cfg.lr, cfg.beta1, cfg.beta2)
        self.adam_value = AdamStateView(self, 1, cfg.lr, cfg.beta1, cfg.beta2)
        self.publish_version = 0
        self.cycles = 0
        self.skipped = 0
        self.obs_updates = 0
        self.reward_updates = 0
        # world-model sub-steps (trainer.py:469-535): float64 device MLPs, created
        # on first use (the bundle's obs/reward models seed them)
        self._wm = {}
        self.scratch = _Scratch(self.device)
        self._staging = PinnedStaging()
        self._rec_host = torch.zeros(64, dtype=F64).pin_memory()
        # Adam hyperparameters of the next step, refreshed on the host and copied
        # to the device inside the step (so a captured CUDA graph replays steps)
        self._hyper_host = torch.zeros(12, dtype=F64).pin_memory()
        self._hyper_dev = torch.zeros(12, dtype=F64, device=self.device)
        self.profile_events = None  # list -> CUDA-event brackets of the hot kernels
        A, K = self.dims.n_actions, self.dims.chunk_len
        # factorized head (no [M, A] logits) wherever the kernel supports the shape
        self.factorized = A % 4 == 0 and 128 <= A <= 1024 and K <= 32
        # recompute_dz: the loss kernel writes 16 B of token scalars instead of the
        # 4A-byte dz row and the (prev, k) grouped sums recompute dz from the
        # L2-resident H2W rows of one block of frames at a time (frame-blocked
        # sort, group_block_chunks 4096-token chunks per block); on by default
        # where the two-phase loss kernel serves the shape (K <= 8, A in {128, 256})
        self.recompute_dz = self.factorized and K <= 8 and A in (128, 256)
        self.group_block_chunks = 64
        torch.backends.cuda.matmul.allow_tf32 = False
        torch.backends.cudnn.allow_tf32 = False

    def gather_moments(self) -> None:
        """Collective under data parallelism: assemble the sharded Adam moments
        (ZeRO-2 keeps only this rank's slices) so `adam_policy.m` / `.v` show
        the full state at the current generation (a no-op on one GPU)."""
        if self.comm is not None:
            self.comm.gather_moments(self.params)

    def _pk_cpb(self) -> int:
        # the frame-blocked recompute rides on the two-phase loss kernel's sorted
        # scalar output (K <= 8, A in {128, 256})
        A, K = self.dims.n_actions, self.dims.chunk_len
        ok = self.recompute_dz and K <= 8 and A in (128, 256)
        return self.group_block_chunks if ok else 0

    # -- bundle <-> device ---------------------------------------------------------
    @property
    def bundle(self):
        for kind, mlp in self._wm.items():  # world-model parameters updated on the device
            model = getattr(self._bundle, kind)
            if model.params is not mlp.params():
                setattr(self._bundle, kind, model.with_params(mlp.params()))
        if self._host_stale:
            pol, val = self.params.to_host()
            b = self._bundle
            b.policy.params = type(b.policy.params)(pol, self._policy_version)
            b.value.params = type(b.value.params)(val, self._value_version)
            self._host_stale = False
        return self._bundle

    @bundle.setter
    def bundle(self, new) -> None:
        dims = Dims.from_models(new.policy, new.value)
        if dims != self.dims:
            raise DimensionError(f"bundle dims {dims} != trainer dims {self.dims}")
        self._bundle = new
        self.params.load(new.policy.params.tensors, new.value.params.tensors)
        self._policy_version = int(getattr(new.policy.params, "version", 0))
        self._value_version = int(getattr(new.value.params, "version", 0))
        self._host_stale = False
        self._param_gen += 1

    # -- publication (trainer.py:328-348) -------------------------------------------
    def snapshot(self) -> VersionedWeights:
        return VersionedWeights.from_device(POLICY, self.publish_version, self)

    def publish_policy(self) -> None:
        if self.service is None:
            return
        self.service.update_weights(self.snapshot())

    def publish_world_model(self, kind: str) -> None:
        """trainer.py:336-342: a snapshot of one world model at its own version."""
        if self.service is None or kind not in getattr(self.service, "configs", {}):
            return
        model = getattr(self.bundle, kind)
        snap = model.with_params(model.params.copy())
        self.service.update_weights(VersionedWeights(kind, int(snap.params.version),
                                                     **{kind: snap}))

    def publish_initial(self) -> None:
        self.publish_policy()
        if self.cfg.world_model:
            self.publish_world_model(OBS_MODEL)
            self.publish_world_model(REWARD_MODEL)

    # -- world-model sub-steps (trainer.py:469-535) ------------------------------------
    def _wm_mlp(self, kind: str) -> DeviceMlp2:
        if kind not in self._wm:
            model = getattr(self._bundle, kind, None)
            if model is None:
                raise DomainError(f"the bundle has no {kind}")
            cfg = self.cfg
            self._wm[kind] = DeviceMlp2(model.params, cfg.lr, cfg.beta1, cfg.beta2, 1e-8,
                                        self.device)
        return self._wm[kind]

    @property
    def adam_obs(self):
        return self._wm_mlp(OBS_MODEL).adam_state()

    @property
    def adam_reward(self):
        return self._wm_mlp(REWARD_MODEL).adam_state()

    def train_obs_model_step(self, trajs) -> float:
        """MSE regression on (o_t, a_t) -> o_{t+1} transitions (trainer.py:469-494)."""
        mlp = self._wm_mlp(OBS_MODEL)
        x, y = obs_model_data(self._bundle.obs_model, trajs, self.cfg.wm_max_transitions,
                              self.rng)
        loss = mlp.update(x, y, 0)
        self.obs_updates += 1
        self.publish_world_model(OBS_MODEL)
        if self.metrics is not None:
            self.metrics.emit("obs_model_step", loss=loss, updates=self.obs_updates)
        return loss

    def train_reward_model_step(self, trajs) -> float:
        """Binary cross-entropy on frames; positives are terminal frames of
        successful episodes, negatives subsampled (trainer.py:496-535)."""
        mlp = self._wm_mlp(REWARD_MODEL)
        x, labels, single_class = reward_model_data(trajs, self.cfg.reward_neg_ratio,
                                                    self.cfg.wm_max_transitions, self.rng)
        loss = mlp.update(x, labels, 1)
        self.reward_updates += 1
        self.publish_world_model(REWARD_MODEL)
        if self.metrics is not None:
            self.metrics.emit("reward_model_step", loss=loss, updates=self.reward_updates,
                              single_class=single_class)
        return loss

    # -- shared forward pieces -------------------------------------------------------
    def _backbone(self, frames, tag: str | None, nonfinite=None):
        """h1, h2 over frame rows (models.py:176-177); tag None -> fresh tensors."""
        P = self.params.pv
        F = frames.shape[0]
        D = self.dims.hidden

        def buf(name):
            if tag is None:
                return torch.empty(F, D, dtype=F32, device=self.device)
            return self.scratch.get(tag + name, (F, D))

        if nonfinite is not None:  # the frame finiteness check rides on this read
            h1 = ops.tc_linear_checked(frames, P["w0"], buf("h1"), nonfinite, bias=P["b0"],
                                       tanh=True)
        else:
            h1 = ops.tc_linear(frames, P["w0"], buf("h1"), bias=P["b0"], tanh=True)
        h2 = ops.tc_linear(h1, P["w1"], buf("h2"), bias=P["b1"], tanh=True)
        return h1, h2

    def _frame_values(self, frames, steps, out, bad_part, keep: bool = False, nonfinite=None):
        """V(o) on every frame: state_values_batch (models.py:411-415).

        keep=True returns the backbone activations (fresh tensors) so a
        train_step under the same parameters can reuse them."""
        P = self.params.pv
        F = frames.shape[0]
        d = self.dims
        h1, h2 = self._backbone(frames, None if keep else "rv.", nonfinite)
        fresh = lambda shape: torch.empty(*shape, dtype=F32, device=self.device)
        U = fresh((F, d.hidden)) if keep else self.scratch.get("rv.U", (F, d.hidden))
        alpha = fresh((F, 2)) if keep else self.scratch.get("rv.alpha", (F, 2))
        g = ops.warp_grid(F)
        ops.value_pool(h1, h2, None, steps, F, d.n_steps, P["w_attn"], P["b_attn"], P["e_step"], U,
                       alpha, bad_part, g)
        zm = ops.tc_linear(U, P["w0v"], fresh((F, d.mlp_hidden)) if keep
                           else self.scratch.get("rv.zm", (F, d.mlp_hidden)))
        ops.value_head(zm, P["b0v"], P["w1v"], P["b1v"], None, 0.0, 0.0, out, None, None,
                       ops.warp_grid(F))
        # keep: the train step under the same parameters reuses the backbone and
        # the value head's pooling / first layer (frame space)
        self._last_h = (h1, h2, U, alpha, zm) if keep else None
        return g

    def recompute_values(self, traj) -> np.ndarray:
        """V(o_t) for all T+1 frames under the current critic (trainer.py:352-356)."""
        assert self.publish_version >= traj.behavior_version
        frames = ops.upload_pitched(np.asarray(traj.observations, dtype=np.float32), self.device)
        steps = _dev(np.asarray(traj.steps), np.int32, self.device)
        if frames.shape[1] != self.dims.obs_dim:
            raise DimensionError(f"observations have dim {frames.shape[1]}, "
                                 f"expected {self.dims.obs_dim}")
        F = frames.shape[0]
        out = torch.empty(F, dtype=F32, device=self.device)
        bad_part = self.scratch.get("rv.bad", (ops.warp_grid(F), 2), F64)
        g = self._frame_values(frames, steps, out, bad_part)
        bad = bad_part[:g].sum(dim=0).cpu().numpy()
        if bad[0] > 0:
            raise DomainError("softmax input contains non-finite values")
        if bad[1] > 0:
            raise DimensionError(f"step index outside value-step table [0, {self.dims.n_steps})")
        return out.double().cpu().numpy()

    # -- batch construction (trainer.py:358-403) --------------------------------------
    def upload(self, pb: PackedBatch, pre: dict | None = None) -> dict:
        """Device copies of a packed batch; `pre` holds fields already uploaded
        while the pack ran ("mu", and "frames_c": contiguous frame rows)."""
        d = self.dims
        if pb.obs_dim != d.obs_dim or pb.chunk_len != d.chunk_len or pb.n_actions != d.n_actions:
            raise DimensionError(
                f"batch (obs {pb.obs_dim}, K {pb.chunk_len}, A {pb.n_actions}) does not match "
                f"the policy (obs {d.obs_dim}, K {d.chunk_len}, A {d.n_actions})")
        dev = self.device
        pre = pre or {}
        if "frames_c" in pre:  # re-pitch the contiguous rows on the device
            fc = pre["frames_c"]
            frames = ops.alloc_pitched(fc.shape[0], fc.shape[1], dev)
            frames = frames.copy_(fc) if not frames.is_contiguous() else fc
        else:
            frames = ops.upload_pitched(np.asarray(pb.frames, dtype=np.float32), dev)
        return {
            "traj_off": _dev(pb.traj_off, np.int64, dev),
            "frames": frames,
            "steps": _dev(pb.steps, np.int32, dev),
            "values": _dev(pb.values, np.float32, dev),
            "tokens": _dev(pb.tokens.reshape(-1), np.int32, dev),
            "rewards": _dev(pb.rewards, np.float32, dev),
            "mu": pre["mu"] if "mu" in pre else _dev(pb.mu.reshape(-1, pb.n_actions), np.float32,
                                                       dev),
            "done": _dev(pb.done, np.uint8, dev),
        }

    def build_train_batch(self, trajs) -> DeviceTrainBatch | None:
        """Recompute, estimate advantages, normalize globally, tensorize."""
        pre = None
        if isinstance(trajs, PackedBatch):
            pb = trajs
        elif trajs and isinstance(trajs[0], DeviceTrajectory):
            # sampled from a DeviceReplayBuffer: the batch is gathered in HBM
            buf = trajs[0].buffer
            if any(not isinstance(t, DeviceTrajectory) or t.buffer is not buf for t in trajs):
                raise DimensionError("a batch mixes trajectories of different replay buffers")
            if self.cfg.revalue:
                for t in trajs:
                    assert self.publish_version >= t.behavior_version
            got = buf.gather(trajs)
            if got is None:  # a sampled trajectory was evicted meanwhile: dropped batch
                return None
            b, n_real, bver = got
            return self.build_from_device(b, n_real=n_real, behavior_version=bver)
        else:
            for t in trajs:
                if self.cfg.revalue:
                    assert self.publish_version >= t.behavior_version
            # one threaded pass casting into page-locked staging, in four chunks:
            # each chunk's behavior logits and frame rows (the bulk of the bytes)
            # go to the device as asynchronous DMA while the next chunk is packed
            # (the build's one host sync orders the staging's reuse)
            pre = {}

            def on_chunk(lo, hi, off, frames, mu):
                if not pre:
                    pre["mu"] = torch.empty(mu.shape[0] * mu.shape[1], mu.shape[2],
                                            dtype=F32, device=self.device)
                    pre["frames_c"] = torch.empty(frames.shape, dtype=F32, device=self.device)
                a, b = int(off[lo]), int(off[hi])
                K = mu.shape[1]
                pre["mu"][a * K:b * K].copy_(torch.from_numpy(mu[a:b].reshape(-1, mu.shape[2])),
                                             non_blocking=True)
                pre["frames_c"][a + lo:b + hi].copy_(torch.from_numpy(frames[a + lo:b + hi]),
                                                     non_blocking=True)

            pb = pack_trajectories(trajs, staging=self._staging, chunks=4, on_chunk=on_chunk)
        dev_batch = self.upload(pb, pre)
        return self.build_from_device(dev_batch, n_real=int(pb.real.sum()),
                                      behavior_version=pb.behavior_version)

    def build_from_device(self, b: dict, n_real: int, behavior_version) -> DeviceTrainBatch | None:
        """The device half of build_train_batch on an uploaded CSR batch."""
        batch, host_dev = self._build_device(b, n_real, behavior_version)
        return self._build_finish(batch, host_dev.cpu().numpy())  # the one host sync

    def _build_device(self, b: dict, n_real: int, behavior_version) -> tuple:
        """Every launch of the build, no host sync: (batch, device flag vector)."""
        cfg, d = self.cfg, self.dims
        n = int(b["traj_off"].shape[0] - 1)
        N = int(b["rewards"].shape[0])
        F = N + n
        M = N * d.chunk_len
        dev = self.device
        flags = torch.zeros(16, dtype=F64, device=dev)
        cnt = torch.zeros(4, dtype=torch.int32, device=dev)
        if cfg.revalue:
            values = torch.empty(F, dtype=F32, device=dev)
            bad_part = self.scratch.get("b.vbad", (ops.warp_grid(F), 2), F64)
            # counts non-finite frame values into cnt[0] (every frame: a bad
            # bootstrap frame makes its revalued V non-finite, rejecting the batch too)
            g = self._frame_values(b["frames"], b["steps"], values, bad_part, keep=True,
                                   nonfinite=cnt[0:1])
            h_cache = (self._param_gen, *self._last_h)
            ops.reduce_f64(bad_part, g, 2, 0, flags[10:12])
        else:
            values = b["values"]
            h_cache = None
        frame_of = torch.empty(N, dtype=I32, device=dev)
        with self._timed("gae"):
            adv_raw, ret, _ = ops.gae_segmented(b["rewards"], values, b["traj_off"], b["done"],
                                                cfg.gae.gamma, cfg.gae.lam, frame_of=frame_of,
                                                sums=flags[0:4])
        if self.comm is None:
            ops.normalize_finalize(flags[0:3], cfg.eps_norm, flags[4:8])
            adv = ops.normalize_apply(adv_raw, flags[4:8])
        # (data parallel: the pooled (sum, sum of squares, count) ride on the one
        # decision all-reduce at the end of the build; normalization follows it)
        with self._timed("token_logp"):
            lp_old, lbad = ops.token_logp(b["mu"], b["tokens"])
        ops.reduce_f64(lbad, ops.token_grid(M), 2, 0, flags[8:10])
        if not cfg.revalue:
            ops.count_nonfinite_rows(b["frames"], frame_of, N, cnt[0:1])
        batch = DeviceTrainBatch(
            frames=b["frames"], steps=b["steps"], tokens=b["tokens"], frame_of=frame_of,
            lp_old=lp_old, adv=adv if self.comm is None else None, ret=ret,
            n_actions=d.n_actions, chunk_len=d.chunk_len,
            critic_version=self.publish_version, n_real=n_real, n_imagined=n - n_real,
            norm_mean=0.0, norm_std=0.0, norm_count=N,
            shard_sizes=_array_split_sizes(N, cfg.k_shards),
            behavior_lag_mean=float(np.mean(self.publish_version - np.asarray(behavior_version))))
        batch.ensure_groupings(d.n_steps, cnt[1:2], factorized=self.factorized,
                               frame_space=h_cache is not None, pk_cpb=self._pk_cpb())
        batch.h_cache = h_cache
        # frame row of each trajectory's bootstrap observation (t = T)
        batch.boot_rows = b["traj_off"][1:] + torch.arange(n, dtype=torch.int64, device=dev)
        if cfg.loss.value_clip is not None:  # rollout-time V per transition
            batch.v_old = b["values"].index_select(0, frame_of)
        host_dev = torch.cat([flags, cnt.double()])
        if self.comm is not None:
            lags = self.publish_version - np.asarray(behavior_version, dtype=np.int64)
            # (page-locked source, asynchronous: a pageable torch.tensor(..., device=)
            # here would block the host until the stream drained)
            counts = torch.tensor([float(n_real), float(n), float(lags.sum())],
                                  dtype=F64).pin_memory().to(dev, non_blocking=True)
            host_dev = torch.cat([host_dev, counts])
            # data parallel: the batch is one shard of the global batch; the pooled
            # advantage statistics, every accept/reject decision, the transition
            # count and the record's trajectory counts / behavior lag are global
            # (all ranks agree) -- one all-reduce of the entries that sum
            idx = self._dec_idx
            if idx is None or idx.device != host_dev.device:
                idx = self._dec_idx = torch.tensor([0, 1, 2, 3, 8, 9, 10, 11, 16, 17, 20, 21, 22],
                                                   device=dev)
            dec = host_dev.index_select(0, idx)
            self.comm.all_reduce_sum(dec)
            host_dev.index_copy_(0, idx, dec)
            ops.normalize_finalize(host_dev[0:3], cfg.eps_norm, host_dev[4:8])
            batch.adv = ops.normalize_apply(adv_raw, host_dev[4:8])
        return batch, host_dev

    def _build_finish(self, batch, host) -> DeviceTrainBatch | None:
        """The host half: the reference's domain errors and the finite check
        (trainer.py:392-402) from the build's flag vector."""
        cfg, d = self.cfg, self.dims
        if host[7] == 1:
            raise DomainError("cannot normalize zero advantages")
        if host[7] == 2:
            raise DomainError(f"negative pooled variance {host[5] ** 2}")
        if host[10] > 0:
            raise DomainError("softmax input contains non-finite values")
        if host[11] > 0 or host[17] > 0:
            raise DimensionError(f"step index outside value-step table [0, {d.n_steps})")
        if host[8] > 0:
            raise DomainError("log_softmax input contains non-finite values")
        if host[9] > 0:
            raise DimensionError("token index outside the action vocabulary")
        batch.norm_mean, batch.norm_std = float(host[4]), float(host[5])
        batch.norm_count = int(host[2])
        batch.global_n = int(host[2])
        if self.comm is not None:  # the global batch's record fields (trainer.py:385-403)
            batch.n_real, batch.n_imagined = int(host[20]), int(host[21] - host[20])
            batch.behavior_lag_mean = float(host[22] / host[21])
            batch.shard_sizes = _array_split_sizes(int(host[2]), cfg.k_shards)
        finite = host[3] == 0 and host[16] == 0
        batch._finite = bool(finite)
        return batch if finite else None

    # -- optimization (trainer.py:407-467) ---------------------------------------------
    def _timed(self, name: str):
        """CUDA-event bracket around one launch when `profile_events` is a list."""
        trainer = self

        class _Ctx:
            def __enter__(self_):
                if trainer.profile_events is not None:
                    self_.e0 = torch.cuda.Event(enable_timing=True)
                    self_.e0.record()

            def __exit__(self_, *exc):
                if trainer.profile_events is not None:
                    e1 = torch.cuda.Event(enable_timing=True)
                    e1.record()
                    trainer.profile_events.append((name, self_.e0, e1))
                return False

        return _Ctx()

    def _wgrad(self, dy, x, out, tag: str, extra: int = 0):
        """Tensor-core dW = dy^T x into per-CTA partial slices (+ `extra` slices
        the caller fills); returns the reduce_segments entry that sums them."""
        F, n = dy.shape
        k = x.shape[1]
        if n > 256 or k > 256:  # wide layers (cfg4): streamed tcgen05 GEMM, split-K slices
            ks = ops.wide_kslices(n, k, F)
            part = self.scratch.get("wg." + tag, (ks + extra, n, k))
            ops.wide_gemm(dy, x, part, a_mn=True, b_mn=True, epi=3, kslices=ks, tag="wgrad")
            return (part, out, ks + extra, n * k, n * k)
        dy, x = ops.pitched(dy), ops.pitched(x)  # no-ops at aligned widths
        ks = max(1, min(ops.tc_sm_count(), -(-F // 32)))
        part = self.scratch.get("wg." + tag, (2 * ks + extra, n, k))
        _lib.call("accel_tc_gemm", ops._pp(dy), ops._pp(x), ops._p(part), None, n, F, k,
                  dy.stride(0), x.stride(0), k, 1, 1, 0, 0, ks, ops._stream())
        return (part, out, 2 * ks + extra, n * k, n * k)

    def _side_stream(self):
        """The stream the value-head branch of a step runs on (per device)."""
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(device=self.device)
        return self._side

    def _write_hyper(self) -> None:
        """Both Adam groups' {lr, beta1, beta2, eps, 1 - beta^t} for the next step."""
        t_pol, t_val = self.adam_policy.step + 1, self.adam_value.step + 1
        self._hyper_host.numpy()[:] = (self.adam_policy.hyper(t_pol)
                                       + self.adam_value.hyper(t_val))

    def _bucket_done(self, tensor_name: str) -> None:
        if self.comm is not None:
            self.comm.bucket_ready(self.layout.bucket_of(tensor_name))

    def train_step(self, batch) -> dict | None:
        """One policy + value update from a TrainBatch; publishes.

        Returns the reference record dict, or None when every token was
        excluded (the batch is skipped, trainer.py:420-424)."""
        if not isinstance(batch, DeviceTrainBatch):
            batch = DeviceTrainBatch.from_host(batch, self.device)
        if batch.n_actions < 0:
            batch.n_actions = self.dims.n_actions
        record = self._step_device(batch)
        return self._finish_step(batch, record)

    def _step_device(self, batch: DeviceTrainBatch) -> torch.Tensor:
        """Launch the whole step on the current stream; returns the device record."""
        cfg, d = self.cfg, self.dims
        lc = cfg.loss
        P, G = self.params.pv, self.params.gv
        S = self.scratch
        dev = self.device
        N, F, K, A, D, H = (batch.n_transitions, batch.n_frames, d.chunk_len, d.n_actions,
                            d.hidden, d.mlp_hidden)
        M = N * K
        if batch.frames.shape[1] != d.obs_dim:
            raise DimensionError(f"obs dim {batch.frames.shape[1]} != {d.obs_dim}")
        cnt = S.get("st.cnt", (4,), torch.int32)
        cnt.zero_()
        fact = self.factorized
        hc = getattr(batch, "h_cache", None)
        vcache = None
        if hc is not None and hc[0] == self._param_gen:
            h1, h2 = hc[1], hc[2]  # revaluation ran under these exact parameters
            vcache = hc[3:]        # (U, alpha, zm) over all frames
            batch.h_cache = None   # consumed: the value backward overwrites zm in place
        batch.ensure_groupings(d.n_steps, cnt[1:2], factorized=fact,
                               frame_space=vcache is not None, pk_cpb=self._pk_cpb())
        if self.comm is None:
            N_glob, M_glob = N, M
        elif getattr(batch, "global_n", None) is not None:
            N_glob, M_glob = batch.global_n, batch.global_n * K
        else:
            N_glob, M_glob = self.comm.global_counts(N, K)
        algo = _algo_id(lc)
        lp_new = S.get("st.lp_new", (M,))
        loss_sums = S.get("st.lsum", (8,), F64)
        loss_max = S.get("st.lmax", (2,), F64)

        if vcache is None:
            h1, h2 = self._backbone(batch.frames, "st.")

        # ZeRO-2: each gradient bucket is reduce-scattered, updated (Adam on this
        # rank's slice, speculative: the host adopts generation nxt only if the
        # record accepts the step) and all-gathered as soon as the backward has
        # written it, on a side stream (dp.DataParallel)
        self._write_hyper()
        self._hyper_dev.copy_(self._hyper_host, non_blocking=True)
        adam_bad = cnt[2:3]
        if self.comm is not None:
            self.comm.begin_step(self.params, self._hyper_dev,
                                 S.get("st.noskip", (1,), torch.int32).zero_(), adam_bad,
                                 adam_fn=ops.adam_dev)

        # the value-head forward / backward depends only on the (detached) hiddens
        # and the targets: it runs on a side stream beside the policy's loss and
        # backward (joined before the record)
        side = self._side_stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            # value head (hiddens detached)
            vclip = {}
            if lc.value_clip is not None:
                v_old = getattr(batch, "v_old", None)
                if v_old is None:
                    raise DomainError("value_clip needs the rollout-time values of the batch")
                vclip = {"v_old": v_old, "vclip": lc.value_clip}
            gw = ops.warp_grid(N)
            vpart = S.get("st.vpart", (gw, 2 * H + 1))
            vdpart = S.get("st.vdpart", (gw, 2), F64)
            if vcache is not None:
                # frame space: the revaluation pass already pooled (U, alpha) and ran the
                # first layer (zm) on every frame; the loss covers the transition
                # frames, bootstrap rows carry zero gradient
                U, alpha, zm = vcache
                ops.value_head(zm, P["b0v"], P["w1v"], P["b1v"], batch.ret, lc.lambda_v, N_glob, None,
                               vpart, vdpart, gw, row_frame=batch.frame_of, rows=N, **vclip)
                if F != N:
                    zm.index_fill_(0, batch.boot_rows, 0.0)
                R, row_frame, step_group = F, None, batch.frame_step_group
                ga = ops.warp_grid(F)
                vbad_part = S.get("st.vbad", (1, 2), F64)
                vbad_part.zero_()  # attention / step checks ran in the revaluation pass
                nbad = 1
            else:
                U = S.get("st.U", (N, D))
                alpha = S.get("st.alpha", (N, 2))
                vbad_part = S.get("st.vbad", (gw, 2), F64)
                nbad = gw
                ops.value_pool(h1, h2, batch.frame_of, batch.frame_steps, N, d.n_steps, P["w_attn"],
                               P["b_attn"], P["e_step"], U, alpha, vbad_part, gw)
                zm = ops.tc_linear(U, P["w0v"], S.get("st.zm", (N, H)))
                ops.value_head(zm, P["b0v"], P["w1v"], P["b1v"], batch.ret, lc.lambda_v, N_glob, None,
                               vpart, vdpart, gw, **vclip)
                R, row_frame, step_group = N, batch.frame_of, batch.step_group
                ga = gw
            w0v_seg = self._wgrad(zm, U, G["w0v"], "w0v")  # dzm^T U
            dU = ops.tc_matmul_nn(zm, P["w0v"], S.get("st.dU", (R, D)))
            battn_part = S.get("st.battn", (ga,))
            wattn_part = S.get("st.wattn", (ga, D))
            gr = ga
            # dalpha, de and the dw_attn / db_attn partials in one pass over (dU, h1, h2)
            # (the de rows are only needed by the two-pass fallback at other widths)
            ops.value_attn_backward(dU, h1, h2, row_frame, alpha, battn_part, wattn_part, ga,
                                    de=S.get("st.de", (R, 2)))
            step_group.rows_sum(dU, G["e_step"])
            # the value bucket is complete: its ZeRO-2 exchange starts now (dp)
            ops.reduce_segments([
                w0v_seg,
                (vpart, G["w1v"], gw, H, 2 * H + 1),
                (vpart[:, H:], G["b0v"], gw, H, 2 * H + 1),
                (vpart[:, 2 * H:], G["b1v"], gw, 1, 2 * H + 1),
                (battn_part, G["b_attn"], ga, 1, 1),
                (wattn_part, G["w_attn"], gr, D, D),
            ])
            value_done = torch.cuda.Event(enable_timing=self.comm is not None
                                          and self.comm.timeline is not None)
            value_done.record()

        if fact:
            # logits = H2W[frame] + EP[prev] + PP[k] + b: three small GEMMs, no [M, A] logits
            h2w = ops.tc_linear(h2, P["w_head"], S.get("st.h2w", (F, A)))
            ep = ops.tc_linear(P["e_prev"], P["w_head"], S.get("st.ep", (A + 1, A)))
            pp = ops.tc_linear(P["e_pos"], P["w_head"], S.get("st.pp", (K, A)))
            epp = ops.ep_plus(ep, pp, P["b_head"], K, S.get("st.epp", ((A + 1) * K, A)))
            gf = ops.fact_partials(N, K, A, self.recompute_dz)
            # recompute_dz (default where K <= 8, A in {128, 256}): per-token
            # scalars instead of dz rows; the frame-blocked grouped sums
            # recompute dz from L2-resident H2W rows (saves the 4A bytes/token
            # dz write + read)
            if self.recompute_dz:
                tsc, dz = S.get("st.tsc", (M, 4)), None
            else:
                tsc, dz = None, S.get("st.dz", (M, A))
            g_frame = S.get("st.gframe", (F, A))
            if F != N:  # bootstrap frames have no transition: their G rows are zero
                boot = getattr(batch, "boot_rows", None)
                if boot is not None:
                    g_frame.index_fill_(0, boot, 0.0)
                else:
                    g_frame.zero_()
            stat_part = S.get("st.stat", (gf, 8), F64)
            max_part = S.get("st.max", (gf, 2), F64)
            loss_args = (h2w, epp, batch.frame_of, batch.tokens_dev, batch.lp_old, batch.adv, N,
                         K, algo, lc.sigma, lc.clip_eps, lc.lambda_h, M_glob, dz, g_frame)
            tsc_pos = None
            if tsc is not None and batch.pk_group.cpb > 0:
                tsc_pos = batch.pk_group.sort_rows(batch.frame_of, batch.tokens_dev, K)
            with self._timed("token_loss"):
                ops.token_loss_fact(*loss_args, lp_new, stat_part, max_part, tsc=tsc,
                                    tsc_pos=tsc_pos)
            gl = gf
        else:
            c = ops.build_c(h2, batch.frame_of, batch.tokens_dev, P["e_prev"], P["e_pos"], N, K,
                            A, S.get("st.c", (M, D)))
            logits = ops.tc_linear(c, P["w_head"], S.get("st.logits", (M, A)))
            gl = ops.token_grid(M)
            dlogits = S.get("st.dlogits", (M, A))
            dbias_part = S.get("st.dbias", (gl, A))
            stat_part = S.get("st.stat", (gl, 8), F64)
            max_part = S.get("st.max", (gl, 2), F64)
            with self._timed("token_loss"):
                ops.token_loss(logits, P["b_head"], batch.tokens_dev, batch.lp_old, batch.adv, K,
                               algo, lc.sigma, lc.clip_eps, lc.lambda_h, M_glob, dlogits, lp_new,
                               dbias_part, stat_part, max_part)
        ops.reduce_f64(stat_part, gl, 8, 0, loss_sums)
        ops.reduce_f64(max_part, gl, 2, 1, loss_max)
        if self.comm is not None:  # C5: token sums and maxima in one collective
            self.comm.all_reduce_sum_max(loss_sums, loss_max)
        # the value bucket's exchange queues after the loss all-reduces above (one
        # process group runs collectives in issue order: issued earlier, it would
        # hold the FIXUP pass behind the whole value-head branch)
        if self.comm is not None:
            self.comm.bucket_ready(self.layout.bucket_of("w_attn"), after=value_done)
        # FIXUP: only does work when 0 < excluded < M_global (decided on the device)
        if fact:
            ops.token_loss_fact(*loss_args, None, None, None, fix_stats=loss_sums, tsc=tsc,
                                tsc_pos=tsc_pos)
        else:
            ops.token_loss(logits, P["b_head"], batch.tokens_dev, batch.lp_old, batch.adv, K,
                           algo, lc.sigma, lc.clip_eps, lc.lambda_h, M_glob, dlogits, None,
                           dbias_part, None, None, fix_stats=loss_sums)


        # policy backward
        if fact:
            # D(prev,k) = grouped sums of dz; Dprev / Dpos marginals
            with self._timed("group_sum"):
                dpk_buf = S.get("st.dpk", ((A + 1) * K, A))
                if self.recompute_dz:
                    dpk = batch.pk_group.fact_rows_sum(h2w, epp, batch.frame_of, batch.tokens_dev,
                                                       tsc, K, dpk_buf)
                else:
                    dpk = batch.pk_group.rows_sum(dz, dpk_buf)
            dpp = S.get("st.dpp", (A + 1 + K, A))  # [Dprev; Dpos]
            dprev, dpos = dpp[:A + 1], dpp[A + 1:]
            ops.pk_marginals(dpk, K, A, dprev, dpos)
            # dW_head = G^T h2 + Dprev^T e_prev + Dpos^T e_pos   (sum_t dz_t (x) c_t):
            # the two small products ride along as one extra partial slice
            seg = self._wgrad(g_frame, h2, G["w_head"], "w_head", extra=1)
            small = seg[0][seg[2] - 1]
            # [Dprev; Dpos]^T [e_prev; e_pos] in one reduction (e_prev and e_pos are
            # adjacent in the flat parameter buffer)
            ops.tc_wgrad(dpp, self.params.rows("e_prev", A + 1 + K), small)
            ops.tc_matmul_nn(dprev, P["w_head"], G["e_prev"])
            ops.tc_matmul_nn(dpos, P["w_head"], G["e_pos"])
            ops.reduce_segments([seg, (dpos, G["b_head"], K, A, A)])
            self._bucket_done("w_head")
            # dpre2 = (G W_head) (1 - h2^2) and its column sums (db1), one kernel
            dz2, db1_part, gd = ops.tc_matmul_nn_dtanh(
                g_frame, P["w_head"], h2, S.get("st.dz2", (F, D)),
                lambda n: S.get("st.db1", (n, D)))
        else:
            seg = self._wgrad(dlogits, c, G["w_head"], "w_head")
            dc = ops.tc_matmul_nn(dlogits, P["w_head"], c)  # c is dead after dW_head: reuse it
            dz2 = S.get("st.dz2", (F, D))
            if F != N:
                dz2.zero_()
            gd = ops.rows_grid(N)
            pos_part = S.get("st.pos", (gd, K, D))
            db1_part = S.get("st.db1", (gd, D))
            ops.dc_reduce(dc, h2, batch.frame_of, N, K, D, dz2, pos_part, db1_part, gd)
            batch.prev_group.rows_sum(dc, G["e_prev"])
            ops.reduce_segments([seg, (dbias_part, G["b_head"], gl, A, A),
                                 (pos_part, G["e_pos"], gd, K * D, K * D)])
            self._bucket_done("w_head")
        ops.reduce_segments([self._wgrad(dz2, h1, G["w1"], "w1"), (db1_part, G["b1"], gd, D, D)])
        self._bucket_done("w1")
        # dpre1 = (dpre2 W1) (1 - h1^2) and its column sums (db0)
        dh1, db0_part, gt = ops.tc_matmul_nn_dtanh(dz2, P["w1"], h1, S.get("st.dh1", (F, D)),
                                                   lambda n: S.get("st.db0", (n, D)))
        ops.reduce_segments([self._wgrad(dh1, batch.frames, G["w0"], "w0"),
                             (db0_part, G["b0"], gt, D, D)])
        self._bucket_done("w0")
        torch.cuda.current_stream().wait_stream(side)  # the value branch has finished
        value_sums = S.get("st.vsum", (2,), F64)
        attn_bad = S.get("st.abad", (2,), F64)
        ops.reduce_f64(vdpart, gw, 2, 0, value_sums)
        ops.reduce_f64(vbad_part, nbad, 2, 0, attn_bad)
        ops.count_nonfinite(self.params.g, cnt[0:1])
        if self.comm is not None:
            # C5 scalars in one fp64 all-reduce; local grads all finite on every
            # rank <=> the reduced grads are finite (barring overflow)
            sc = torch.cat([value_sums, attn_bad, cnt[0:2].double()])
            self.comm.all_reduce_sum(sc)
            value_sums.copy_(sc[0:2])
            attn_bad.copy_(sc[2:4])
            cnt[0:2].copy_(sc[4:6].to(torch.int32))
        record = S.get("st.record", (17,), F64)
        skip = S.get("st.skip", (1,), torch.int32)
        ops.step_finalize(loss_sums, loss_max, value_sums, cnt, attn_bad, algo, lc.lambda_v,
                          lc.lambda_h, M_glob, N_glob, record, skip)

        # Adam on both groups (ping-pong; no-op when skip)
        cur, nxt = self.params.cur, self.params.cur ^ 1
        if self.comm is not None:
            self.comm.finish_step()  # the last buckets' exchange; the stream waits for it
            ops.count_nonfinite(self.params.p[nxt], adam_bad)
        else:
            ops.adam_dev(self.params.p[cur], self.params.g, self.params.m[cur],
                         self.params.v[cur], self.params.p[nxt], self.params.m[nxt],
                         self.params.v[nxt], self.layout.n_policy, self._hyper_dev, skip,
                         adam_bad)
        out = S.get("st.out", (18,), F64)
        out[:17].copy_(record)
        out[17:18].copy_(adam_bad.double())
        return out

    def _finish_step(self, batch, record_dev: torch.Tensor | None, rec=None) -> dict | None:
        if rec is None:
            host = self._rec_host[:18]
            host.copy_(record_dev, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            rec = host.numpy().copy()
        if rec[11] > 0:
            raise DomainError("log_softmax input contains non-finite values")
        if rec[12] > 0:
            raise DimensionError("token index outside the action vocabulary")
        if rec[13] > 0:
            raise DomainError("softmax input contains non-finite values")
        if rec[15] > 0:
            raise DimensionError(f"step index outside value-step table [0, {self.dims.n_steps})")
        if rec[10] > 0:
            self.skipped += 1
            if self.metrics is not None:
                self.metrics.emit("train_skip", skipped=self.skipped)
            return None
        if rec[14] > 0:
            raise NonFiniteError("gradient contains non-finite values")
        if rec[17] > 0:
            raise NonFiniteError("parameter update produced non-finite values")
        self.params.flip()
        self._param_gen += 1
        self.adam_policy.step += 1
        self.adam_value.step += 1
        self._policy_version += 1
        self._value_version += 1
        self._host_stale = True
        self.cycles += 1
        self.publish_version += 1
        self.publish_policy()
        out = {
            "loss": float(rec[0]), "policy_loss": float(rec[1]), "value_loss": float(rec[2]),
            "entropy": float(rec[3]), "version": self.publish_version,
            "critic_version": batch.critic_version, "behavior_lag": batch.behavior_lag_mean,
            "n_real": batch.n_real, "n_imagined": batch.n_imagined,
            "excluded_tokens": int(rec[4]),
        }
        if self.cfg.loss.algorithm == "trust":
            out["trust_weight_mean"] = float(rec[7])
            out["trust_weight_min"] = float(rec[8])
        else:
            out["clipped_fraction"] = float(rec[9])
        out["ratio_mean"] = float(rec[5])
        out["ratio_max"] = float(rec[6])
        if self.metrics is not None:
            self.metrics.emit("train_step", **out)
        return out

    # -- CUDA graphs ------------------------------------------------------------------
    def capture_step(self, inputs: dict, n_real: int, behavior_version) -> "CapturedStep":
        """build_from_device + train_step of a fixed-shape device batch as CUDA
        graphs (see CapturedStep): the launch-bound small configurations (cfg1)
        run as one graph launch and one pinned readback per step."""
        return CapturedStep(self, inputs, n_real, behavior_version)

    # -- loop (trainer.py:539-560) -------------------------------------------------------
    def run(self, cache, wm_buffer, stop) -> Generator:
        """Consume TrainBatches from the prefetch channel until stopped.

        Yields the reference runtime's effects (`Get`, `Sleep`), so it runs
        on the reference `Scheduler` unchanged; effect classes are taken from
        the channel's module to stay duck-typed."""
        from importlib import import_module
        rt = import_module(type(cache).__module__)
        cfg = self.cfg
        while not stop.is_set:
            item = yield rt.Get(cache, timeout=cfg.poll_interval)
            if item is rt.CLOSED:
                return
            if item is rt.TIMEOUT:
                continue
            if cfg.train_service_time > 0:
                yield rt.Sleep(cfg.train_service_time)
            record = self.train_step(item)
            # world-model updates every t_obs / t_reward optimizer cycles (trainer.py:552-560)
            if record is not None and cfg.world_model and wm_buffer is not None:
                if self.cycles % cfg.t_obs == 0:
                    trajs = wm_buffer.sample(cfg.wm_batch_episodes, self.rng)
                    if trajs:
                        self.train_obs_model_step(trajs)
                if self.cycles % cfg.t_reward == 0:
                    trajs = wm_buffer.sample(cfg.wm_batch_episodes, self.rng)
                    if trajs:
                        self.train_reward_model_step(trajs)


class CapturedStep:
    """One optimizer step (build_from_device + train_step) on a fixed set of
    device input buffers, captured as CUDA graphs.

    Every launch of the step -- revaluation, GAE, normalization, behavior
    log-probs, the fused loss, backward, Adam, the record -- is stream-ordered
    with its decisions made on the device (the FIXUP pass, the skip flag), so
    the only host work per step is one replay, one pinned readback of the
    build flags + the record, and the reference's record / error logic.  The
    parameters are ping-ponged (Adam reads generation cur, writes cur ^ 1), so
    one graph is captured per parity, on first use; the Adam step counters
    enter through device memory (Trainer._hyper_dev, refreshed before each
    replay).  Refill the `inputs` tensors in place between runs (same shapes);
    the trainer must not be given other batch shapes while a CapturedStep is
    live (its scratch buffers are the graphs' buffers).  Single GPU only.
    """

    def __init__(self, trainer: Trainer, inputs: dict, n_real: int, behavior_version) -> None:
        if trainer.comm is not None:
            raise DomainError("graph capture is single-GPU (the ZeRO-2 path has host-side "
                              "collectives)")
        if trainer.profile_events is not None:
            raise DomainError("disable profile_events before capturing")
        self.tr = trainer
        self.inputs = inputs
        self.n_real = int(n_real)
        self.bver = np.asarray(behavior_version, dtype=np.int64)
        self.n = int(inputs["traj_off"].shape[0] - 1)
        self._graphs: dict = {}
        ops.retain_workspaces()  # captured addresses must stay valid
        self._out_host = torch.zeros(64, dtype=F64).pin_memory()

    def _run_eager(self):
        tr = self.tr
        batch, host_dev = tr._build_device(self.inputs, self.n_real, self.bver)
        rec = tr._step_device(batch)
        return batch, torch.cat([host_dev, rec])

    def _capture(self):
        # warm-up on a side stream (every scratch buffer and workspace sized),
        # then capture; neither result is adopted (the host does not flip)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self._run_eager()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            batch, out = self._run_eager()
        return g, batch, out

    def run(self) -> dict | None:
        """Replay one step; returns the train_step record, or None when the
        batch is rejected (non-finite) or dropped (every token excluded)."""
        tr = self.tr
        cur = tr.params.cur
        if cur not in self._graphs:
            self._graphs[cur] = self._capture()
        g, batch, out = self._graphs[cur]
        tr._write_hyper()  # the graph copies it to the device first
        g.replay()
        host = self._out_host[:out.numel()]
        host.copy_(out, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        vals = host.numpy().copy()
        nb = out.numel() - 18
        batch.critic_version = tr.publish_version
        batch.behavior_lag_mean = float(np.mean(tr.publish_version - self.bver))
        if tr._build_finish(batch, vals[:nb]) is None:
            return None
        return tr._finish_step(batch, None, rec=vals[nb:])


__all__ = [
    "GaeConfig", "LossConfig", "TrainerConfig", "Trainer", "ShardStats", "compute_gae",
    "shard_statistics", "global_normalize", "trust_weight", "chunk_ratio", "policy_surrogate",
    "entropy_bonus", "total_loss", "behavior_log_probs", "POLICY_NAMES", "VALUE_NAMES",
    "CapturedStep",
]
