"""World-model training sub-steps on the device.

Reference: `Trainer.train_obs_model_step` / `train_reward_model_step`
(trainer.py:469-535) with `mlp_forward` / `mlp_backward` (numerics.py:174-220)
and `adam_step` (numerics.py:95-126).  The host keeps the reference's control
flow -- which frames and transitions enter a sub-step, the `rng.choice`
subsampling on the trainer's own generator, the error conventions -- and the
arithmetic (2-layer tanh MLP forward, MSE / BCE loss, backward, Adam) runs on
the device in float64, the reference's dtype (`csrc/world_model.cu`).
Parameters and Adam moments stay resident between sub-steps; host model
objects are rebuilt only when the bundle is read.
"""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np
import torch

from . import ops
from .errors import DimensionError, DomainError, NonFiniteError

F64 = torch.float64
NAMES = ("w0", "b0", "w1", "b1")  # flat layout of csrc/world_model.cu


def chunk_onehot(tokens: np.ndarray, n_actions: int) -> np.ndarray:
    """(..., K) int tokens -> (..., K * n_actions) one-hot (models.py:53-58)."""
    t = np.asarray(tokens, dtype=np.int64)
    out = np.zeros(t.shape + (n_actions,), dtype=np.float64)
    np.put_along_axis(out, t[..., None], 1.0, axis=-1)
    return out.reshape(t.shape[:-1] + (t.shape[-1] * n_actions,))


class DeviceMlp2:
    """A 2-layer tanh MLP's parameters, gradients and Adam moments (float64,
    device-resident), with the reference's ParamSet version and AdamState step."""

    def __init__(self, params, lr: float, beta1: float, beta2: float, eps: float,
                 device) -> None:
        t = params.tensors
        if set(t) != set(NAMES):
            raise DimensionError(f"world-model MLP needs tensors {NAMES}, got {sorted(t)}")
        self.dh, self.din = t["w0"].shape
        self.dout = t["w1"].shape[0]
        self.shapes = {k: np.asarray(t[k]).shape for k in NAMES}
        self.version = int(getattr(params, "version", 0))
        self.param_type = type(params)
        flat = np.concatenate([np.asarray(t[k], dtype=np.float64).ravel() for k in NAMES])
        self.p = torch.from_numpy(flat).to(device)
        self.g = torch.zeros_like(self.p)
        self.m = torch.zeros_like(self.p)
        self.v = torch.zeros_like(self.p)
        self.loss = torch.zeros(1, dtype=F64, device=device)
        self.flags = torch.zeros(2, dtype=torch.int32, device=device)
        self.step = 0
        self.lr, self.beta1, self.beta2, self.eps = lr, beta1, beta2, eps
        self._host = None

    def tensors(self, flat: torch.Tensor) -> dict:
        host = flat.cpu().numpy()
        out, i = {}, 0
        for k in NAMES:
            n = int(np.prod(self.shapes[k]))
            out[k] = host[i:i + n].reshape(self.shapes[k]).copy()
            i += n
        return out

    def params(self):
        """Host ParamSet (cached until the next update)."""
        if self._host is None:
            self._host = self.param_type(self.tensors(self.p), self.version)
        return self._host

    def adam_state(self):
        """AdamState-like view (m, v, step, hyperparameters) for inspection."""
        return SimpleNamespace(m=self.tensors(self.m), v=self.tensors(self.v), step=self.step,
                               lr=self.lr, beta1=self.beta1, beta2=self.beta2, eps=self.eps)

    def update(self, x: np.ndarray, target: np.ndarray, kind: int) -> float:
        """One forward/backward + Adam step; returns the loss (one host sync for
        the loss and the gradient check, one for the parameter check)."""
        dev = self.p.device
        xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(dev)
        td = torch.from_numpy(np.ascontiguousarray(target, dtype=np.float64)).to(dev)
        nonfinite = self.flags[0:1]
        ops.wm_mlp2_grad(xd, td, self.din, self.dh, self.dout, kind, self.p, self.g, self.loss,
                         nonfinite)
        host = torch.cat([self.loss, self.flags[0:1].double()]).cpu().numpy()
        if host[1] != 0:  # adam_step raises before touching the parameters
            raise NonFiniteError("world-model gradient contains non-finite values")
        t = self.step + 1
        ops.wm_adam(self.p, self.g, self.m, self.v, self.lr, self.beta1, self.beta2, self.eps, t,
                    self.flags[1:2])
        self.step = t
        self.version += 1
        self._host = None
        if int(self.flags[1].item()) != 0:  # ParamSet.check_finite on the new parameters
            raise NonFiniteError("world-model parameters became non-finite")
        return float(host[0])


def obs_model_data(obs_model, trajs, max_rows: int, rng):
    """(x, y) of train_obs_model_step (trainer.py:471-483): encode_input(o_t, a_t)
    -> o_{t+1} over every transition, subsampled to max_rows by rng.choice."""
    n_actions = obs_model.cfg.n_actions
    xs, ys = [], []
    for traj in trajs:
        T = traj.tokens.shape[0]
        if T == 0:
            continue
        obs = np.asarray(traj.observations, dtype=np.float64)
        xs.append(np.concatenate([obs[:T], chunk_onehot(traj.tokens[:T], n_actions)], axis=1))
        ys.append(obs[1:T + 1])
    if not xs:
        raise DomainError("no transitions to fit")
    x, y = np.concatenate(xs), np.concatenate(ys)
    if x.shape[0] > max_rows:
        idx = rng.choice(x.shape[0], size=max_rows, replace=False)
        x, y = x[idx], y[idx]
    return x, y


def reward_model_data(trajs, neg_ratio: int, max_rows: int, rng):
    """(frames, labels, single_class) of train_reward_model_step (trainer.py:498-518):
    positives are the terminal frames of successful episodes, negatives every other
    frame, subsampled to neg_ratio per positive (or max_rows without positives)."""
    pos, neg = [], []
    for traj in trajs:
        succeeded = bool(np.sum(traj.rewards) > 0)
        frames = traj.observations
        last = frames.shape[0] - 1
        for i in range(frames.shape[0]):
            (pos if succeeded and i == last else neg).append(frames[i])
    max_neg = len(pos) * neg_ratio if pos else max_rows
    if len(neg) > max_neg:
        idx = rng.choice(len(neg), size=max_neg, replace=False)
        neg = [neg[i] for i in idx]
    single_class = not pos or not neg
    frames = pos + neg
    labels = np.concatenate([np.ones(len(pos)), np.zeros(len(neg))])
    x = np.stack(frames).astype(np.float64)
    return x, labels, single_class
