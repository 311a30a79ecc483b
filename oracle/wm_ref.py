"""Float64 NumPy restatement of the world-model training sub-steps.

TEST INFRASTRUCTURE ONLY: the product never imports this module; tests use it
as the checker.  Reference: `mlp_forward` / `mlp_backward` (numerics.py:174-220),
`adam_step` (numerics.py:95-126) and the losses of `train_obs_model_step` /
`train_reward_model_step` (trainer.py:484-489, :519-523).  Parity is pinned to
fixtures made by the real reference (tests/golden/make_golden_wm.py).
"""

from __future__ import annotations

import numpy as np

NAMES = ("w0", "b0", "w1", "b1")


def mlp2_forward(p: dict, x: np.ndarray):
    h = np.tanh(x @ p["w0"].T + p["b0"])          # numerics.py:189-192
    return h @ p["w1"].T + p["b1"], h


def mlp2_backward(p: dict, x: np.ndarray, h: np.ndarray, g: np.ndarray) -> dict:
    grads = {"w1": g.T @ h, "b1": g.sum(axis=0)}   # numerics.py:212-216
    gh = (g @ p["w1"]) * (1.0 - h ** 2)            # tanh' (numerics.py:218)
    grads["w0"] = gh.T @ x
    grads["b0"] = gh.sum(axis=0)
    return grads


def loss_and_grad(p: dict, x: np.ndarray, target: np.ndarray, kind: int):
    out, h = mlp2_forward(p, x)
    if kind == 0:                                  # MSE (trainer.py:484-487)
        err = out - target
        loss = float(np.mean(err ** 2))
        g = 2.0 * err / err.size
    else:                                          # BCE from logits (trainer.py:519-523)
        z = out[:, 0]
        loss = float(np.mean(np.logaddexp(0.0, z) - target * z))
        g = ((1.0 / (1.0 + np.exp(-z)) - target) / target.size)[:, None]
    return loss, mlp2_backward(p, x, h, g)


def adam(p: dict, g: dict, m: dict, v: dict, t: int, lr: float, b1: float = 0.9,
         b2: float = 0.999, eps: float = 1e-8):
    """numerics.py:106-116; returns new (p, m, v)."""
    np_, nm, nv = {}, {}, {}
    for k in p:
        nm[k] = b1 * m[k] + (1.0 - b1) * g[k]
        nv[k] = b2 * v[k] + (1.0 - b2) * g[k] * g[k]
        mh = nm[k] / (1.0 - b1 ** t)
        vh = nv[k] / (1.0 - b2 ** t)
        np_[k] = p[k] - lr * mh / (np.sqrt(vh) + eps)
    return np_, nm, nv
