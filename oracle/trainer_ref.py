"""Float64 NumPy restatement of the reference trainer path (TEST INFRASTRUCTURE).

Every function names the reference lines it restates (paths relative to
`/root/reference/pkg/src/asyncrl/`).  Parameters are plain ``dict[str,
ndarray]``; trajectories are any objects exposing the reference
`Trajectory` fields (`rollout.py:31-86`).  The arithmetic order follows the
reference wherever it affects float64 rounding that the golden fixtures pin.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


class OracleDomainError(ValueError):
    """Mirrors numerics.DomainError (numerics.py:24-25)."""


class OracleDimensionError(ValueError):
    """Mirrors numerics.DimensionError (numerics.py:20-21)."""


class OracleNonFiniteError(ValueError):
    """Mirrors numerics.NonFiniteError (numerics.py:28-29)."""


# ---------------------------------------------------------------------------
# softmax family — numerics.py:133-151 (max-shifted, float64)


def log_softmax(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.float64)
    if z.size == 0:
        raise OracleDomainError("log_softmax of an empty vector")
    if not np.isfinite(z).all():
        raise OracleDomainError("log_softmax input contains non-finite values")
    s = z - z.max(axis=-1, keepdims=True)
    return s - np.log(np.exp(s).sum(axis=-1, keepdims=True))


def softmax(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.float64)
    if z.size == 0:
        raise OracleDomainError("softmax of an empty vector")
    if not np.isfinite(z).all():
        raise OracleDomainError("softmax input contains non-finite values")
    e = np.exp(z - z.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


# ---------------------------------------------------------------------------
# (a) advantages — trainer.py:79-101 (GAE), :108-158 (pooled normalization)


def gae(rewards, values, done: bool, gamma: float, lam: float):
    """Reverse recursion A_t = delta_t + gamma*lam*A_{t+1}; trainer.py:79-101.

    values holds T+1 entries (bootstrap last); a done episode zeroes the
    bootstrap (trainer.py:92-93).  Returns (advantages, value targets).
    """
    r = np.asarray(rewards, dtype=np.float64)
    v = np.array(values, dtype=np.float64)
    T = r.shape[0]
    if v.shape != (T + 1,):
        raise OracleDomainError(f"values must have length T+1={T + 1}, got {v.shape}")
    if T == 0:
        raise OracleDomainError("empty trajectory")
    if done:
        v[T] = 0.0
    delta = r + gamma * v[1:] - v[:T]
    out = np.empty(T)
    carry = 0.0
    decay = gamma * lam
    for t in range(T - 1, -1, -1):
        carry = delta[t] + decay * carry
        out[t] = carry
    return out, out + v[:T]


def shard_stats(shards):
    """(S, Q, N) per shard — trainer.py:128-132; Cauchy-Schwarz check :121."""
    s = np.array([float(np.sum(a)) for a in shards])
    q = np.array([float(np.sum(np.square(a))) for a in shards])
    n = np.array([float(np.size(a)) for a in shards])
    if np.any(n * q - s * s < -1e-9):
        raise OracleDomainError("inconsistent shard stats: N*Q < S^2")
    return s, q, n


def pooled_normalize(shards, eps: float = 1e-8):
    """Eqs. 5-7 from shard sums — trainer.py:135-158."""
    s, q, n = shard_stats(shards)
    total = float(np.sum(n))
    if total == 0:
        raise OracleDomainError("cannot normalize zero advantages")
    mean = float(np.sum(s)) / total
    var = float(np.sum(q)) / total - mean * mean
    if var < -1e-12:
        raise OracleDomainError(f"negative pooled variance {var}")
    var = max(var, 0.0)
    scale = np.sqrt(var) + eps
    out = [(np.asarray(a, dtype=np.float64) - mean) / scale for a in shards]
    return out, {"mean": mean, "std": float(np.sqrt(var)), "n": int(total),
                 "shard_sizes": tuple(int(k) for k in n)}


# ---------------------------------------------------------------------------
# (b) token loss — trainer.py:165-256, models.py:219-223, trainer.py:289-293


def trust_weight(ratio, sigma: float):
    """Gaussian weight in log-ratio space — trainer.py:165-175."""
    r = np.asarray(ratio, dtype=np.float64)
    if np.any(r <= 0) or not np.all(np.isfinite(r)):
        raise OracleDomainError("trust weight needs finite ratios > 0")
    w = np.exp(-0.5 * np.square(np.log(r) / sigma))
    return float(w) if np.isscalar(ratio) else w


def chosen_logp(logits, tokens):
    """log_softmax gathered at the chosen token — models.py:219-223 and
    trainer.py:289-293 (behavior_log_probs is the same arithmetic)."""
    lp = log_softmax(logits)
    t = np.asarray(tokens, dtype=np.int64)
    return np.take_along_axis(lp, t[..., None], axis=-1)[..., 0]


def surrogate(lp_new, lp_old, adv, algorithm: str = "trust", sigma: float = 0.3,
              clip_eps: float = 0.2, trust_weights=None):
    """Token surrogate and d loss / d lp_new — trainer.py:183-239.

    Returns (loss, dlogp, diag); diag["dropped"] marks an all-excluded batch.
    """
    lpn = np.asarray(lp_new, dtype=np.float64)
    lpo = np.asarray(lp_old, dtype=np.float64)
    a_tok = np.broadcast_to(np.asarray(adv, dtype=np.float64)[:, None], lpn.shape)
    with np.errstate(over="ignore", invalid="ignore"):
        ratio = np.exp(lpn - lpo)
    inc = np.isfinite(ratio) & (ratio > 0)
    diag = {"excluded_tokens": int(inc.size - inc.sum()), "dropped": False}
    grad = np.zeros_like(lpn)
    if not inc.any():
        diag["dropped"] = True
        return 0.0, grad, diag
    m = float(inc.sum())
    r = np.where(inc, ratio, 1.0)
    a = np.where(inc, a_tok, 0.0)
    if algorithm == "trust":
        if trust_weights is None:
            w = np.where(inc, trust_weight(r, sigma), 0.0)
        else:
            w = np.where(inc, trust_weights, 0.0)
        loss = -float((w * r * a)[inc].sum()) / m
        grad = -(w * r * a) / m
        grad[~inc] = 0.0
        diag["trust_weight_mean"] = float(w[inc].mean())
        diag["trust_weight_min"] = float(w[inc].min())
    elif algorithm == "clip":
        lo, hi = 1.0 - clip_eps, 1.0 + clip_eps
        rc = np.clip(r, lo, hi)
        loss = -float(np.minimum(r * a, rc * a)[inc].sum()) / m
        grad = np.where(r * a <= rc * a, -(r * a) / m, 0.0)
        grad[~inc] = 0.0
        diag["clipped_fraction"] = float(((r < lo) | (r > hi))[inc].mean())
    else:
        raise OracleDomainError(f"unknown algorithm {algorithm!r}")
    diag["ratio_mean"] = float(r[inc].mean())
    diag["ratio_max"] = float(r[inc].max())
    return loss, grad, diag


def entropy(logits):
    """Mean token entropy and its logits gradient — trainer.py:242-251."""
    lp = log_softmax(logits)
    p = np.exp(lp)
    h_tok = -np.sum(p * lp, axis=-1)
    count = float(h_tok.size)
    return float(h_tok.sum()) / count, -p * (lp + h_tok[..., None]) / count


def loss_dlogits(logits, tokens, dlogp, lambda_h: float):
    """dlogits assembly of train_step — trainer.py:425-435."""
    _, d_ent = entropy(logits)
    p = softmax(logits)
    d = -dlogp[..., None] * p
    flat = d.reshape(-1, d.shape[-1])
    np.add.at(flat, (np.arange(dlogp.size), np.asarray(tokens).ravel()), dlogp.ravel())
    return d - lambda_h * d_ent


# ---------------------------------------------------------------------------
# models — models.py:165-217 (teacher-forced policy), :273-314 (value head)


def backbone(p: dict, x):
    """h1, h2 — models.py:211-217 (same math as forward_teacher :176-177)."""
    x = np.asarray(x, dtype=np.float64)
    h1 = np.tanh(x @ p["w0"].T + p["b0"])
    h2 = np.tanh(h1 @ p["w1"].T + p["b1"])
    return h1, h2


def policy_forward(p: dict, n_actions: int, x, tokens):
    """Teacher-forced logits (N, K, A) plus cache — models.py:165-184."""
    x = np.asarray(x, dtype=np.float64)
    t = np.asarray(tokens, dtype=np.int64)
    h1, h2 = backbone(p, x)
    prev = np.empty_like(t)
    prev[:, 0] = n_actions
    prev[:, 1:] = t[:, :-1]
    c = h2[:, None, :] + p["e_prev"][prev] + p["e_pos"][None, :, :]
    logits = c @ p["w_head"].T + p["b_head"]
    return logits, {"x": x, "h1": h1, "h2": h2, "prev": prev, "c": c}


def policy_backward(p: dict, cache: dict, dlogits):
    """Gradients of sum(dlogits * logits) — models.py:186-209."""
    x, h1, h2, prev, c = (cache[k] for k in ("x", "h1", "h2", "prev", "c"))
    d = h2.shape[1]
    g = {"w_head": np.einsum("nka,nkd->ad", dlogits, c),
         "b_head": dlogits.sum(axis=(0, 1))}
    dc = dlogits @ p["w_head"]
    g["e_prev"] = np.zeros_like(p["e_prev"])
    np.add.at(g["e_prev"], prev.ravel(), dc.reshape(-1, d))
    g["e_pos"] = dc.sum(axis=0)
    dz2 = dc.sum(axis=1) * (1.0 - h2 ** 2)
    g["w1"] = dz2.T @ h1
    g["b1"] = dz2.sum(axis=0)
    dz1 = (dz2 @ p["w1"]) * (1.0 - h1 ** 2)
    g["w0"] = dz1.T @ x
    g["b0"] = dz1.sum(axis=0)
    return g


def value_forward(vp: dict, n_steps: int, hs, steps):
    """Attention-pooled value head — models.py:273-290 (bounds :261-267)."""
    hs = np.asarray(hs, dtype=np.float64)
    t = np.asarray(steps, dtype=np.int64)
    if np.any(t < 0) or np.any(t >= n_steps):
        raise OracleDimensionError(f"step index outside value-step table [0, {n_steps})")
    e = hs @ vp["w_attn"] + vp["b_attn"][0]
    alpha = softmax(e)
    u = np.einsum("ni,nid->nd", alpha, hs) + vp["e_step"][t]
    m = np.tanh(u @ vp["w0v"].T + vp["b0v"])
    v = (m @ vp["w1v"].T + vp["b1v"])[:, 0]
    return v, {"hs": hs, "t": t, "alpha": alpha, "u": u, "m": m}


def value_backward(vp: dict, cache: dict, dv):
    """Value-head parameter gradients, hiddens detached — models.py:292-314."""
    hs, t, alpha, u, m = (cache[k] for k in ("hs", "t", "alpha", "u", "m"))
    dv = np.asarray(dv, dtype=np.float64)[:, None]
    g = {"w1v": dv.T @ m, "b1v": dv.sum(axis=0)}
    dzm = (dv @ vp["w1v"]) * (1.0 - m ** 2)
    g["w0v"] = dzm.T @ u
    g["b0v"] = dzm.sum(axis=0)
    du = dzm @ vp["w0v"]
    g["e_step"] = np.zeros_like(vp["e_step"])
    np.add.at(g["e_step"], t, du)
    da = np.einsum("nd,nid->ni", du, hs)
    de = alpha * (da - (alpha * da).sum(axis=1, keepdims=True))
    g["w_attn"] = np.einsum("ni,nid->d", de, hs)
    g["b_attn"] = np.array([de.sum()])
    return g


# ---------------------------------------------------------------------------
# optimizer — numerics.py:95-126


@dataclass
class AdamSlots:
    m: dict
    v: dict
    step: int = 0
    lr: float = 3e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8

    @classmethod
    def zeros(cls, params: dict, **hyper) -> "AdamSlots":
        return cls({k: np.zeros_like(a) for k, a in params.items()},
                   {k: np.zeros_like(a) for k, a in params.items()}, **hyper)


def adam(params: dict, grads: dict, st: AdamSlots):
    """Bias-corrected Adam, pure — numerics.py:95-126."""
    if set(grads) != set(params):
        raise OracleDimensionError("gradient names do not match parameters")
    t = st.step + 1
    new_p, new_m, new_v = {}, {}, {}
    for k, w in params.items():
        g = np.asarray(grads[k], dtype=np.float64)
        if g.shape != w.shape:
            raise OracleDimensionError(f"gradient {k!r}: shape mismatch")
        if not np.all(np.isfinite(g)):
            raise OracleNonFiniteError(f"gradient {k!r} contains non-finite values")
        m = st.beta1 * st.m[k] + (1.0 - st.beta1) * g
        v = st.beta2 * st.v[k] + (1.0 - st.beta2) * g * g
        mh = m / (1.0 - st.beta1 ** t)
        vh = v / (1.0 - st.beta2 ** t)
        new_p[k] = w - st.lr * mh / (np.sqrt(vh) + st.eps)
        new_m[k], new_v[k] = m, v
    for k, w in new_p.items():
        if not np.all(np.isfinite(w)):
            raise OracleNonFiniteError(f"parameter tensor {k!r} contains non-finite values")
    return new_p, AdamSlots(new_m, new_v, t, st.lr, st.beta1, st.beta2, st.eps)


# ---------------------------------------------------------------------------
# trainer — trainer.py:263-467


@dataclass
class OracleConfig:
    """TrainerConfig subset on the hot path — trainer.py:44-72, :263-286."""
    gamma: float = 0.99
    lam: float = 0.95
    algorithm: str = "trust"
    sigma: float = 0.3
    clip_eps: float = 0.2
    lambda_v: float = 0.5
    lambda_h: float = 0.01
    lr: float = 3e-4
    beta1: float = 0.9
    beta2: float = 0.999
    k_shards: int = 4
    eps_norm: float = 1e-8
    revalue: bool = True
    value_clip: float | None = None  # north-star value-clip loss (no reference counterpart)


def value_loss_clipped(v, ret, v_old, eps):
    """PPO value clipping: mean(max((v - R)^2, (v_old + clip(v - v_old, +-eps) - R)^2)) and
    dL/dv (per element, before the 1/N mean).  Not in the reference (trainer.py:438-443 is
    plain MSE): restated here so the opt-in kernel path has a float64 checker."""
    v, ret, v_old = (np.asarray(a, dtype=np.float64) for a in (v, ret, v_old))
    d = v - v_old
    vc = v_old + np.clip(d, -eps, eps)
    l1, l2 = (v - ret) ** 2, (vc - ret) ** 2
    loss = np.maximum(l1, l2)
    g = np.where(l1 >= l2, 2.0 * (v - ret), np.where(np.abs(d) < eps, 2.0 * (vc - ret), 0.0))
    return float(np.mean(loss)), g


@dataclass
class OracleBatch:
    """TrainBatch fields — buffers.py:97-122."""
    obs: np.ndarray
    steps: np.ndarray
    tokens: np.ndarray
    behavior_logp: np.ndarray
    advantages: np.ndarray
    value_targets: np.ndarray
    critic_version: int
    n_real: int
    n_imagined: int
    norm_mean: float
    norm_std: float
    norm_count: int
    shard_sizes: tuple
    behavior_lag_mean: float
    old_values: np.ndarray | None = None  # rollout-time V per transition (value clipping)

    @property
    def n_transitions(self) -> int:
        return int(self.obs.shape[0])

    def check_finite(self) -> bool:
        return all(np.all(np.isfinite(a)) for a in
                   (self.obs, self.behavior_logp, self.advantages, self.value_targets))


@dataclass
class OracleTrainer:
    """build_train_batch / train_step of trainer.py:358-467 on dict params.

    policy/value: parameter dicts; n_actions and n_steps size the heads.
    """
    policy: dict
    value: dict
    n_actions: int
    n_steps: int
    cfg: OracleConfig = field(default_factory=OracleConfig)
    publish_version: int = 0
    cycles: int = 0
    skipped: int = 0
    policy_version: int = 0
    value_version: int = 0

    def __post_init__(self) -> None:
        self.policy = {k: np.array(a, dtype=np.float64) for k, a in self.policy.items()}
        self.value = {k: np.array(a, dtype=np.float64) for k, a in self.value.items()}
        hyper = dict(lr=self.cfg.lr, beta1=self.cfg.beta1, beta2=self.cfg.beta2)
        self.adam_policy = AdamSlots.zeros(self.policy, **hyper)
        self.adam_value = AdamSlots.zeros(self.value, **hyper)

    def state_values(self, obs, steps):
        """state_values_batch — models.py:411-415."""
        h1, h2 = backbone(self.policy, obs)
        v, _ = value_forward(self.value, self.n_steps, np.stack([h1, h2], axis=1), steps)
        return v

    def build_train_batch(self, trajs):
        """trainer.py:358-403."""
        c = self.cfg
        parts = {k: [] for k in ("obs", "steps", "tokens", "logp", "adv", "ret", "vold")}
        lags, n_real = [], 0
        for tr in trajs:
            if c.revalue:
                vals = self.state_values(tr.observations, tr.steps)
            else:
                vals = np.append(tr.values, tr.bootstrap_value)
            adv, ret = gae(tr.rewards, vals, bool(tr.done), c.gamma, c.lam)
            parts["obs"].append(np.asarray(tr.observations)[:-1])
            parts["steps"].append(np.asarray(tr.steps)[:-1])
            parts["tokens"].append(np.asarray(tr.tokens))
            parts["logp"].append(chosen_logp(tr.behavior_logits, tr.tokens))
            parts["adv"].append(adv)
            parts["ret"].append(ret)
            parts["vold"].append(np.asarray(tr.values, dtype=np.float64))
            lags.append(self.publish_version - tr.behavior_version)
            n_real += tr.source == "real"
        normalized, summ = pooled_normalize(np.array_split(np.concatenate(parts["adv"]),
                                                           c.k_shards), c.eps_norm)
        batch = OracleBatch(
            obs=np.concatenate(parts["obs"]),
            steps=np.concatenate(parts["steps"]).astype(np.int64),
            tokens=np.concatenate(parts["tokens"]).astype(np.int64),
            behavior_logp=np.concatenate(parts["logp"]),
            advantages=np.concatenate(normalized),
            value_targets=np.concatenate(parts["ret"]),
            critic_version=self.publish_version, n_real=n_real,
            n_imagined=len(trajs) - n_real, norm_mean=summ["mean"],
            norm_std=summ["std"], norm_count=summ["n"],
            shard_sizes=summ["shard_sizes"], behavior_lag_mean=float(np.mean(lags)),
            old_values=np.concatenate(parts["vold"]))
        return batch if batch.check_finite() else None

    def step_gradients(self, batch):
        """Forward + loss + backward of train_step (trainer.py:413-443),
        without the optimizer; returns (record-or-None, policy grads, value grads)."""
        c = self.cfg
        logits, cache = policy_forward(self.policy, self.n_actions, batch.obs, batch.tokens)
        lp_new = chosen_logp(logits, batch.tokens)
        l_pi, dlogp, diag = surrogate(lp_new, batch.behavior_logp, batch.advantages,
                                      c.algorithm, c.sigma, c.clip_eps)
        if diag["dropped"]:
            return None, None, None
        h_mean, _ = entropy(logits)
        dlogits = loss_dlogits(logits, batch.tokens, dlogp, c.lambda_h)
        g_pol = policy_backward(self.policy, cache, dlogits)
        hs = np.stack([cache["h1"], cache["h2"]], axis=1)
        v, vcache = value_forward(self.value, self.n_steps, hs, batch.steps)
        err = v - batch.value_targets
        if c.value_clip is not None:
            l_v, gv = value_loss_clipped(v, batch.value_targets, batch.old_values, c.value_clip)
            g_val = value_backward(self.value, vcache, c.lambda_v * gv / err.size)
        else:
            l_v = float(np.mean(err ** 2))
            g_val = value_backward(self.value, vcache, c.lambda_v * 2.0 * err / err.size)
        rec = {"loss": l_pi + c.lambda_v * l_v - c.lambda_h * h_mean,
               "policy_loss": l_pi, "value_loss": l_v, "entropy": h_mean,
               **{k: val for k, val in diag.items() if k != "dropped"}}
        return rec, g_pol, g_val

    def train_step(self, batch):
        """trainer.py:407-467 (publication reduced to the version counter)."""
        rec, g_pol, g_val = self.step_gradients(batch)
        if rec is None:
            self.skipped += 1
            return None
        self.policy, self.adam_policy = adam(self.policy, g_pol, self.adam_policy)
        self.value, self.adam_value = adam(self.value, g_val, self.adam_value)
        self.policy_version += 1
        self.value_version += 1
        self.cycles += 1
        self.publish_version += 1
        rec.update(version=self.publish_version, critic_version=batch.critic_version,
                   behavior_lag=batch.behavior_lag_mean, n_real=batch.n_real,
                   n_imagined=batch.n_imagined)
        return rec
