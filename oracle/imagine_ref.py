"""Float64 restatement of the imagination step (TEST INFRASTRUCTURE).

Follows `RolloutWorker.imagine_episode` (rollout.py:295-362) with the
per-request model evaluations of `inference.run_batch` (inference.py:146-159):
`PolicyModel.sample_chunk` (models.py:135-150), `state_value`
(models.py:406-408), `ObsModel.predict` (models.py:349-355),
`GridTaskSuite.snap_observation` (env.py:259-283) and `RewardModel.predict`
(models.py:375-377).  Randomness is injected: `uniforms[r]` holds the K
draws of the r-th policy request (the tail request included).
"""

from __future__ import annotations

import numpy as np

from .trainer_ref import softmax


def _backbone(p, x):
    h1 = np.tanh(p["w0"] @ x + p["b0"])
    h2 = np.tanh(p["w1"] @ h1 + p["b1"])
    return h1, h2


def sample_chunk(p, n_actions, x, u):
    """models.py:135-150 with rng.random() -> u[k]."""
    _, h2 = _backbone(p, x)
    k_len = p["e_pos"].shape[0]
    tokens = np.zeros(k_len, dtype=np.int64)
    logits = np.zeros((k_len, n_actions))
    prev = n_actions
    for k in range(k_len):
        lg = p["w_head"] @ (h2 + p["e_prev"][prev] + p["e_pos"][k]) + p["b_head"]
        logits[k] = lg
        tok = int(np.searchsorted(np.cumsum(softmax(lg)), u[k]))
        tokens[k] = min(tok, n_actions - 1)
        prev = int(tokens[k])
    return tokens, logits


def state_value(p, vp, x, step):
    """models.py:406-408 -> ValueHead.forward_batch on one row (:273-290)."""
    hs = np.stack(_backbone(p, x))
    e = hs @ vp["w_attn"] + vp["b_attn"][0]
    a = softmax(e)
    u = a @ hs + vp["e_step"][step]
    m = np.tanh(vp["w0v"] @ u + vp["b0v"])
    return float((vp["w1v"] @ m + vp["b1v"])[0])


def mlp(params, x):
    h = np.tanh(params["w0"] @ x + params["b0"])
    return params["w1"] @ h + params["b1"]


def obs_predict(op, n_actions, x, tokens):
    """models.py:349-355: input [obs, one-hot(chunk)]."""
    oh = np.zeros((len(tokens), n_actions))
    oh[np.arange(len(tokens)), tokens] = 1.0
    return mlp(op, np.concatenate([x, oh.ravel()]))


def reward_predict(rp, x):
    """models.py:375-377."""
    return float(1.0 / (1.0 + np.exp(-mlp(rp, x)[0])))


def snap(vec, height, width, n_kinds=3):
    """env.py:259-283: nearest valid grid encoding, first index wins ties."""
    n_cells = 3 * height * width
    grid = vec[:n_cells].reshape(3, height, width)
    out = np.zeros_like(grid)
    agent = np.unravel_index(int(np.argmax(grid[0])), grid[0].shape)
    out[0][agent] = 1.0
    obj_flat = int(np.argmax(grid[1]))
    if grid[1].flat[obj_flat] > 1.5:
        out[1][agent] = 2.0
    else:
        out[1][np.unravel_index(obj_flat, grid[1].shape)] = 1.0
    out[2][np.unravel_index(int(np.argmax(grid[2])), grid[2].shape)] = 1.0
    kind = np.zeros(n_kinds)
    kind[int(np.argmax(vec[n_cells:]))] = 1.0
    return np.concatenate([out.ravel(), kind])


def imagine_episode(p, vp, op, rp, n_actions, start_vec, start_step, uniforms, h_img,
                    threshold=0.9, grid=None):
    """rollout.py:295-362.  Returns a dict of trajectory arrays, or
    {"discarded": reason} for a non-finite prediction (:315-331)."""
    x = np.asarray(start_vec, dtype=np.float64)
    step = int(start_step)
    obs, steps = [x], [step]
    tokens, rewards, logits, values = [], [], [], []
    p_cur = reward_predict(rp, x)
    done = False
    r = 0
    for _ in range(h_img):
        tok, lg = sample_chunk(p, n_actions, x, uniforms[r])
        val = state_value(p, vp, x, step)
        r += 1
        nxt = obs_predict(op, n_actions, x, tok)
        if not np.all(np.isfinite(nxt)):
            return {"discarded": "nonfinite_obs"}
        if grid is not None:
            nxt = snap(nxt, *grid)
        p_next = reward_predict(rp, nxt)
        if not np.isfinite(p_next):
            return {"discarded": "nonfinite_reward"}
        tokens.append(tok)
        logits.append(lg)
        values.append(val)
        rewards.append(p_next - p_cur)
        p_cur = p_next
        x, step = nxt, step + 1
        obs.append(x)
        steps.append(step)
        if p_next >= threshold:
            done = True
            break
    boot = state_value(p, vp, x, step)
    return {"observations": np.stack(obs), "steps": np.asarray(steps),
            "tokens": np.stack(tokens), "rewards": np.asarray(rewards),
            "behavior_logits": np.stack(logits), "values": np.asarray(values),
            "bootstrap_value": boot, "done": done, "t_len": len(tokens)}
