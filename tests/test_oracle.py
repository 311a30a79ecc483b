"""Pin the float64 oracle (CPU) against the reference's golden outputs and the
reference tests' own known-answer values (tests/test_trainer.py,
tests/test_numerics.py of the reference; cited per test)."""

from __future__ import annotations

import numpy as np
import pytest

from golden_io import CASES, Golden
from oracle import c_oracle
from oracle.trainer_ref import (OracleConfig, OracleDomainError, OracleTrainer, adam,
                                AdamSlots, entropy, gae, pooled_normalize, surrogate,
                                trust_weight)


# -- known-answer values from the reference test-suite --------------------------------


def test_gae_worked_example():  # reference tests/test_trainer.py:67-75
    adv, ret = gae([1.0, 0.0], [0.5, 0.25, 0.4], True, 0.9, 0.95)
    np.testing.assert_allclose(adv, [0.51125, -0.25], atol=1e-12)
    np.testing.assert_allclose(ret, [1.01125, 0.0], atol=1e-12)


def test_gae_terminal_and_truncation():  # :78-87
    np.testing.assert_allclose(gae([1.0], [0.0, 7.0], True, 0.9, 0.95)[0], [1.0])
    adv, ret = gae([0.0], [0.0, 1.0], False, 0.5, 0.9)
    np.testing.assert_allclose(adv, [0.5])
    np.testing.assert_allclose(ret, [0.5])


def test_gae_double_sum(rng):  # :35-64 (independent O(T^2) oracle)
    for _ in range(200):
        T = int(rng.integers(1, 21))
        r, v = rng.normal(size=T), rng.normal(size=T + 1)
        done = bool(rng.integers(0, 2))
        g, lam = float(rng.uniform(0.5, 1.0)), float(rng.uniform(0.0, 1.0))
        vv = v.copy()
        if done:
            vv[-1] = 0.0
        delta = r + g * vv[1:] - vv[:-1]
        ref = np.array([sum((g * lam) ** l * delta[t + l] for l in range(T - t))
                        for t in range(T)])
        np.testing.assert_allclose(gae(r, v, done, g, lam)[0], ref, atol=1e-10)


def test_gae_c_restatement_matches_python(rng):
    lens = rng.integers(1, 30, size=40)
    off = np.concatenate([[0], np.cumsum(lens)])
    r = rng.normal(size=off[-1])
    v = rng.normal(size=off[-1] + 40)
    d = (rng.random(40) < 0.5).astype(np.uint8)
    adv, ret = c_oracle.gae_csr(r, v, off, d, 0.97, 0.9)
    for s in range(40):
        a, b = off[s], off[s + 1]
        ea, er = gae(r[a:b], v[a + s:b + s + 1], bool(d[s]), 0.97, 0.9)
        np.testing.assert_allclose(adv[a:b], ea, atol=1e-13)
        np.testing.assert_allclose(ret[a:b], er, atol=1e-13)


def test_gae_validation():  # :98-106
    with pytest.raises(OracleDomainError):
        gae([1.0], [0.0], False, 0.9, 0.9)
    with pytest.raises(OracleDomainError):
        gae([], [0.0], False, 0.9, 0.9)


def test_pooled_worked_example():  # :136-144
    out, s = pooled_normalize([np.array([1.0, 2.0, 3.0]), np.array([4.0, 5.0])])
    assert s["mean"] == pytest.approx(3.0) and s["std"] == pytest.approx(np.sqrt(2.0))
    assert s["shard_sizes"] == (3, 2)
    assert out[0][0] == pytest.approx(-2.0 / np.sqrt(2.0), abs=1e-6)


def test_pooled_shard_invariance(rng):  # :112-125
    x = rng.normal(loc=1.0, scale=3.0, size=200)
    base = np.concatenate(pooled_normalize(np.array_split(x, 1))[0])
    for k in (2, 4, 8):
        np.testing.assert_allclose(np.concatenate(pooled_normalize(np.array_split(x, k))[0]),
                                   base, atol=1e-10)


def test_pooled_empty():  # :154-173
    with pytest.raises(OracleDomainError):
        pooled_normalize([np.array([])])
    out, s = pooled_normalize([np.array([1.0, 3.0]), np.array([])])
    assert s["shard_sizes"] == (2, 0) and out[1].size == 0


def test_trust_weight_values():  # :179-185
    assert trust_weight(1.0, 0.3) == 1.0
    assert trust_weight(2.0, 0.3) == pytest.approx(0.06930879903414185, abs=1e-15)
    assert trust_weight(float(np.exp(0.3)), 0.3) == pytest.approx(np.exp(-0.5), abs=1e-12)


def test_surrogate_known_answers():
    lp = np.log(np.full((2, 2), 0.25))  # :246-257 on-policy collapse
    for algo in ("trust", "clip"):
        loss, g, diag = surrogate(lp, lp.copy(), np.array([1.0, -2.0]), algo)
        assert loss == pytest.approx(0.5)
        np.testing.assert_allclose(g, -np.array([[1.0, 1.0], [-2.0, -2.0]]) / 4.0)
    loss, g, _ = surrogate(np.array([[np.log(2.0)]]), np.array([[0.0]]), np.array([1.5]))
    assert loss == pytest.approx(-0.20792639710242555, abs=1e-15)  # :260-267
    r = np.array([[0.9, 1.5], [0.7, 1.1]])  # clip example :290-304
    loss, g, diag = surrogate(np.log(r), np.zeros((2, 2)), np.array([1.0, -2.0]), "clip")
    assert loss == pytest.approx(0.425, abs=1e-12)
    np.testing.assert_allclose(g, -np.array([[0.9, 0.0], [0.0, -2.2]]) / 4.0, atol=1e-12)
    assert diag["clipped_fraction"] == pytest.approx(0.5)
    # degenerate ratios excluded (:270-278), all excluded drops (:281-287)
    _, g, diag = surrogate(np.array([[0.0, 1000.0], [-1000.0, 0.1]]), np.zeros((2, 2)),
                           np.ones(2))
    assert diag["excluded_tokens"] == 2 and g[0, 1] == 0 and g[1, 0] == 0
    loss, g, diag = surrogate(np.full((2, 2), -2000.0), np.zeros((2, 2)), np.ones(2))
    assert diag["dropped"] and loss == 0.0


def test_entropy_uniform():  # :362-376
    h, d = entropy(np.zeros((2, 2, 7)))
    assert h == pytest.approx(np.log(7.0), abs=1e-12)
    np.testing.assert_allclose(d, 0.0, atol=1e-12)


def test_adam_three_steps():  # reference tests/test_numerics.py:57-69
    p = {"w": np.array([1.0])}
    st = AdamSlots.zeros(p, lr=0.1)
    ws = []
    for grad in (0.5, -0.25, 0.1):
        p, st = adam(p, {"w": np.array([grad])}, st)
        ws.append(float(p["w"][0]))
    np.testing.assert_allclose(ws, [0.900000002, 0.8733662987078463, 0.8418419430257161],
                               rtol=0, atol=1e-15)
    assert st.step == 3


# -- golden fixtures from the real reference Trainer ---------------------------------------


def oracle_trainer(g: Golden) -> OracleTrainer:
    c = g.cfg
    cfg = OracleConfig(gamma=c["gamma"], lam=c["lam"], algorithm=c["algorithm"],
                       sigma=c["sigma"], clip_eps=c["clip_eps"], lambda_v=c["lambda_v"],
                       lambda_h=c["lambda_h"], lr=c["lr"], k_shards=c["k_shards"],
                       revalue=c["revalue"])
    return OracleTrainer(g.init_policy(), g.init_value(), g.meta["a"], g.meta["n_steps"], cfg)


@pytest.mark.parametrize("name", CASES)
def test_oracle_reproduces_reference_trainer(name):
    g = Golden(name)
    tr = oracle_trainer(g)
    for s in range(g.meta["steps"]):
        batch = tr.build_train_batch(g.trajectories(s))
        ref = g.batch(s)
        for f in ("obs", "steps", "tokens", "behavior_logp", "advantages", "value_targets"):
            np.testing.assert_allclose(getattr(batch, f), ref[f], rtol=0, atol=1e-11, err_msg=f)
        bm = g.batch_meta(s)
        assert batch.shard_sizes == tuple(bm["shard_sizes"])
        assert batch.norm_count == bm["norm_count"]
        assert batch.behavior_lag_mean == bm["behavior_lag_mean"]
        rec = tr.train_step(batch)
        exp = g.record(s)
        assert set(rec) == set(exp)
        for k, v in exp.items():
            assert rec[k] == pytest.approx(v, rel=1e-9, abs=1e-12), k
        for which, mine in (("policy", tr.policy), ("value", tr.value)):
            for k, v in g.after(s, which).items():
                np.testing.assert_allclose(mine[k], v, rtol=0, atol=1e-11, err_msg=f"{which}.{k}")


def test_value_clip_restatement_known_answers():
    """PPO value clipping (north-star option; the reference is plain MSE)."""
    from oracle.trainer_ref import value_loss_clipped
    v = np.array([1.0, 0.0, 0.5, 2.0])
    ret = np.array([0.0, 1.0, 0.5, 1.0])
    old = np.array([0.9, 0.5, 0.0, 1.0])
    loss, g = value_loss_clipped(v, ret, old, 0.2)
    # row 0: |d|=0.1 <= eps, vc = v -> both branches (1.0)^2, grad 2(v - R) = 2
    # row 1: d=-0.5, vc = 0.3 -> max(1.0, 0.49) = 1.0 from the unclipped branch
    # row 2: d=0.5, vc=0.2 -> max(0, 0.09) = 0.09 clipped, |d| > eps -> grad 0
    # row 3: d=1.0, vc=1.2 -> max(1.0, 0.04) = 1.0 unclipped, grad 2
    np.testing.assert_allclose(loss, (1.0 + 1.0 + 0.09 + 1.0) / 4)
    np.testing.assert_allclose(g, [2.0, -2.0, 0.0, 2.0])
