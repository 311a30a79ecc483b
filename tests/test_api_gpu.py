"""The drop-in's module-level functions (importable "with the
same semantics") against the reference's own known answers and the oracle.

Reference: trainer.py:79-294 and the known-answer tests in
tests/test_trainer.py:67-95 (GAE), :112-173 (pooled normalization),
:179-207 (trust weight), :226-240 (chunk ratio), :246-314 (surrogate),
:362-365 (entropy), :453-458 (behavior log-probs).  GAE and behavior
log-probs run in the fp32 kernels (north-star tolerance 1e-5 relative);
the scalar functions run float64 on the device and keep the reference's
tolerances.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import scaled_err
from oracle import trainer_ref as ref

pytestmark = pytest.mark.gpu
FP32 = 1e-6  # fp32 kernels on O(1) known answers


def T():
    from paper_2603_18464_b200 import trainer
    return trainer


def test_compute_gae_known_answers():
    t = T()
    adv, targets = t.compute_gae([1.0, 0.0], [0.5, 0.25, 0.4], True, t.GaeConfig(0.9, 0.95))
    np.testing.assert_allclose(adv, [0.51125, -0.25], atol=FP32)
    np.testing.assert_allclose(targets, [1.01125, 0.0], atol=FP32)
    adv, _ = t.compute_gae([1.0], [0.0, 7.0], True, t.GaeConfig(0.9, 0.95))
    np.testing.assert_allclose(adv, [1.0], atol=FP32)  # bootstrap ignored on done
    adv, targets = t.compute_gae([0.0], [0.0, 1.0], False, t.GaeConfig(0.5, 0.9))
    np.testing.assert_allclose(adv, [0.5], atol=FP32)
    np.testing.assert_allclose(targets, [0.5], atol=FP32)
    rng = np.random.default_rng(0)
    r, v = rng.normal(size=6), rng.normal(size=7)
    adv, _ = t.compute_gae(r, v, False, t.GaeConfig(0.9, 0.0))  # lambda 0 -> one-step TD
    np.testing.assert_allclose(adv, r + 0.9 * v[1:] - v[:-1], atol=1e-5)


def test_compute_gae_random_vs_oracle():
    t = T()
    rng = np.random.default_rng(1)
    for _ in range(40):
        n = int(rng.integers(1, 700))
        r, v = rng.normal(size=n), rng.normal(size=n + 1)
        done = bool(rng.random() < 0.5)
        g, lam = float(rng.uniform(0.5, 1.0)), float(rng.uniform(0.0, 1.0))
        adv, ret = t.compute_gae(r, v, done, t.GaeConfig(g, lam))
        ra, rr = ref.gae(r, v, done, g, lam)
        assert scaled_err(adv, ra) < 1e-5 and scaled_err(ret, rr) < 1e-5


def test_compute_gae_validation():
    t = T()
    with pytest.raises(t.DomainError):
        t.compute_gae([1.0], [0.0], False, t.GaeConfig())
    with pytest.raises(t.DomainError):
        t.compute_gae([], [0.0], False, t.GaeConfig())


def test_global_normalize_known_answers():
    t = T()
    out, summ = t.global_normalize([np.array([1.0, 2.0, 3.0]), np.array([4.0, 5.0])])
    assert summ["mean"] == pytest.approx(3.0)
    assert summ["std"] == pytest.approx(np.sqrt(2.0))
    assert summ["n"] == 5 and summ["shard_sizes"] == (3, 2)
    assert out[0][0] == pytest.approx(-2.0 / np.sqrt(2.0), abs=1e-6)
    out, summ = t.global_normalize([np.full(4, 2.5), np.full(2, 2.5)])
    assert summ["std"] == 0.0
    for s in out:
        np.testing.assert_array_equal(s, np.zeros_like(s))
    out, summ = t.global_normalize([np.array([1.0, 3.0]), np.array([])])
    assert summ["shard_sizes"] == (2, 0) and out[1].size == 0
    for bad in ([np.array([])], []):
        with pytest.raises(t.DomainError):
            t.global_normalize(bad)


def test_global_normalize_shard_invariance_and_moments():
    t = T()
    rng = np.random.default_rng(2)
    adv = rng.normal(loc=1.0, scale=3.0, size=257)
    base = None
    for k in (1, 2, 4, 8):
        out, summ = t.global_normalize(np.array_split(adv, k))
        flat = np.concatenate(out)
        assert sum(summ["shard_sizes"]) == adv.size
        want, _ = ref.pooled_normalize(np.array_split(adv, k))
        assert scaled_err(flat, np.concatenate(want)) < 1e-5
        if base is None:
            base = flat
        np.testing.assert_allclose(flat, base, atol=1e-6)
    flat = np.concatenate(t.global_normalize(np.array_split(
        rng.normal(loc=-2.0, scale=5.0, size=400), 4))[0])
    assert abs(flat.mean()) < 1e-6 and abs(flat.std() - 1.0) < 1e-5


def test_shard_statistics_and_validation():
    t = T()
    st = t.shard_statistics([np.array([1.0, 2.0])])
    assert st.s[0] == 3.0 and st.q[0] == 5.0 and st.n[0] == 2.0
    with pytest.raises(t.DomainError, match="N\\*Q < S\\^2"):
        t.ShardStats(s=np.array([5.0]), q=np.array([1.0]), n=np.array([1.0]))
    with pytest.raises(t.DomainError):
        t.ShardStats(s=np.zeros(2), q=np.zeros(3), n=np.zeros(2))


def test_trust_weight_laws():
    t = T()
    assert t.trust_weight(1.0, sigma=0.3) == 1.0
    for sigma in (0.1, 0.3, 1.0):
        assert t.trust_weight(float(np.exp(sigma)), sigma) == pytest.approx(np.exp(-0.5), abs=1e-12)
    assert t.trust_weight(2.0, 0.3) == pytest.approx(0.06930879903414185, abs=1e-15)
    r = np.random.default_rng(3).uniform(0.05, 20.0, size=10_000)
    np.testing.assert_allclose(t.trust_weight(r, 0.3), t.trust_weight(1.0 / r, 0.3), rtol=1e-9)
    w = t.trust_weight(np.exp(np.linspace(0.0, 3.0, 50)), 0.5)
    assert np.all(np.diff(w) < 0) and w[0] == 1.0
    for bad in (0.0, -1.0, np.inf, np.nan):
        with pytest.raises(t.DomainError):
            t.trust_weight(bad, 0.3)
    with pytest.raises(t.DomainError):
        t.trust_weight(np.array([1.0, -2.0]), 0.3)


def test_chunk_ratio():
    t = T()
    assert t.chunk_ratio(np.log([[2.0, 1.0]]), np.log([[1.0, 1.0]]))[0] == pytest.approx(2.0, rel=1e-12)
    assert t.chunk_ratio(np.full((1, 8), np.log(0.9)), np.zeros((1, 8)))[0] == \
        pytest.approx(0.43046721, rel=1e-12)
    rng = np.random.default_rng(4)
    a, b = rng.normal(size=(5, 4)) * 0.1, rng.normal(size=(5, 4)) * 0.1
    np.testing.assert_allclose(t.chunk_ratio(a, b), np.prod(np.exp(a - b), axis=-1), rtol=1e-9)


def test_policy_surrogate_known_answers():
    t = T()
    lp = np.log(np.full((2, 2), 0.25))
    adv = np.array([1.0, -2.0])
    for algo in ("trust", "clip"):
        loss, dlogp, diag = t.policy_surrogate(lp, lp.copy(), adv, t.LossConfig(algorithm=algo))
        assert loss == pytest.approx(0.5)
        np.testing.assert_allclose(dlogp, -np.array([[1.0, 1.0], [-2.0, -2.0]]) / 4.0)
        assert diag["excluded_tokens"] == 0 and diag["ratio_mean"] == pytest.approx(1.0)
    _, _, diag = t.policy_surrogate(lp, lp.copy(), adv, t.LossConfig("trust"))
    assert diag["trust_weight_mean"] == pytest.approx(1.0)
    loss, dlogp, _ = t.policy_surrogate(np.array([[np.log(2.0)]]), np.array([[0.0]]),
                                        np.array([1.5]), t.LossConfig("trust", sigma=0.3))
    assert loss == pytest.approx(-0.20792639710242555, abs=1e-15)
    assert dlogp[0, 0] == pytest.approx(-0.20792639710242555, abs=1e-15)
    # degenerate ratios (overflow to inf, underflow to 0) drop out
    loss, dlogp, diag = t.policy_surrogate(np.array([[0.0, 1000.0], [-1000.0, 0.1]]),
                                           np.zeros((2, 2)), np.array([1.0, 1.0]),
                                           t.LossConfig("trust"))
    assert diag["excluded_tokens"] == 2 and dlogp[0, 1] == 0.0 and dlogp[1, 0] == 0.0
    assert np.isfinite(loss)
    loss, dlogp, diag = t.policy_surrogate(np.full((2, 2), -2000.0), np.zeros((2, 2)),
                                           np.ones(2), t.LossConfig())
    assert diag["dropped"] is True and loss == 0.0
    np.testing.assert_array_equal(dlogp, np.zeros((2, 2)))
    # clip arm worked example
    loss, dlogp, diag = t.policy_surrogate(np.log(np.array([[0.9, 1.5], [0.7, 1.1]])),
                                           np.zeros((2, 2)), np.array([1.0, -2.0]),
                                           t.LossConfig(algorithm="clip", clip_eps=0.2))
    assert loss == pytest.approx(0.425, abs=1e-12)
    np.testing.assert_allclose(dlogp, -np.array([[0.9, 0.0], [0.0, 1.1 * -2.0]]) / 4.0, atol=1e-12)
    assert diag["clipped_fraction"] == pytest.approx(0.5)
    # pinned trust weights reduce to importance sampling
    loss, dlogp, _ = t.policy_surrogate(np.log(np.array([[1.3, 0.6]])), np.zeros((1, 2)),
                                        np.array([2.0]), t.LossConfig("trust"),
                                        trust_weights=np.ones((1, 2)))
    assert loss == pytest.approx(-(1.3 * 2.0 + 0.6 * 2.0) / 2.0)
    np.testing.assert_allclose(dlogp, [[-1.3, -0.6]])


@pytest.mark.parametrize("algo", ["trust", "clip"])
def test_policy_surrogate_random_vs_oracle(algo):
    t = T()
    rng = np.random.default_rng(5)
    lpn, lpo = rng.normal(size=(64, 7)) * 0.3 - 5.5, rng.normal(size=(64, 7)) * 0.3 - 5.5
    adv = rng.normal(size=64)
    loss, dlogp, diag = t.policy_surrogate(lpn, lpo, adv, t.LossConfig(algorithm=algo))
    rl, rd, rdiag = ref.surrogate(lpn, lpo, adv, algo, 0.3, 0.2)
    assert loss == pytest.approx(rl, rel=1e-12, abs=1e-15)
    np.testing.assert_allclose(dlogp, rd, rtol=1e-12, atol=1e-15)
    for k, v in rdiag.items():
        assert diag[k] == pytest.approx(v, rel=1e-12, abs=1e-15), k


def test_entropy_bonus():
    t = T()
    h, dz = t.entropy_bonus(np.zeros((2, 2, 7)))
    assert h == pytest.approx(np.log(7.0), abs=1e-12)
    np.testing.assert_allclose(dz, np.zeros((2, 2, 7)), atol=1e-12)
    z = np.random.default_rng(6).normal(size=(2, 2, 5))
    h, dz = t.entropy_bonus(z)
    rh, rdz = ref.entropy(z)
    assert h < np.log(5.0) and h == pytest.approx(rh, rel=1e-12)
    np.testing.assert_allclose(dz, rdz, rtol=1e-10, atol=1e-15)


def test_total_loss():
    t = T()
    assert t.total_loss(1.0, 2.0, 3.0, t.LossConfig(lambda_v=0.5, lambda_h=0.01)) == \
        pytest.approx(1.0 + 0.5 * 2.0 - 0.01 * 3.0)


def test_behavior_log_probs():
    t = T()
    logits = np.log(np.array([[[1.0, 1.0, 2.0]]]))
    assert t.behavior_log_probs(logits, np.array([[2]]))[0, 0] == pytest.approx(np.log(0.5), abs=FP32)
    assert t.behavior_log_probs(logits, np.array([[0]]))[0, 0] == pytest.approx(np.log(0.25), abs=FP32)
    rng = np.random.default_rng(7)
    for a in (7, 128, 256, 300):
        mu = rng.normal(size=(9, 3, a)) * 2.0
        tok = rng.integers(0, a, size=(9, 3))
        assert scaled_err(t.behavior_log_probs(mu, tok), ref.chosen_logp(mu, tok)) < 1e-5
    with pytest.raises(t.DimensionError):
        t.behavior_log_probs(np.zeros((2, 3, 4)), np.zeros((2, 2), dtype=np.int64))
    with pytest.raises(t.DimensionError):
        t.behavior_log_probs(np.zeros((1, 1, 4)), np.array([[4]]))
    bad = np.zeros((1, 1, 4))
    bad[0, 0, 1] = np.nan
    with pytest.raises(t.DomainError):
        t.behavior_log_probs(bad, np.array([[0]]))


def test_recompute_values_matches_oracle():
    """Trainer.recompute_values (trainer.py:352-356 -> models.py:411-415) over
    all T+1 frames, and its step-index domain check (models.py:261-267)."""
    from paper_2603_18464_b200.trainer import Trainer, TrainerConfig
    from paper_2603_18464_b200.types import (ModelBundle, PolicyConfig, PolicyModel, ValueConfig,
                                             ValueHead)
    from paper_2603_18464_b200.workload import synthetic_trajectories

    rng = np.random.default_rng(8)
    for D, O in ((64, 195), (256, 51)):
        bundle = ModelBundle(PolicyModel.init(rng, PolicyConfig(obs_dim=O, hidden_dim=D,
                                                                chunk_len=7, n_actions=256,
                                                                vocab_size=300, action_start=1)),
                             ValueHead.init(rng, ValueConfig(hidden_dim=D, n_steps=60)))
        tr = Trainer(bundle, TrainerConfig())
        orc = ref.OracleTrainer(bundle.policy.params.tensors, bundle.value.params.tensors, 256, 60)
        for traj in synthetic_trajectories(rng, [1, 17, 55], [True, False, True], 7, 256, O,
                                           n_steps=60):
            v = tr.recompute_values(traj)
            assert v.shape == (traj.t_len + 1,)
            assert scaled_err(v, orc.state_values(traj.observations, traj.steps)) < 1e-5
    bad = synthetic_trajectories(rng, [3], [False], 7, 256, 51, n_steps=60)[0]
    object.__setattr__(bad, "steps", np.asarray(bad.steps) + 1000)
    with pytest.raises(T().DimensionError):
        tr.recompute_values(bad)
