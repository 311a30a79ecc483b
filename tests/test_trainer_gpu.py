"""GPU drop-in Trainer vs the reference (golden fixtures) and the float64 oracle.

Tolerances (north star): token indexing / segmentation / masks bit-exact;
advantages and value targets within 1e-5 (scaled relative); losses within
1e-4 (scaled); gradients within 1e-4 relative to each tensor's max |g|.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import scaled_err
from golden_io import CASES, Golden
from oracle.trainer_ref import OracleBatch, OracleConfig, OracleTrainer

pytestmark = pytest.mark.gpu

LOSS_TOL = 1e-4
ADV_TOL = 1e-5
GRAD_TOL = 1e-4


def grad_err(x, y, floor: float = 0.0) -> float:
    """max |x - y| relative to the tensor's max |y|; `floor` (1e-3 of the
    model-wide gradient scale) keeps analytically-zero gradients such as
    b_attn (softmax shift invariance: pure round-off in both) comparable."""
    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
    scale = max(float(np.max(np.abs(y))), floor, 1e-30)
    return float(np.max(np.abs(x - y))) / scale


def check_grads(dev_pol, dev_val, g_pol, g_val, tag=""):
    gscale = max(float(np.max(np.abs(v))) for d in (g_pol, g_val) for v in d.values())
    for mine, want in ((dev_pol, g_pol), (dev_val, g_val)):
        for k in want:
            e = grad_err(mine[k], want[k], 1e-3 * gscale)
            assert e < GRAD_TOL, (tag, k, e)


def make_bundle(policy: dict, value: dict, meta: dict):
    from paper_2603_18464_b200.types import (ModelBundle, ParamSet, PolicyConfig, PolicyModel,
                                             ValueConfig, ValueHead)
    pc = PolicyConfig(obs_dim=meta["o"], hidden_dim=meta["d"], chunk_len=meta["k"],
                      n_actions=meta["a"], vocab_size=meta["a"] + 1, action_start=0)
    vc = ValueConfig(hidden_dim=meta["d"], n_steps=meta["n_steps"], mlp_hidden=meta["mlp_hidden"])
    return ModelBundle(PolicyModel(pc, ParamSet(dict(policy))), ValueHead(vc, ParamSet(dict(value))))


def trainer_cfg(c: dict):
    from paper_2603_18464_b200.trainer import GaeConfig, LossConfig, TrainerConfig
    return TrainerConfig(gae=GaeConfig(c["gamma"], c["lam"]),
                         loss=LossConfig(algorithm=c["algorithm"], sigma=c["sigma"],
                                         clip_eps=c["clip_eps"], lambda_v=c["lambda_v"],
                                         lambda_h=c["lambda_h"]),
                         lr=c["lr"], k_shards=c["k_shards"], revalue=c["revalue"])


def oracle_for(g: Golden, policy=None, value=None):
    c = g.cfg
    cfg = OracleConfig(gamma=c["gamma"], lam=c["lam"], algorithm=c["algorithm"], sigma=c["sigma"],
                       clip_eps=c["clip_eps"], lambda_v=c["lambda_v"], lambda_h=c["lambda_h"],
                       lr=c["lr"], k_shards=c["k_shards"], revalue=c["revalue"])
    return OracleTrainer(policy or g.init_policy(), value or g.init_value(), g.meta["a"],
                         g.meta["n_steps"], cfg)


def oracle_batch(g: Golden, s: int) -> OracleBatch:
    b, m = g.batch(s), g.batch_meta(s)
    return OracleBatch(obs=b["obs"], steps=b["steps"], tokens=b["tokens"],
                       behavior_logp=b["behavior_logp"], advantages=b["advantages"],
                       value_targets=b["value_targets"], critic_version=m["critic_version"],
                       n_real=m["n_real"], n_imagined=m["n_imagined"], norm_mean=m["norm_mean"],
                       norm_std=m["norm_std"], norm_count=m["norm_count"],
                       shard_sizes=tuple(m["shard_sizes"]),
                       behavior_lag_mean=m["behavior_lag_mean"])


@pytest.mark.parametrize("name", CASES)
def test_trainer_matches_reference_golden(name):
    from paper_2603_18464_b200.trainer import Trainer

    g = Golden(name)
    tr = Trainer(make_bundle(g.init_policy(), g.init_value(), g.meta), trainer_cfg(g.cfg))
    for s in range(g.meta["steps"]):
        before_pol, before_val = tr.params.to_host()
        batch = tr.build_train_batch(g.trajectories(s))
        assert batch is not None
        ref = g.batch(s)
        np.testing.assert_array_equal(batch.tokens, ref["tokens"])
        np.testing.assert_array_equal(batch.steps, ref["steps"])
        np.testing.assert_allclose(batch.obs, ref["obs"], rtol=1e-6, atol=1e-6)
        assert scaled_err(batch.advantages, ref["advantages"]) < ADV_TOL
        assert scaled_err(batch.value_targets, ref["value_targets"]) < ADV_TOL
        assert scaled_err(batch.behavior_logp, ref["behavior_logp"]) < ADV_TOL
        bm = g.batch_meta(s)
        assert batch.shard_sizes == tuple(bm["shard_sizes"])
        assert batch.norm_count == bm["norm_count"]
        assert batch.n_real == bm["n_real"] and batch.n_imagined == bm["n_imagined"]
        assert batch.behavior_lag_mean == bm["behavior_lag_mean"]
        assert abs(batch.norm_mean - bm["norm_mean"]) <= 1e-5 * max(1.0, abs(bm["norm_mean"]))
        assert abs(batch.norm_std - bm["norm_std"]) <= 1e-5 * max(1.0, bm["norm_std"])

        rec = tr.train_step(batch)
        exp = g.record(s)
        assert set(rec) == set(exp)
        for k, v in exp.items():
            if isinstance(v, int):
                assert rec[k] == v, k
            else:
                assert abs(rec[k] - v) <= LOSS_TOL * max(1.0, abs(v)), (k, rec[k], v)

        # gradients vs the (reference-pinned) oracle on the reference's own batch
        orc = oracle_for(g, before_pol, before_val)
        _, g_pol, g_val = orc.step_gradients(oracle_batch(g, s))
        dev_pol, dev_val = tr.params.grads_to_host()
        check_grads(dev_pol, dev_val, g_pol, g_val, (name, s))

        # parameters after Adam: exact up to float32 storage, except entries
        # whose reference gradient is ~0 (their first Adam step is +-lr by sign)
        after_pol, after_val = tr.params.to_host()
        for which, mine, grads in (("policy", after_pol, g_pol), ("value", after_val, g_val)):
            for k, want in g.after(s, which).items():
                gmax = np.max(np.abs(grads[k])) if grads[k].size else 0.0
                solid = np.abs(grads[k]) > 1e-3 * gmax
                np.testing.assert_allclose(mine[k][solid], want[solid], rtol=0, atol=2e-6,
                                           err_msg=f"{which}.{k}")
                assert np.all(np.abs(mine[k] - want) <= 2 * tr.cfg.lr + 1e-6)
    assert tr.cycles == g.meta["steps"] and tr.publish_version == g.meta["steps"]
    assert tr.bundle.policy.params.version == g.meta["steps"]


def _random_setup(seed=0, n_traj=12, K=7, A=256, D=64, O=195, algo="trust", revalue=True,
                  max_len=40, value_clip=None):
    from paper_2603_18464_b200.trainer import LossConfig, Trainer, TrainerConfig
    from paper_2603_18464_b200.types import (ModelBundle, PolicyConfig, PolicyModel, ValueConfig,
                                             ValueHead)
    from paper_2603_18464_b200.workload import synthetic_trajectories

    rng = np.random.default_rng(seed)
    pc = PolicyConfig(obs_dim=O, hidden_dim=D, chunk_len=K, n_actions=A, vocab_size=A + 8,
                      action_start=4)
    vc = ValueConfig(hidden_dim=D, n_steps=max_len + 2, mlp_hidden=32)
    bundle = ModelBundle(PolicyModel.init(rng, pc), ValueHead.init(rng, vc))
    lens = rng.integers(1, max_len + 1, size=n_traj)
    trajs = synthetic_trajectories(rng, lens, rng.random(n_traj) < 0.5, K, A, O)
    cfg = TrainerConfig(loss=LossConfig(algorithm=algo, value_clip=value_clip), revalue=revalue)
    pol0 = {k: v.copy() for k, v in bundle.policy.params.tensors.items()}
    val0 = {k: v.copy() for k, v in bundle.value.params.tensors.items()}
    return Trainer(bundle, cfg), trajs, pol0, val0, cfg


def _oracle_from(cfg, pol0, val0, A, S):
    oc = OracleConfig(gamma=cfg.gae.gamma, lam=cfg.gae.lam, algorithm=cfg.loss.algorithm,
                      sigma=cfg.loss.sigma, clip_eps=cfg.loss.clip_eps, lambda_v=cfg.loss.lambda_v,
                      lambda_h=cfg.loss.lambda_h, lr=cfg.lr, k_shards=cfg.k_shards,
                      revalue=cfg.revalue, value_clip=cfg.loss.value_clip)
    return OracleTrainer(pol0, val0, A, S, oc)


@pytest.mark.parametrize("algo", ["trust", "clip"])
@pytest.mark.parametrize("factorized", [True, False, "recompute"])
def test_random_batch_matches_oracle(algo, factorized):
    tr, trajs, pol0, val0, cfg = _random_setup(seed=3, algo=algo)
    tr.factorized = bool(factorized)
    tr.recompute_dz = factorized == "recompute"  # dz rebuilt from token scalars
    orc = _oracle_from(cfg, pol0, val0, 256, tr.dims.n_steps)
    ob = orc.build_train_batch(trajs)
    batch = tr.build_train_batch(trajs)
    assert scaled_err(batch.advantages, ob.advantages) < ADV_TOL
    rec = tr.train_step(batch)
    orec, g_pol, g_val = orc.step_gradients(ob)
    for k, v in orec.items():
        assert abs(rec[k] - v) <= LOSS_TOL * max(1.0, abs(v)), (k, rec[k], v)
    dev_pol, dev_val = tr.params.grads_to_host()
    check_grads(dev_pol, dev_val, g_pol, g_val, algo)


@pytest.mark.parametrize("K,A", [(3, 128), (8, 256), (1, 256), (9, 256), (7, 512)])
def test_loss_kernel_shapes_match_oracle(K, A):
    """Two-phase loss kernel (K <= 8, A in {128, 256}) and the grouped kernel
    beyond it (K = 9, A = 512) against the float64 oracle."""
    tr, trajs, pol0, val0, cfg = _random_setup(seed=11, K=K, A=A, n_traj=10, max_len=30)
    orc = _oracle_from(cfg, pol0, val0, A, tr.dims.n_steps)
    ob = orc.build_train_batch(trajs)
    rec = tr.train_step(tr.build_train_batch(trajs))
    orec, g_pol, g_val = orc.step_gradients(ob)
    for k, v in orec.items():
        assert abs(rec[k] - v) <= LOSS_TOL * max(1.0, abs(v)), (k, rec[k], v)
    dev_pol, dev_val = tr.params.grads_to_host()
    check_grads(dev_pol, dev_val, g_pol, g_val, (K, A))


@pytest.mark.parametrize("algo", ["trust", "clip"])
def test_frame_blocked_recompute_matches_oracle(algo):
    """dz-free grouped sums over several frame blocks (one 4096-token chunk per
    block): the loss kernel writes token scalars, the grouped pass recomputes dz
    block by block and folds the blocks in order."""
    tr, trajs, pol0, val0, cfg = _random_setup(seed=13, algo=algo, n_traj=40, max_len=90)
    tr.recompute_dz = True
    tr.group_block_chunks = 1
    orc = _oracle_from(cfg, pol0, val0, 256, tr.dims.n_steps)
    ob = orc.build_train_batch(trajs)
    batch = tr.build_train_batch(trajs)
    assert batch.n_tokens > 3 * 4096  # several blocks
    rec = tr.train_step(batch)
    assert batch.pk_group.nblocks > 2
    orec, g_pol, g_val = orc.step_gradients(ob)
    for k, v in orec.items():
        assert abs(rec[k] - v) <= LOSS_TOL * max(1.0, abs(v)), (k, rec[k], v)
    dev_pol, dev_val = tr.params.grads_to_host()
    check_grads(dev_pol, dev_val, g_pol, g_val, ("blocked", algo))


@pytest.mark.parametrize("factorized", [True, False, "recompute"])
def test_partial_exclusion_runs_fixup_pass(factorized):
    """Some tokens with log-ratio < -745 are excluded: the surrogate mean is
    over the included count (trainer.py:211), entropy still over all tokens."""
    from paper_2603_18464_b200.batch import DeviceTrainBatch

    tr, trajs, pol0, val0, cfg = _random_setup(seed=5)
    tr.factorized = bool(factorized)
    tr.recompute_dz = factorized == "recompute"
    orc = _oracle_from(cfg, pol0, val0, 256, tr.dims.n_steps)
    ob = orc.build_train_batch(trajs)
    poisoned = ob.behavior_logp.copy()
    poisoned.ravel()[::17] = 2000.0  # exp(lp_new - 2000) == 0 -> excluded
    ob.behavior_logp = poisoned
    rec = tr.train_step(ob)  # host TrainBatch path
    orec, g_pol, g_val = orc.step_gradients(ob)
    assert rec["excluded_tokens"] == orec["excluded_tokens"] > 0
    for k, v in orec.items():
        assert abs(rec[k] - v) <= LOSS_TOL * max(1.0, abs(v)), (k, rec[k], v)
    dev_pol, dev_val = tr.params.grads_to_host()
    check_grads(dev_pol, dev_val, g_pol, g_val, "fixup")
    assert isinstance(DeviceTrainBatch.from_host(ob, tr.device), DeviceTrainBatch)


def test_all_excluded_batch_is_skipped():
    tr, trajs, *_ = _random_setup(seed=6)
    batch = tr.build_train_batch(trajs)
    before = tr.params.p[tr.params.cur].clone()
    batch.lp_old.fill_(2000.0)
    assert tr.train_step(batch) is None
    assert tr.skipped == 1 and tr.cycles == 0 and tr.publish_version == 0
    assert bool((tr.params.p[tr.params.cur] == before).all())


def test_train_step_is_bitwise_deterministic():
    """Parameters (reference test_trainer.py:572-583) and the records: the loss
    kernel's statistics go to fixed per-chunk rows under its dynamic schedule."""
    outs, recs = [], []
    for _ in range(2):
        tr, trajs, *_ = _random_setup(seed=9, n_traj=40, max_len=90)
        rr = []
        for _ in range(2):
            rr.append(tr.train_step(tr.build_train_batch(trajs)))
        outs.append(tr.params.p[tr.params.cur].cpu().numpy())
        recs.append(rr)
    np.testing.assert_array_equal(outs[0], outs[1])
    assert recs[0] == recs[1]


def test_build_rejects_nonfinite_and_bad_domains():
    from paper_2603_18464_b200.errors import DimensionError, DomainError
    from paper_2603_18464_b200.types import Trajectory

    tr, trajs, *_ = _random_setup(seed=8, n_traj=3)
    t0 = trajs[0]

    def variant(**kw):
        f = {k: getattr(t0, k) for k in ("task_id", "source", "observations", "steps", "tokens",
                                         "rewards", "behavior_logits", "values",
                                         "bootstrap_value", "done", "behavior_version")}
        f.update(kw)
        return Trajectory(**f)

    r = np.array(t0.rewards)
    r[0] = np.nan
    assert tr.build_train_batch([variant(rewards=r)] + trajs[1:]) is None  # test_trainer.py:540-543
    mu = np.array(t0.behavior_logits)
    mu[0, 0, 0] = np.inf
    with pytest.raises(DomainError):
        tr.build_train_batch([variant(behavior_logits=mu)])
    steps = np.array(t0.steps) + 10_000
    with pytest.raises(DimensionError):
        tr.build_train_batch([variant(steps=steps)])


def test_value_loss_decreases():  # reference test_trainer.py:608-612
    from paper_2603_18464_b200.trainer import TrainerConfig
    tr, trajs, *_ = _random_setup(seed=10, n_traj=4, A=16, D=16, O=20, K=3)
    tr.cfg = TrainerConfig(lr=0.01)
    for st in (tr.adam_policy, tr.adam_value):
        st.lr = 0.01
    batch = tr.build_train_batch(trajs)
    losses = [tr.train_step(batch)["value_loss"] for _ in range(30)]
    assert losses[-1] < losses[0]


def test_publication_versions():
    class PubStub:
        def __init__(self):
            self.configs = {"policy": object()}
            self.published = []

        def update_weights(self, w):
            self.published.append((w.kind, w.version))

    tr, trajs, *_ = _random_setup(seed=11, n_traj=3)
    tr.service = PubStub()
    for v in (1, 2, 3):
        rec = tr.train_step(tr.build_train_batch(trajs))
        assert rec["version"] == v
    assert tr.service.published == [("policy", 1), ("policy", 2), ("policy", 3)]


@pytest.mark.parametrize("D,O", [(512, 320), (4096, 4096)])
def test_wide_layers_match_oracle(D, O):
    """cfg4-style widths (O = D = 4096): products wider than the
    tensor-core row kernel's resident weight fall back to cuBLAS fp32; the step
    still matches the float64 oracle."""
    tr, trajs, pol0, val0, cfg = _random_setup(seed=11, n_traj=4, K=7, A=256, D=D, O=O,
                                               max_len=12)
    orc = _oracle_from(cfg, pol0, val0, 256, tr.dims.n_steps)
    ob = orc.build_train_batch(trajs)
    batch = tr.build_train_batch(trajs)
    assert scaled_err(batch.advantages, ob.advantages) < ADV_TOL
    rec = tr.train_step(batch)
    orec, g_pol, g_val = orc.step_gradients(ob)
    for k, v in orec.items():
        assert abs(rec[k] - v) <= LOSS_TOL * max(1.0, abs(v)), (k, rec[k], v)
    dev_pol, dev_val = tr.params.grads_to_host()
    check_grads(dev_pol, dev_val, g_pol, g_val, "trust")


@pytest.mark.parametrize("revalue", [True, False])
def test_value_clip_loss_matches_oracle(revalue):
    """North-star value-clip loss (opt-in; the reference trains plain MSE): the
    clipped objective and its gradient against the float64 restatement."""
    tr, trajs, pol0, val0, cfg = _random_setup(seed=13, revalue=revalue, value_clip=0.2)
    orc = _oracle_from(cfg, pol0, val0, 256, tr.dims.n_steps)
    ob = orc.build_train_batch(trajs)
    batch = tr.build_train_batch(trajs)
    rec = tr.train_step(batch)
    orec, g_pol, g_val = orc.step_gradients(ob)
    for k, v in orec.items():
        assert abs(rec[k] - v) <= LOSS_TOL * max(1.0, abs(v)), (k, rec[k], v)
    dev_pol, dev_val = tr.params.grads_to_host()
    check_grads(dev_pol, dev_val, g_pol, g_val, "trust")
    # the clip is active for some transitions (else this tests plain MSE)
    import numpy as np
    from oracle.trainer_ref import value_loss_clipped
    l_clip, _ = value_loss_clipped(np.zeros(1), np.ones(1), np.full(1, 0.5), 0.2)
    assert l_clip == 1.0
