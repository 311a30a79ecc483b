"""GPU batched serving (inference.run_batch, inference.py:129-160) against the
reference's own responses (tests/golden/make_golden_serve.py): tokens
bit-exact, logits / values / next observations / probabilities to 1e-12
(float64 on the device); batched == solo (reference test_inference.py:148-159);
empty / mixed batches and out-of-range steps raise like the reference."""

from __future__ import annotations

import numpy as np
import pytest

from serve_fixture import ServeGolden

pytestmark = pytest.mark.gpu


def weights(g: ServeGolden, kind: str):
    from paper_2603_18464_b200.publish import VersionedWeights
    from paper_2603_18464_b200.types import (ObsModel, ObsModelConfig, ParamSet, PolicyConfig,
                                             PolicyModel, RewardModel, ValueConfig, ValueHead)
    m = g.meta
    pc = PolicyConfig(obs_dim=m["O"], hidden_dim=m["D"], chunk_len=m["K"], n_actions=m["A"],
                      vocab_size=m["vocab"], action_start=m["action_start"])
    pol = PolicyModel(pc, ParamSet(g.params("pol_")))
    val = ValueHead(ValueConfig(m["D"], m["n_steps"], m["mlp_hidden"]), ParamSet(g.params("val_")))
    obs = ObsModel(ObsModelConfig(obs_dim=m["O"], chunk_len=m["K"], n_actions=m["A"],
                                  hidden_dim=m["obs_hidden"]), ParamSet(g.params("obs_")))
    rew = RewardModel(m["O"], ParamSet(g.params("rew_")), hidden_dim=m["reward_hidden"])
    return VersionedWeights(kind, m["version"], policy=pol, value=val, obs_model=obs,
                            reward_model=rew)


def test_serve_matches_reference_run_batch():
    from paper_2603_18464_b200.publish import OBS_MODEL, POLICY, REWARD_MODEL
    from paper_2603_18464_b200.serve import DeviceServer
    g = ServeGolden()
    z, seed = g.z, g.meta["base_seed"]
    srv = DeviceServer()
    res = srv.run_batch(weights(g, POLICY), g.requests(POLICY), seed)
    np.testing.assert_array_equal(np.stack([r.tokens for r in res]), z["tokens"])
    np.testing.assert_allclose(np.stack([r.logits for r in res]), z["logits"], rtol=0, atol=1e-12)
    np.testing.assert_allclose([r.value for r in res], z["values"], rtol=0, atol=1e-12)
    assert all(r.version == g.meta["version"] for r in res)
    res = srv.run_batch(weights(g, OBS_MODEL), g.requests(OBS_MODEL), seed)
    np.testing.assert_allclose(np.stack([r.next_obs for r in res]), z["next_obs"], rtol=0,
                               atol=1e-12)
    res = srv.run_batch(weights(g, REWARD_MODEL), g.requests(REWARD_MODEL), seed)
    np.testing.assert_allclose([r.probability for r in res], z["probs"], rtol=0, atol=1e-12)


def test_batched_equals_solo():
    from paper_2603_18464_b200.publish import POLICY
    from paper_2603_18464_b200.serve import DeviceServer
    g = ServeGolden()
    srv = DeviceServer()
    w = weights(g, POLICY)
    reqs = g.requests(POLICY)[:8]
    together = srv.run_batch(w, reqs, 0)
    for req, batched in zip(reqs, together):
        solo = srv.run_batch(w, [req], 0)[0]
        np.testing.assert_array_equal(batched.tokens, solo.tokens)
        np.testing.assert_array_equal(batched.logits, solo.logits)
        assert batched.value == solo.value


def test_serve_errors():
    from paper_2603_18464_b200.errors import DimensionError, PayloadError
    from paper_2603_18464_b200.publish import POLICY, REWARD_MODEL
    from paper_2603_18464_b200.serve import DeviceServer
    g = ServeGolden()
    srv = DeviceServer()
    w = weights(g, POLICY)
    with pytest.raises(PayloadError):
        srv.run_batch(w, [], 0)
    mixed = g.requests(POLICY)[:1] + g.requests(REWARD_MODEL)[:1]
    with pytest.raises(PayloadError):
        srv.run_batch(w, mixed, 0)
    bad = g.requests(POLICY)[:2]
    bad[1].obs.step = g.meta["n_steps"]
    with pytest.raises(DimensionError, match="step index"):
        srv.run_batch(w, bad, 0)


def test_device_snapshot_serves_without_host_round_trip():
    """SURVEY 8(f) rows 1+2: a trainer's device snapshot (Trainer.snapshot) is
    served straight from its flat fp32 buffer -- the snapshot's host models are
    never materialized -- with responses identical to serving the same weights
    through host model objects."""
    from paper_2603_18464_b200.publish import POLICY, VersionedWeights
    from paper_2603_18464_b200.serve import DeviceServer
    from paper_2603_18464_b200.trainer import Trainer, TrainerConfig
    from paper_2603_18464_b200.types import (ModelBundle, PolicyConfig, PolicyModel, ValueConfig,
                                             ValueHead)
    from paper_2603_18464_b200.workload import synthetic_trajectories
    g = ServeGolden()
    m = g.meta
    rng = np.random.default_rng(3)
    pc = PolicyConfig(obs_dim=m["O"], hidden_dim=m["D"], chunk_len=m["K"], n_actions=m["A"],
                      vocab_size=m["vocab"], action_start=m["action_start"])
    bundle = ModelBundle(PolicyModel.init(rng, pc),
                         ValueHead.init(rng, ValueConfig(m["D"], m["n_steps"], m["mlp_hidden"])))
    tr = Trainer(bundle, TrainerConfig())
    trajs = synthetic_trajectories(rng, [5, 9, 3], [True, False, True], m["K"], m["A"], m["O"],
                                   n_steps=m["n_steps"])
    tr.train_step(tr.build_train_batch(trajs))  # the snapshot is of trained parameters
    snap = tr.snapshot()
    reqs = g.requests(POLICY)
    got = DeviceServer().run_batch(snap, reqs, m["base_seed"])
    assert snap._policy is None and snap._value is None  # no host materialization
    host_w = VersionedWeights(POLICY, snap.version, policy=tr.bundle.policy, value=tr.bundle.value)
    want = DeviceServer().run_batch(host_w, reqs, m["base_seed"])
    np.testing.assert_array_equal(np.stack([r.tokens for r in got]),
                                  np.stack([r.tokens for r in want]))
    np.testing.assert_array_equal(np.stack([r.logits for r in got]),
                                  np.stack([r.logits for r in want]))
    np.testing.assert_array_equal([r.value for r in got], [r.value for r in want])


def test_device_ticket_uniforms_equal_the_host_draws():
    """The serving kernel's per-ticket uniforms == numpy's SeedSequence draws."""
    import torch

    from paper_2603_18464_b200.serve import _device_ticket_uniforms, ticket_uniforms
    tickets = [0, 5, 2 ** 32, 2 ** 40 + 3] + list(range(1000, 5096))
    for base in (3, 2 ** 33 + 1):
        got = _device_ticket_uniforms(base, tickets, 4, torch.device("cuda")).cpu().numpy()
        np.testing.assert_array_equal(got, ticket_uniforms(base, tickets, 4))
    # integers past the kernel's range take the host path, same values
    big = _device_ticket_uniforms(2 ** 70, [1, 2], 3, torch.device("cuda")).cpu().numpy()
    np.testing.assert_array_equal(big, ticket_uniforms(2 ** 70, [1, 2], 3))
