"""GPU world-model training sub-steps (trainer.py:469-535) against fixtures
made by the reference trainer (tests/golden/make_golden_wm.py): losses and
parameters after every obs-model / reward-model sub-step (float64 on the
device: 1e-10), update counters and versions, publication, the run-loop
schedule (reference tests/test_trainer.py:636-770), and the error paths."""

from __future__ import annotations

import numpy as np
import pytest

import fake_runtime as rt
from wm_fixture import WM_CASES, WmGolden

pytestmark = pytest.mark.gpu


def make_trainer(g: WmGolden, **cfg_kw):
    from paper_2603_18464_b200.trainer import Trainer, TrainerConfig
    from paper_2603_18464_b200.types import (ModelBundle, ObsModel, ObsModelConfig, ParamSet,
                                             PolicyConfig, PolicyModel, RewardModel,
                                             ValueConfig, ValueHead)
    m = g.meta
    pc = PolicyConfig(obs_dim=m["o"], hidden_dim=16, chunk_len=m["k"], n_actions=m["a"],
                      vocab_size=m["a"], action_start=0)
    bundle = ModelBundle(
        PolicyModel(pc, ParamSet(g.params("pol_"))),
        ValueHead(ValueConfig(16, 40, 8), ParamSet(g.params("val_"))),
        ObsModel(ObsModelConfig(obs_dim=m["o"], chunk_len=m["k"], n_actions=m["a"],
                                hidden_dim=m["obs_hidden"]), ParamSet(g.params("obs0_"))),
        RewardModel(m["o"], ParamSet(g.params("rew0_")), hidden_dim=m["reward_hidden"]))
    cfg = TrainerConfig(lr=m["lr"], wm_max_transitions=m["max_rows"],
                        reward_neg_ratio=m["neg_ratio"], k_shards=1, **cfg_kw)
    return Trainer(bundle, cfg, seed=m["seed"], **({}))


@pytest.mark.parametrize("name", WM_CASES)
def test_wm_substeps_match_reference(name):
    g = WmGolden(name)
    m = g.meta
    tr = make_trainer(g)
    trajs = g.trajectories()
    for s, kind in enumerate(m["seq"]):
        loss = (tr.train_obs_model_step if kind == "obs" else tr.train_reward_model_step)(trajs)
        want = m["losses"][s]
        assert abs(loss - want) <= 1e-10 * max(1.0, abs(want)), (s, kind, loss, want)
        model = tr.bundle.obs_model if kind == "obs" else tr.bundle.reward_model
        for n, w in g.after(s).items():
            np.testing.assert_allclose(model.params.tensors[n], w, rtol=0, atol=1e-10,
                                       err_msg=f"step {s} {kind}.{n}")
    assert tr.obs_updates == m["obs_updates"] and tr.reward_updates == m["reward_updates"]
    assert tr.bundle.obs_model.params.version == m["obs_version"]
    assert tr.bundle.reward_model.params.version == m["reward_version"]
    assert tr.adam_obs.step == m["obs_updates"]


class PubStub:
    def __init__(self, kinds):
        self.configs = {k: object() for k in kinds}
        self.published = []

    def update_weights(self, w):
        self.published.append((w.kind, w.version))


def test_wm_publication_versions():  # reference test_trainer.py:696-711
    from paper_2603_18464_b200.publish import OBS_MODEL, POLICY, REWARD_MODEL
    g = WmGolden("full")
    tr = make_trainer(g, world_model=True)
    tr.service = PubStub((POLICY, OBS_MODEL, REWARD_MODEL))
    tr.publish_initial()
    assert set(tr.service.published) == {(POLICY, 0), (OBS_MODEL, 0), (REWARD_MODEL, 0)}
    trajs = g.trajectories()
    tr.train_obs_model_step(trajs)
    tr.train_obs_model_step(trajs)
    tr.train_reward_model_step(trajs)
    assert (OBS_MODEL, 1) in tr.service.published and (OBS_MODEL, 2) in tr.service.published
    assert (REWARD_MODEL, 1) in tr.service.published


def _batches(tr, g, n):
    rng = np.random.default_rng(3)
    from paper_2603_18464_b200.workload import synthetic_trajectories
    m = g.meta
    out = []
    for _ in range(n):
        trajs = synthetic_trajectories(rng, [4, 3], [True, False], m["k"], m["a"], m["o"])
        out.append(tr.build_train_batch(trajs))
    return out


@pytest.mark.parametrize("n_buf,t_obs,t_reward,want_obs,want_rew",
                         [(6, 2, 4, 4, 2),    # test_trainer.py:724-739
                          (1, 1, 1, 0, 0)])   # buffer below wm_batch_episodes: :742-755
def test_wm_run_schedule(n_buf, t_obs, t_reward, want_obs, want_rew):
    g = WmGolden("full")
    tr = make_trainer(g, world_model=True, t_obs=t_obs, t_reward=t_reward, wm_batch_episodes=4)
    batches = _batches(tr, g, 8 if want_obs else 3)
    wm = rt.ReplayBuffer(g.trajectories() * 2 if n_buf > 1 else g.trajectories()[:1])
    rt.drive(tr.run(rt.Channel(batches), wm, rt.StopFlag()))
    assert tr.cycles == len(batches)
    assert tr.obs_updates == want_obs and tr.reward_updates == want_rew


def test_model_free_run_never_touches_world_models():  # test_trainer.py:758-770
    g = WmGolden("full")
    tr = make_trainer(g)
    batches = _batches(tr, g, 4)
    rt.drive(tr.run(rt.Channel(batches), rt.ReplayBuffer(g.trajectories() * 3), rt.StopFlag()))
    assert tr.cycles == 4 and tr.obs_updates == 0 and tr.reward_updates == 0


def test_wm_errors():
    from paper_2603_18464_b200.errors import DomainError, NonFiniteError
    g = WmGolden("full")
    tr = make_trainer(g)
    with pytest.raises(DomainError, match="no transitions"):
        tr.train_obs_model_step([])
    bad = g.trajectories()
    bad[0].observations = bad[0].observations.copy()
    bad[0].observations[1, 0] = np.nan
    before = tr.bundle.obs_model.params.tensors["w0"].copy()
    with pytest.raises(NonFiniteError):
        tr.train_obs_model_step(bad)
    np.testing.assert_array_equal(tr.bundle.obs_model.params.tensors["w0"], before)
