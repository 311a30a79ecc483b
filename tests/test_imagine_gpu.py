"""(c) Imagination kernel vs the real reference worker (golden) and the float64 oracle.

Injected uniforms reproduce the reference's per-ticket RNG, so tokens, frame
steps, done-hat, lengths and discards must match exactly; observations are
snapped grid encodings (exact), logits/values/rewards agree to float64
round-off of a different summation order.
"""

from __future__ import annotations

import numpy as np
import pytest

from golden_io import IMAGINE_CASES, ImagineGolden
from oracle.imagine_ref import imagine_episode

pytestmark = pytest.mark.gpu
FTOL = 1e-9


def bundle_from(g: ImagineGolden):
    from paper_2603_18464_b200.types import (ModelBundle, ObsModel, ObsModelConfig, ParamSet,
                                             PolicyConfig, PolicyModel, RewardModel,
                                             ValueConfig, ValueHead)
    m = g.meta
    pc = PolicyConfig(obs_dim=m["obs_dim"], hidden_dim=m["hidden"], chunk_len=m["chunk_len"],
                      n_actions=m["n_actions"], vocab_size=32, action_start=16)
    vc = ValueConfig(hidden_dim=m["hidden"], n_steps=m["n_steps"], mlp_hidden=m["mlp_hidden"])
    oc = ObsModelConfig(obs_dim=m["obs_dim"], chunk_len=m["chunk_len"], hidden_dim=m["obs_hidden"])
    return ModelBundle(PolicyModel(pc, ParamSet(g.params("policy"))),
                       ValueHead(vc, ParamSet(g.params("value"))),
                       ObsModel(oc, ParamSet(g.params("obs"))),
                       RewardModel(m["obs_dim"], ParamSet(g.params("reward")), m["reward_hidden"]))


@pytest.mark.parametrize("name", IMAGINE_CASES)
def test_imagination_matches_reference(name):
    from paper_2603_18464_b200.imagine import Imaginer

    g = ImagineGolden(name)
    m = g.meta
    H, K = m["h_img"], m["chunk_len"]
    im = Imaginer(bundle_from(g), grid=(m["height"], m["width"]), threshold=m["threshold"])
    n = len(g.episodes)
    vecs = np.stack([g.start(e)[0] for e in range(n)])
    steps = [g.start(e)[1] for e in range(n)]
    u = np.zeros((n, H + 1, K))
    for e in range(n):
        ue = g.uniforms(e)
        u[e, :ue.shape[0]] = ue
    res = im.imagine(vecs, steps, H, uniforms=u)
    for e, ep in enumerate(g.episodes):
        if ep["discarded"]:
            assert res["status"][e] != 0
            continue
        assert res["status"][e] == 0
        T = ep["t_len"]
        ref = g.traj(e)
        assert res["t_len"][e] == T and bool(res["done"][e]) == ep["done"]
        np.testing.assert_array_equal(res["tokens"][e, :T], ref["tokens"])
        np.testing.assert_array_equal(res["steps"][e, :T + 1], ref["steps"])
        np.testing.assert_array_equal(res["observations"][e, :T + 1], ref["observations"])
        np.testing.assert_allclose(res["behavior_logits"][e, :T], ref["behavior_logits"],
                                   rtol=0, atol=FTOL)
        np.testing.assert_allclose(res["values"][e, :T], ref["values"], rtol=0, atol=FTOL)
        np.testing.assert_allclose(res["rewards"][e, :T], ref["rewards"], rtol=0, atol=FTOL)
        assert abs(res["bootstrap_value"][e] - ep["bootstrap_value"]) < FTOL


def test_imagination_cfg3_scale_against_oracle_sample():
    """cfg3: 4096 trajectories x H = 16 in one launch; a sample checked vs the oracle."""
    from paper_2603_18464_b200.imagine import Imaginer

    g = ImagineGolden("imagine_default_dims")
    m = g.meta
    H, K, n = 16, m["chunk_len"], 4096
    im = Imaginer(bundle_from(g), grid=(m["height"], m["width"]), threshold=m["threshold"])
    rng = np.random.default_rng(3)
    base = np.stack([g.start(e)[0] for e in range(len(g.episodes))])
    vecs = base[rng.integers(0, base.shape[0], size=n)]
    steps = rng.integers(0, 20, size=n)
    u = rng.random((n, H + 1, K))
    res = im.imagine(vecs, steps, H, uniforms=u)
    assert np.all(res["status"] == 0)
    for e in rng.choice(n, size=24, replace=False):
        out = imagine_episode(g.params("policy"), g.params("value"), g.params("obs"),
                              g.params("reward"), m["n_actions"], vecs[e], steps[e], u[e], H,
                              m["threshold"], (m["height"], m["width"]))
        T = out["t_len"]
        assert res["t_len"][e] == T
        np.testing.assert_array_equal(res["tokens"][e, :T], out["tokens"])
        np.testing.assert_allclose(res["rewards"][e, :T], out["rewards"], atol=FTOL)
        # telescoping: sum of imagined rewards = p_last - p_first (tests/test_rollout.py:355-363)


def test_imagined_trajectories_feed_the_trainer():
    """Imagined episodes are valid TrainBatch input (source 'imagined')."""
    from paper_2603_18464_b200.imagine import Imaginer
    from paper_2603_18464_b200.trainer import Trainer, TrainerConfig

    g = ImagineGolden("imagine_small")
    m = g.meta
    b = bundle_from(g)
    im = Imaginer(b, grid=(m["height"], m["width"]))
    class Obs:
        def __init__(self, vec, step, task_id):
            self.vec, self.step, self.task_id = vec, step, task_id
    starts = [Obs(*g.start(e)) for e in range(len(g.episodes))]
    trajs = [t for t in im.imagine_trajectories(starts, m["h_img"], seed=5) if t is not None]
    assert trajs and all(t.source == "imagined" for t in trajs)
    tr = Trainer(b, TrainerConfig())
    batch = tr.build_train_batch(trajs)
    assert batch is not None and batch.n_imagined == len(trajs)
    assert tr.train_step(batch) is not None
