"""CPU: the float64 world-model restatement (oracle/wm_ref.py) and the host
data selection of the device sub-steps (paper_2603_18464_b200.world_model:
which transitions / frames enter, rng.choice subsampling) reproduce the
reference trainer's fixtures (tests/golden/make_golden_wm.py)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import wm_ref
from paper_2603_18464_b200.world_model import obs_model_data, reward_model_data
from wm_fixture import WM_CASES, WmGolden


class _ObsCfg:
    def __init__(self, a):
        self.cfg = type("C", (), {"n_actions": a})()


@pytest.mark.parametrize("name", WM_CASES)
def test_wm_oracle_matches_reference_fixture(name):
    g = WmGolden(name)
    m = g.meta
    rng = np.random.default_rng(np.random.SeedSequence([m["seed"], 7]))
    trajs = g.trajectories()
    models = {"obs": g.params("obs0_"), "reward": g.params("rew0_")}
    state = {k: ({n: np.zeros_like(v) for n, v in p.items()},
                 {n: np.zeros_like(v) for n, v in p.items()}, 0) for k, p in models.items()}
    for s, kind in enumerate(m["seq"]):
        if kind == "obs":
            x, y = obs_model_data(_ObsCfg(m["a"]), trajs, m["max_rows"], rng)
            loss, grads = wm_ref.loss_and_grad(models[kind], x, y, 0)
        else:
            x, y, _ = reward_model_data(trajs, m["neg_ratio"], m["max_rows"], rng)
            loss, grads = wm_ref.loss_and_grad(models[kind], x, y, 1)
        mm, vv, t = state[kind]
        models[kind], mm, vv = wm_ref.adam(models[kind], grads, mm, vv, t + 1, m["lr"])
        state[kind] = (mm, vv, t + 1)
        assert abs(loss - m["losses"][s]) <= 1e-12 * max(1.0, abs(m["losses"][s])), (s, kind)
        for n, want in g.after(s).items():
            np.testing.assert_allclose(models[kind][n], want, rtol=0, atol=1e-12,
                                       err_msg=f"step {s} {kind}.{n}")


def test_wm_data_selection_errors():
    from paper_2603_18464_b200.errors import DomainError
    with pytest.raises(DomainError, match="no transitions"):
        obs_model_data(_ObsCfg(3), [], 8, np.random.default_rng(0))
