"""Golden fixtures for the world-model training sub-steps, made by running the
REAL reference trainer in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_wm.py

Reference: `Trainer.train_obs_model_step` / `train_reward_model_step`
(trainer.py:469-535).  A reference Trainer (seed 5) runs an interleaved
sequence of obs-model and reward-model sub-steps on fixed trajectories, with
`wm_max_transitions` and `reward_neg_ratio` small enough that both
`rng.choice` subsampling paths fire; the fixture stores the initial world-model
parameters, the trajectories, and after every sub-step the loss and the updated
parameters.  The GPU box has no reference checkout: tests read only the .npz.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from asyncrl.models import (  # noqa: E402
    ModelBundle, ObsModel, ObsModelConfig, PolicyConfig, PolicyModel, RewardModel,
    ValueConfig, ValueHead)
from asyncrl.rollout import Trajectory  # noqa: E402
from asyncrl.trainer import Trainer, TrainerConfig  # noqa: E402

OUT = Path(__file__).resolve().parent
SEQ = ["obs", "reward", "obs", "obs", "reward", "reward", "obs"]


def make(name: str, o: int, k: int, a: int, lens, success, lr: float, max_rows: int,
         neg_ratio: int, seed: int = 5) -> None:
    rng = np.random.default_rng(seed)
    pc = PolicyConfig(obs_dim=o, hidden_dim=16, chunk_len=k, n_actions=a, vocab_size=a,
                      action_start=0)
    bundle = ModelBundle(PolicyModel.init(rng, pc), ValueHead.init(rng, ValueConfig(16, 40, 8)),
                         ObsModel.init(rng, ObsModelConfig(obs_dim=o, chunk_len=k, n_actions=a,
                                                           hidden_dim=24)),
                         RewardModel.init(rng, o, hidden_dim=12))
    trajs = []
    for i, (t, ok) in enumerate(zip(lens, success)):
        rew = np.zeros(t)
        if ok:
            rew[-1] = 1.0
        trajs.append(Trajectory(
            task_id=i, source="real", observations=rng.normal(size=(t + 1, o)),
            steps=np.arange(t + 1), tokens=rng.integers(0, a, size=(t, k)), rewards=rew,
            behavior_logits=rng.normal(size=(t, k, a)), values=rng.normal(size=t),
            bootstrap_value=0.0, done=bool(ok), behavior_version=0,
            step_versions=np.zeros(t, dtype=np.int64)))
    out = {"obs0_" + n: v for n, v in bundle.obs_model.params.tensors.items()}
    out.update({"rew0_" + n: v for n, v in bundle.reward_model.params.tensors.items()})
    out.update({"pol_" + n: v for n, v in bundle.policy.params.tensors.items()})
    out.update({"val_" + n: v for n, v in bundle.value.params.tensors.items()})
    for i, tr in enumerate(trajs):
        out[f"traj{i}_obs"] = tr.observations
        out[f"traj{i}_tokens"] = tr.tokens
        out[f"traj{i}_rewards"] = tr.rewards
    cfg = TrainerConfig(lr=lr, wm_max_transitions=max_rows, reward_neg_ratio=neg_ratio,
                        k_shards=1)
    trainer = Trainer(bundle, cfg, seed=seed)
    losses = []
    for s, kind in enumerate(SEQ):
        if kind == "obs":
            losses.append(trainer.train_obs_model_step(trajs))
            for n, v in trainer.bundle.obs_model.params.tensors.items():
                out[f"step{s}_{n}"] = v
        else:
            losses.append(trainer.train_reward_model_step(trajs))
            for n, v in trainer.bundle.reward_model.params.tensors.items():
                out[f"step{s}_{n}"] = v
    meta = {"o": o, "k": k, "a": a, "lens": list(lens), "success": list(map(bool, success)),
            "lr": lr, "max_rows": max_rows, "neg_ratio": neg_ratio, "seed": seed, "seq": SEQ,
            "losses": losses, "obs_updates": trainer.obs_updates,
            "reward_updates": trainer.reward_updates,
            "obs_version": trainer.bundle.obs_model.params.version,
            "reward_version": trainer.bundle.reward_model.params.version,
            "obs_hidden": 24, "reward_hidden": 12}
    np.savez_compressed(OUT / f"wm_{name}.npz", **out)
    (OUT / f"wm_{name}.json").write_text(json.dumps(meta, indent=1))
    print(name, losses)


if __name__ == "__main__":
    # subsampled: 52 transitions > 24 rows; 3 positives x ratio 2 < 55 negatives
    make("subsampled", o=19, k=3, a=5, lens=[9, 4, 14, 7, 6, 12], success=[1, 0, 1, 0, 1, 0],
         lr=0.01, max_rows=24, neg_ratio=2)
    # full: no subsampling; single-class reward batches (no successes)
    make("full", o=11, k=2, a=7, lens=[5, 3, 8], success=[0, 0, 0], lr=0.003, max_rows=512,
         neg_ratio=4)
