"""Golden OUTPUTS of the REAL reference at BASELINE cfg1 full size.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_cfg1.py

cfg1: 64 trajectories x 128 steps (N = 8192, M = 57,344
tokens), K = 7, A = 256 (slim head of a 32000 vocabulary at 31744), D = 64,
obs 195, value n_steps 130 / mlp 32.  The inputs are regenerated from their
seed by `tests/cfg1_workload.py` (pure NumPy) on both sides, so only the
initial parameters and the reference's outputs are stored: per step the
batch (advantages, value targets, behavior log-probs as float32), its
metadata, the train_step record and the parameters after the update.

Cases: trust arm with revaluation (two steps, the second on fresh
trajectories under the updated critic, behavior lag 1), clip arm without
revaluation (one step).  The reference is imported, never copied.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))

from asyncrl.models import (  # noqa: E402
    ModelBundle, ObsModel, ObsModelConfig, PolicyConfig, PolicyModel, RewardModel, ValueConfig,
    ValueHead)
from asyncrl.rollout import Trajectory  # noqa: E402
from asyncrl.trainer import GaeConfig, LossConfig, Trainer, TrainerConfig  # noqa: E402

from cfg1_workload import A, D, K, MLP, N_STEPS, O, cfg1_trajectories  # noqa: E402

CASES = {
    "trainer_cfg1_full_trust": dict(seed=1001, steps=2, lag=1,
                                    cfg=TrainerConfig(gae=GaeConfig(0.99, 0.95), k_shards=4)),
    "trainer_cfg1_full_clip": dict(seed=1002, steps=1, lag=0,
                                   cfg=TrainerConfig(loss=LossConfig(algorithm="clip"),
                                                     revalue=False, k_shards=4)),
}


def run_case(name, seed, steps, lag, cfg):
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0]))
    bundle = ModelBundle(
        policy=PolicyModel.init(rng, PolicyConfig(obs_dim=O, hidden_dim=D, chunk_len=K,
                                                  n_actions=A, vocab_size=32000,
                                                  action_start=31744)),
        value=ValueHead.init(rng, ValueConfig(hidden_dim=D, n_steps=N_STEPS, mlp_hidden=MLP)),
        obs_model=ObsModel.init(rng, ObsModelConfig(obs_dim=O, chunk_len=K, n_actions=A)),
        reward_model=RewardModel.init(rng, O))
    tr = Trainer(bundle, cfg)
    arrays = {}
    for k, v in bundle.policy.params.tensors.items():
        arrays[f"init.policy.{k}"] = v.copy()
    for k, v in bundle.value.params.tensors.items():
        arrays[f"init.value.{k}"] = v.copy()
    meta = {"name": name, "seed": seed, "steps": steps, "lag": lag, "o": O, "d": D, "k": K, "a": A,
            "n_steps": N_STEPS, "mlp_hidden": MLP,
            "cfg": {"gamma": cfg.gae.gamma, "lam": cfg.gae.lam, "algorithm": cfg.loss.algorithm,
                    "sigma": cfg.loss.sigma, "clip_eps": cfg.loss.clip_eps,
                    "lambda_v": cfg.loss.lambda_v, "lambda_h": cfg.loss.lambda_h, "lr": cfg.lr,
                    "k_shards": cfg.k_shards, "revalue": cfg.revalue},
            "records": [], "batch_meta": []}
    for s in range(steps):
        version = max(0, tr.publish_version - lag)
        trajs = cfg1_trajectories(seed, s, cls=Trajectory, version=version)
        batch = tr.build_train_batch(trajs)
        assert batch is not None
        for f in ("advantages", "value_targets", "behavior_logp"):
            arrays[f"s{s}.batch.{f}"] = np.asarray(getattr(batch, f), dtype=np.float32)
        meta["batch_meta"].append({
            "version": version, "critic_version": batch.critic_version, "n_real": batch.n_real,
            "n_imagined": batch.n_imagined, "norm_mean": batch.norm_mean,
            "norm_std": batch.norm_std, "norm_count": batch.norm_count,
            "shard_sizes": list(batch.shard_sizes), "behavior_lag_mean": batch.behavior_lag_mean})
        rec = tr.train_step(batch)
        assert rec is not None
        meta["records"].append({k2: (float(v) if isinstance(v, (float, np.floating)) else int(v))
                                for k2, v in rec.items()})
        for k, v in tr.bundle.policy.params.tensors.items():
            arrays[f"s{s}.after.policy.{k}"] = v.copy()
        for k, v in tr.bundle.value.params.tensors.items():
            arrays[f"s{s}.after.value.{k}"] = v.copy()
    np.savez_compressed(HERE / f"{name}.npz", **arrays)
    (HERE / f"{name}.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print(name, meta["records"])


if __name__ == "__main__":
    for nm, kw in CASES.items():
        run_case(nm, **kw)
