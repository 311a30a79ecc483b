"""Generate golden fixtures by running the REAL reference in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference (`/root/reference/pkg/src/asyncrl`, pure NumPy float64) is
imported, never copied.  Each fixture stores the inputs (float64), the
reference outputs, and the parameters before/after the reference's own
`Trainer.build_train_batch` + `Trainer.train_step`.  The GPU box has no
reference checkout; tests read only these files.
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
from asyncrl.trainer import GaeConfig, LossConfig, Trainer, TrainerConfig  # noqa: E402

OUT = Path(__file__).resolve().parent


def make_trajs(rng, lengths, done, k, a, o, n_steps, imagined_every=0, version=0):
    trajs = []
    for i, (t, d) in enumerate(zip(lengths, done)):
        start = int(rng.integers(0, max(1, n_steps - t - 1)))
        trajs.append(Trajectory(
            task_id=i % 3, source="imagined" if imagined_every and i % imagined_every == 1
            else "real",
            observations=rng.normal(size=(t + 1, o)), steps=np.arange(start, start + t + 1),
            tokens=rng.integers(0, a, size=(t, k)), rewards=rng.normal(size=t),
            behavior_logits=rng.normal(size=(t, k, a)), values=rng.normal(size=t),
            bootstrap_value=float(rng.normal()), done=bool(d), behavior_version=version,
            step_versions=np.full(t, version, dtype=np.int64)))
    return trajs


def flat_traj_arrays(trajs, prefix):
    out = {}
    lens = np.array([t.t_len for t in trajs])
    out[prefix + "traj_off"] = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    out[prefix + "frames"] = np.concatenate([t.observations for t in trajs])
    out[prefix + "steps"] = np.concatenate([t.steps for t in trajs])
    out[prefix + "tokens"] = np.concatenate([t.tokens for t in trajs])
    out[prefix + "rewards"] = np.concatenate([t.rewards for t in trajs])
    out[prefix + "mu"] = np.concatenate([t.behavior_logits for t in trajs])
    out[prefix + "values"] = np.concatenate([np.append(t.values, t.bootstrap_value)
                                             for t in trajs])
    out[prefix + "done"] = np.array([t.done for t in trajs], dtype=np.uint8)
    out[prefix + "real"] = np.array([t.source == "real" for t in trajs], dtype=np.uint8)
    out[prefix + "bver"] = np.array([t.behavior_version for t in trajs], dtype=np.int64)
    return out


def params_arrays(bundle, prefix):
    out = {}
    for k, v in bundle.policy.params.tensors.items():
        out[f"{prefix}policy.{k}"] = v.copy()
    for k, v in bundle.value.params.tensors.items():
        out[f"{prefix}value.{k}"] = v.copy()
    return out


def run_case(name, *, seed, o, d, k, a, vocab, start, n_steps, mlp_hidden, lengths, done,
             cfg: TrainerConfig, steps=2, imagined_every=0, lag_version=0):
    rng = np.random.default_rng(seed)
    pol_cfg = PolicyConfig(obs_dim=o, hidden_dim=d, chunk_len=k, n_actions=a,
                           vocab_size=vocab, action_start=start)
    val_cfg = ValueConfig(hidden_dim=d, n_steps=n_steps, mlp_hidden=mlp_hidden)
    bundle = ModelBundle(
        policy=PolicyModel.init(rng, pol_cfg), value=ValueHead.init(rng, val_cfg),
        obs_model=ObsModel.init(rng, ObsModelConfig(obs_dim=o, chunk_len=k, n_actions=a)),
        reward_model=RewardModel.init(rng, o))
    trainer = Trainer(bundle, cfg)
    arrays = params_arrays(bundle, "init.")
    meta = {"name": name, "o": o, "d": d, "k": k, "a": a, "n_steps": n_steps,
            "mlp_hidden": mlp_hidden, "steps": steps,
            "cfg": {"gamma": cfg.gae.gamma, "lam": cfg.gae.lam, "algorithm": cfg.loss.algorithm,
                    "sigma": cfg.loss.sigma, "clip_eps": cfg.loss.clip_eps,
                    "lambda_v": cfg.loss.lambda_v, "lambda_h": cfg.loss.lambda_h,
                    "lr": cfg.lr, "k_shards": cfg.k_shards, "revalue": cfg.revalue},
            "records": [], "batch_meta": []}
    for s in range(steps):
        trajs = make_trajs(rng, lengths, done, k, a, o, n_steps, imagined_every,
                           version=max(0, trainer.publish_version - lag_version))
        arrays.update(flat_traj_arrays(trajs, f"s{s}."))
        batch = trainer.build_train_batch(trajs)
        assert batch is not None
        for f in ("obs", "steps", "tokens", "behavior_logp", "advantages", "value_targets"):
            arrays[f"s{s}.batch.{f}"] = np.asarray(getattr(batch, f))
        meta["batch_meta"].append({
            "critic_version": batch.critic_version, "n_real": batch.n_real,
            "n_imagined": batch.n_imagined, "norm_mean": batch.norm_mean,
            "norm_std": batch.norm_std, "norm_count": batch.norm_count,
            "shard_sizes": list(batch.shard_sizes), "behavior_lag_mean": batch.behavior_lag_mean})
        rec = trainer.train_step(batch)
        assert rec is not None
        meta["records"].append({k2: (float(v) if isinstance(v, (float, np.floating)) else int(v))
                                for k2, v in rec.items()})
        arrays.update(params_arrays(bundle, f"s{s}.after."))
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    (OUT / f"{name}.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print(name, "records:", meta["records"])


def main():
    small = dict(o=20, d=16, k=3, a=16, vocab=64, start=40, n_steps=48, mlp_hidden=8,
                 lengths=[5, 1, 9, 3, 12, 7], done=[True, False, True, False, False, True])
    run_case("trainer_trust_revalue", seed=101, cfg=TrainerConfig(k_shards=4), **small,
             imagined_every=2, lag_version=1)
    run_case("trainer_clip_stored", seed=202,
             cfg=TrainerConfig(loss=LossConfig(algorithm="clip", clip_eps=0.2), revalue=False,
                               k_shards=3), **small)
    run_case("trainer_cfg1_dims", seed=303,
             cfg=TrainerConfig(gae=GaeConfig(0.99, 0.95), k_shards=4),
             o=195, d=64, k=7, a=256, vocab=32000, start=31744, n_steps=140, mlp_hidden=32,
             lengths=[8, 5, 11], done=[True, False, True], steps=2)


if __name__ == "__main__":
    main()
