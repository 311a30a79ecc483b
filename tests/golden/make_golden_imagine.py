"""Golden fixtures for the imagination step, from the REAL reference worker.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_imagine.py

Runs `RolloutWorker.imagine_episode` (rollout.py:295-362) through the
reference InferenceService on its virtual-clock scheduler, records every
policy request's ticket (by wrapping `inference.run_batch`) and derives the
uniforms that request consumed: `default_rng(SeedSequence([base_seed,
ticket])).random()` K times (inference.py:147, models.py:146).  The GPU
imagination kernel is then fed the same uniforms.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import asyncrl.inference as inf  # noqa: E402
from asyncrl.buffers import IMAGINED, MAIN, WORLD_MODEL, ReplayBuffer  # noqa: E402
from asyncrl.env import GridTaskSuite, TaskSuiteConfig  # noqa: E402
from asyncrl.models import (ModelBundle, ObsModel, ObsModelConfig, PolicyConfig,  # noqa: E402
                            PolicyModel, RewardModel, ValueConfig, ValueHead)
from asyncrl.rollout import EpisodeBuffer, RolloutWorker, TaskStats, WorkerConfig  # noqa: E402
from asyncrl.runtime import Scheduler  # noqa: E402

OUT = Path(__file__).resolve().parent
BASE_SEED = 17

_calls = []
_orig_run_batch = inf.run_batch


def _recording_run_batch(weights, requests, base_seed):
    for r in requests:
        _calls.append((r.kind, r.ticket))
    return _orig_run_batch(weights, requests, base_seed)


inf.run_batch = _recording_run_batch


def run_case(name, *, height, width, chunk_len, hidden, obs_hidden, reward_hidden, h_img,
             n_starts, seed, rig=None, threshold=0.9):
    suite = GridTaskSuite(TaskSuiteConfig(height=height, width=width, num_tasks=3,
                                          horizon=40, chunk_len=chunk_len,
                                          kinds=("reach", "fetch", "transport")))
    o = suite.cfg.obs_dim
    rng = np.random.default_rng(np.random.SeedSequence([seed, 3]))
    bundle = ModelBundle(
        policy=PolicyModel.init(rng, PolicyConfig(obs_dim=o, hidden_dim=hidden,
                                                  chunk_len=chunk_len, vocab_size=32,
                                                  action_start=16)),
        value=ValueHead.init(rng, ValueConfig(hidden_dim=hidden, n_steps=64, mlp_hidden=8)),
        obs_model=ObsModel.init(rng, ObsModelConfig(obs_dim=o, chunk_len=chunk_len,
                                                    hidden_dim=obs_hidden)),
        reward_model=RewardModel.init(rng, o, hidden_dim=reward_hidden))
    if rig is not None:
        rig(bundle)
    sched = Scheduler()
    window = inf.BatchWindowConfig(batch_size=1, max_wait=0.005)
    kinds = (inf.POLICY, inf.OBS_MODEL, inf.REWARD_MODEL)
    service = inf.InferenceService(sched, {k: window for k in kinds}, obs_dim=o,
                                   base_seed=BASE_SEED)
    for k in kinds:
        service.update_weights(inf.VersionedWeights.from_bundle(k, 0, bundle))
    worker = RolloutWorker(worker_id=0, suite=suite, service=service,
                           main_buffer=ReplayBuffer(MAIN, 8), wm_buffer=ReplayBuffer(WORLD_MODEL, 8),
                           img_buffer=ReplayBuffer(IMAGINED, 8), episode_buffer=EpisodeBuffer(8),
                           task_stats=TaskStats(3),
                           cfg=WorkerConfig(n_imagined_per_real=1, h_img=h_img,
                                            success_threshold=threshold),
                           run_seed=7)
    starts = [suite.reset(i % 3, 1000 + i).observation() for i in range(n_starts)]
    results = []

    def body():
        for st in starts:
            _calls.clear()
            traj = yield from worker.imagine_episode(st)
            pol_tickets = [t for kind, t in _calls if kind == inf.POLICY]
            results.append((traj, pol_tickets))
        service.shutdown()

    sched.spawn("body", body())
    service.start()
    sched.run()

    arrays = {}
    for which, model in (("policy", bundle.policy), ("value", bundle.value),
                         ("obs", bundle.obs_model), ("reward", bundle.reward_model)):
        for k, v in model.params.tensors.items():
            arrays[f"{which}.{k}"] = v
    meta = {"name": name, "height": height, "width": width, "obs_dim": o,
            "chunk_len": chunk_len, "n_actions": 7, "hidden": hidden, "n_steps": 64,
            "mlp_hidden": 8, "obs_hidden": obs_hidden, "reward_hidden": reward_hidden,
            "h_img": h_img, "threshold": threshold, "base_seed": BASE_SEED, "episodes": []}
    for e, (st, (traj, tickets)) in enumerate(zip(starts, results)):
        u = np.stack([np.random.default_rng(np.random.SeedSequence([BASE_SEED, t])).random(chunk_len)
                      for t in tickets]) if tickets else np.zeros((0, chunk_len))
        arrays[f"e{e}.start_vec"] = st.vec
        arrays[f"e{e}.uniforms"] = u
        ep = {"start_step": int(st.step), "task_id": int(st.task_id), "tickets": tickets,
              "discarded": traj is None}
        if traj is not None:
            for f in ("observations", "steps", "tokens", "rewards", "behavior_logits", "values"):
                arrays[f"e{e}.{f}"] = np.asarray(getattr(traj, f))
            ep.update(bootstrap_value=float(traj.bootstrap_value), done=bool(traj.done),
                      t_len=int(traj.t_len))
        meta["episodes"].append(ep)
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    (OUT / f"{name}.json").write_text(json.dumps(meta, indent=1))
    print(name, [(ep.get("t_len"), ep.get("done"), ep["discarded"]) for ep in meta["episodes"]])


def main():
    run_case("imagine_small", height=4, width=4, chunk_len=2, hidden=16, obs_hidden=24,
             reward_hidden=12, h_img=6, n_starts=6, seed=1)
    run_case("imagine_default_dims", height=8, width=8, chunk_len=4, hidden=64, obs_hidden=96,
             reward_hidden=64, h_img=16, n_starts=5, seed=2)

    def high_reward(b):  # sigmoid(10) > 0.9 everywhere: done-hat after one step
        b.reward_model.params.tensors["w1"][:] = 0.0
        b.reward_model.params.tensors["b1"][:] = 10.0

    run_case("imagine_done_hat", height=4, width=4, chunk_len=2, hidden=16, obs_hidden=24,
             reward_hidden=12, h_img=5, n_starts=3, seed=3, rig=high_reward)

    def nan_obs(b):  # non-finite obs prediction: discarded (rollout.py:315-320)
        b.obs_model.params.tensors["b1"][0] = np.nan

    run_case("imagine_nan_obs", height=4, width=4, chunk_len=2, hidden=16, obs_hidden=24,
             reward_hidden=12, h_img=5, n_starts=2, seed=4, rig=nan_obs)


if __name__ == "__main__":
    main()
