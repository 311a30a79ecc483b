"""Batch build from the on-device replay buffer vs from host trajectories.

    python profiles/replay_bench.py [n_traj]

LIBERO-Long-like trajectories (K = 7, A = 256, O = 195) are pushed once into a
DeviceReplayBuffer; then batches of n_traj sampled trajectories are built
(a) from the buffer's handles (on-device gathers) and (b) from the same host
Trajectory objects (host pack + host-to-device copy), each followed by the
train step.  Wall time per batch, best of 3.
"""

import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2603_18464_b200.replay import DeviceReplayBuffer  # noqa: E402
from paper_2603_18464_b200.trainer import Trainer, TrainerConfig  # noqa: E402
from paper_2603_18464_b200.types import (ModelBundle, PolicyConfig, PolicyModel,  # noqa: E402
                                         ValueConfig, ValueHead)
from paper_2603_18464_b200.workload import libero_long_lengths, synthetic_trajectories  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    K, A, O, D = 7, 256, 195, 64
    rng = np.random.default_rng(0)
    pc = PolicyConfig(obs_dim=O, hidden_dim=D, chunk_len=K, n_actions=A, vocab_size=32000,
                      action_start=31744)
    bundle = ModelBundle(PolicyModel.init(rng, pc), ValueHead.init(rng, ValueConfig(D, 522, 32)))
    lens, done = libero_long_lengths(rng, n)
    trajs = synthetic_trajectories(rng, lens, done, K, A, O)
    buf = DeviceReplayBuffer("main", capacity=n, obs_dim=O, chunk_len=K, n_actions=A,
                             max_transitions=int(lens.sum()) + 1)
    t0 = time.perf_counter()
    for t in trajs:
        buf.push(t)
    torch.cuda.synchronize()
    push_s = time.perf_counter() - t0
    tr = Trainer(bundle, TrainerConfig())
    out = {}
    for name in ("device", "host"):
        best = 1e9
        for rep in range(4):
            g = np.random.default_rng(rep)
            picks = buf.sample(n, g)
            host = [trajs[len(trajs) - len(buf) + int(i)]
                    for i in np.random.default_rng(rep).integers(0, len(buf), size=n)]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            batch = tr.build_train_batch(picks if name == "device" else host)
            tr.train_step(batch)
            torch.cuda.synchronize()
            if rep:
                best = min(best, time.perf_counter() - t0)
        out[name + "_ms_per_batch"] = best * 1e3
    out.update({"trajectories": n, "transitions": int(lens.sum()), "push_s_total": push_s,
                "speedup": out["host_ms_per_batch"] / out["device_ms_per_batch"]})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
