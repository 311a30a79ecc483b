"""cfg5 loop benchmark: world-model-augmented PPO cycles on one B200.

    python profiles/loop_bench.py [--n 4096] [--h 16] [--cycles 5]
    torchrun --nproc-per-node R --master-addr 127.0.0.1 profiles/loop_bench.py

Under torchrun each rank imagines its own n episodes (replicas), the
PPO step is data-parallel over NCCL (ZeRO-2, `dp.DataParallel`), and every rank
runs the same world-model sub-steps on the same data (float64, deterministic,
so the replicas stay identical without a collective).  Cycle time = max over
ranks; trained transitions are summed over ranks.

The reference's world-model mode (harness.py:220-221: the trainer's batches
come from the imagination buffer) with its default grid dimensions (8x8: obs
195, K = 4, A = 7, D = 64; obs-model hidden 96, reward hidden 64).  One cycle:

  1. imagine n start frames x H steps in one persistent launch
     (`Imaginer.imagine_device`, rollout.py:295-362);
  2. push the kept episodes into the HBM imagination buffer without a host
     round trip (`DeviceReplayBuffer.push_imagined`, buffers.py:44-94);
  3. sample n episodes, build the TrainBatch on the device and take one PPO
     step (`build_train_batch` + `train_step`, trainer.py:365-467);
  4. one obs-model and one reward-model training sub-step on the world-model
     buffer's real trajectories (trainer.py:469-535, schedule :552-560) with the
     reference's default wm_batch_episodes = 8.

Random-init models, synthetic real trajectories (N(0,1) frames) for the world
model.  Wall time per cycle (torch.cuda.synchronize on both sides), best of
`--cycles` after 2 warm-up cycles; prints one JSON line with the per-phase split.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--h", type=int, default=16)
    ap.add_argument("--cycles", type=int, default=5)
    args = ap.parse_args()
    import torch

    from paper_2603_18464_b200.imagine import Imaginer
    from paper_2603_18464_b200.replay import DeviceReplayBuffer
    from paper_2603_18464_b200.trainer import Trainer, TrainerConfig
    from paper_2603_18464_b200.types import (ModelBundle, ObsModel, ObsModelConfig,
                                             PolicyConfig, PolicyModel, RewardModel, ValueConfig,
                                             ValueHead)
    from paper_2603_18464_b200.workload import synthetic_trajectories

    import os

    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    comm = None
    if world > 1:
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from paper_2603_18464_b200.dp import DataParallel
        comm = DataParallel()
    O, K, A, D = 195, 4, 7, 64
    n, H = args.n, args.h
    rng = np.random.default_rng(0)
    bundle = ModelBundle(PolicyModel.init(rng, PolicyConfig(obs_dim=O, hidden_dim=D, chunk_len=K)),
                         ValueHead.init(rng, ValueConfig(hidden_dim=D, n_steps=64, mlp_hidden=32)),
                         ObsModel.init(rng, ObsModelConfig(obs_dim=O, chunk_len=K, hidden_dim=96)),
                         RewardModel.init(rng, O, hidden_dim=64))
    starts = np.zeros((n, O))
    for e in range(n):
        for c in range(3):
            starts[e, c * 64 + rng.integers(64)] = 1.0
        starts[e, 192 + e % 3] = 1.0
    start_steps = rng.integers(0, 16, size=n)
    srng = np.random.default_rng(100 + rank)  # this rank's start frames (replicas)
    starts = starts[srng.permutation(n)]
    # world-model buffer: real trajectories (the reference's wm_buffer holds real episodes)
    lens = rng.integers(8, 41, size=64)
    real = synthetic_trajectories(rng, lens, rng.random(64) < 0.5, K, A, O, n_steps=64)

    trainer = Trainer(bundle, TrainerConfig(), comm=comm)
    rng = np.random.default_rng(1000 + rank)  # this rank's replay sampling
    im = Imaginer(bundle, grid=(8, 8))
    img = DeviceReplayBuffer("imagined", capacity=2 * n, obs_dim=O, chunk_len=K, n_actions=A,
                             max_transitions=2 * n * H)
    x0 = torch.as_tensor(starts, device="cuda")
    wm_rng = np.random.default_rng(7)
    phases = ("imagine_push", "build_step", "world_model")
    best = {p: 1e9 for p in phases}
    best_total, pushed, transitions = 1e9, 0, 0
    for cyc in range(args.cycles + 2):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t = [time.perf_counter()]
        out = im.imagine_device(x0, start_steps, H, seed=cyc)
        pushed = img.push_imagined(out, version=trainer.publish_version)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        picks = img.sample(min(n, len(img)), rng)
        batch = trainer.build_train_batch(picks)
        rec = trainer.train_step(batch)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        wm = [real[int(i)] for i in wm_rng.integers(0, len(real), size=8)]
        trainer.train_obs_model_step(wm)
        trainer.train_reward_model_step(wm)
        im.update(trainer.bundle, trainer.publish_version)  # fresh weights for the next cycle
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        span = torch.tensor([t[-1] - t[0], float(batch.n_transitions)], dtype=torch.float64,
                            device="cuda")
        if world > 1:  # cycle time = max over ranks, transitions summed
            mx = span[:1].clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            dist.all_reduce(span[1:], op=dist.ReduceOp.SUM)
            span[0] = mx[0]
        cyc_s, cyc_tr = span.tolist()
        if cyc >= 2:
            for p, a, b in zip(phases, t, t[1:]):
                best[p] = min(best[p], (b - a) * 1e3)
            if cyc_s < best_total:
                best_total = cyc_s
                transitions = int(cyc_tr)
        assert rec is not None, "the PPO step dropped its batch"
    if rank != 0:
        dist.destroy_process_group()
        return
    print(json.dumps({
        "workload": f"cfg5 world-model-augmented PPO cycle, {world} GPU (grid 8x8: obs 195, K=4, "
                    "A=7, D=64)",
        "n_gpus": world, "scaling": "weak (n imagined episodes per GPU)",
        "imagined_episodes_per_cycle_per_gpu": n, "horizon": H, "pushed_last_cycle": pushed,
        "trained_transitions_per_cycle": transitions,
        "ms_per_cycle": best_total * 1e3,
        "trained_transitions_per_s": transitions / best_total,
        "phase_ms_best": best,
        "timing": f"wall clock, cuda synchronize on both sides, best of {args.cycles} after 2 warm-up",
        "data": "random-init models, synthetic real trajectories for the world-model sub-steps",
    }))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
