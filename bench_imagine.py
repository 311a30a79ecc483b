"""cfg3 imagination benchmark (secondary line; bench.py carries the headline).

4096 start frames x H = 16 imagined steps with the reference's default
harness dimensions (8x8 grid: obs 195, K = 4, A = 7, policy D = 64, obs-model
hidden 96, reward hidden 64), snap on, threshold 0.9, random-init models
(an untrained reward head never reaches the threshold, so every episode runs
the full horizon).  Prints one JSON line: imagined steps/s for the
single-launch GPU kernel (device-timed), the end-to-end call (host starts in,
host trajectories out) and the float64 restatement of the reference's
per-request loop on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--h", type=int, default=16)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--cpu-sample", type=int, default=64)
    args = ap.parse_args()
    print(json.dumps(run(args.n, args.h, args.steps, args.cpu_sample)))


def run(n: int = 4096, h: int = 16, steps: int = 5, cpu_sample: int = 64) -> dict:
    """The cfg3 line (bench.py carries it as its `cfg3` extra)."""
    import torch
    args = argparse.Namespace(n=n, h=h, steps=steps, cpu_sample=cpu_sample)

    from paper_2603_18464_b200.imagine import Imaginer
    from paper_2603_18464_b200.types import (ModelBundle, ObsModel, ObsModelConfig,
                                             PolicyConfig, PolicyModel, RewardModel, ValueConfig,
                                             ValueHead)
    O, K, A, D = 195, 4, 7, 64
    rng = np.random.default_rng(0)
    b = ModelBundle(PolicyModel.init(rng, PolicyConfig(obs_dim=O, hidden_dim=D, chunk_len=K)),
                    ValueHead.init(rng, ValueConfig(hidden_dim=D, n_steps=64, mlp_hidden=32)),
                    ObsModel.init(rng, ObsModelConfig(obs_dim=O, chunk_len=K, hidden_dim=96)),
                    RewardModel.init(rng, O, hidden_dim=64))
    starts = np.zeros((args.n, O))
    for e in range(args.n):
        for c in range(3):
            starts[e, c * 64 + rng.integers(64)] = 1.0
        starts[e, 192 + e % 3] = 1.0
    steps = rng.integers(0, 16, size=args.n)
    im = Imaginer(b, grid=(8, 8))
    # warm-up until torch's page-locked host cache holds two live result sets (the
    # returned arrays own their buffers; a loop keeps the previous batch while the
    # next one lands)
    for _ in range(4):
        res = im.imagine(starts, steps, args.h, seed=1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s in range(args.steps):
        res = im.imagine(starts, steps, args.h, seed=s)  # includes H2D + D2H of the batch
    e2e_s = (time.perf_counter() - t0) / args.steps
    imagined = int(res["t_len"].sum())
    # device-only timing: inputs resident, outputs left on the device
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x = torch.as_tensor(starts, device="cuda")
    st = torch.as_tensor(steps, dtype=torch.int32, device="cuda")
    im.imagine_device(x, st, args.h, seed=0)
    torch.cuda.synchronize()
    ev0.record()
    for s in range(args.steps):
        im.imagine_device(x, st, args.h, seed=s)
    ev1.record()
    torch.cuda.synchronize()
    # CPU reference loop (float64 restatement of the per-request evaluations)
    from oracle.imagine_ref import imagine_episode
    u = np.random.default_rng(2).random((args.cpu_sample, args.h + 1, K))
    t1 = time.perf_counter()
    cpu_steps = 0
    for e in range(args.cpu_sample):
        out = imagine_episode(b.policy.params.tensors, b.value.params.tensors,
                              b.obs_model.params.tensors, b.reward_model.params.tensors, A,
                              starts[e], int(steps[e]), u[e], args.h, 0.9, (8, 8))
        cpu_steps += out["t_len"]
    cpu_rate = cpu_steps / (time.perf_counter() - t1) if args.cpu_sample else None
    return ({
        "metric": "imagined steps/s", "unit": "steps/s",
        "value": imagined / e2e_s,
        "config": {"workload": f"cfg3 imagination {args.n} x H{args.h}, obs 195, K 4, A 7, D 64",
                   "trajectories": args.n, "horizon": args.h},
        "e2e_ms_per_batch": e2e_s * 1e3,
        "device_ms_per_batch": ev0.elapsed_time(ev1) / args.steps,
        "device_steps_per_s": imagined / (ev0.elapsed_time(ev1) / args.steps / 1e3),
        "cpu_baseline": None if cpu_rate is None else {
            "value": cpu_rate, "unit": "steps/s", "cores": 1, "kind": "port",
            "sample": f"{args.cpu_sample} episodes x H{args.h}, float64 per-request loop"},
    })


if __name__ == "__main__":
    main()
