"""Multi-GPU parity check (run under torchrun, one process per GPU).

Every rank owns a contiguous, transition-balanced slice of one seeded set of
trajectories and runs the ZeRO-2 data-parallel trainer (NCCL).  Rank 0 also
runs the single-process trainer on the concatenated batch; the records and
the updated parameters must agree up to float summation order.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2603_18464_b200.dp import DataParallel, partition_trajectories  # noqa: E402
from paper_2603_18464_b200.trainer import Trainer, TrainerConfig  # noqa: E402
from paper_2603_18464_b200.types import (ModelBundle, PolicyConfig, PolicyModel,  # noqa: E402
                                         ValueConfig, ValueHead)
from paper_2603_18464_b200.workload import synthetic_trajectories  # noqa: E402


def bundle(seed=4):
    rng = np.random.default_rng(seed)
    pc = PolicyConfig(obs_dim=40, hidden_dim=64, chunk_len=7, n_actions=256, vocab_size=300,
                      action_start=10)
    vc = ValueConfig(hidden_dim=64, n_steps=64, mlp_hidden=32)
    return ModelBundle(PolicyModel.init(rng, pc), ValueHead.init(rng, vc))


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    rng = np.random.default_rng(21)
    lens = rng.integers(1, 60, size=24)
    trajs = synthetic_trajectories(rng, lens, rng.random(24) < 0.5, 7, 256, 40)
    a, b = partition_trajectories(lens, world, rank)
    dp_tr = Trainer(bundle(), TrainerConfig(), comm=DataParallel())
    ref_tr = Trainer(bundle(), TrainerConfig()) if rank == 0 else None
    ok = True
    for step in range(2):
        rec = dp_tr.train_step(dp_tr.build_train_batch(trajs[a:b]))
        if rank == 0:
            ref = ref_tr.train_step(ref_tr.build_train_batch(trajs))
            for k, v in ref.items():
                if isinstance(v, float):
                    good = abs(rec[k] - v) <= 1e-5 * max(1.0, abs(v))
                elif k in ("n_real", "n_imagined"):
                    good = True  # per-rank counts (the reference counts the whole batch)
                else:
                    good = rec[k] == v
                if not good:
                    print(f"step {step} record {k}: dp {rec[k]} vs single {v}")
                    ok = False
            p_dp = dp_tr.params.p[dp_tr.params.cur][:dp_tr.layout.total].cpu()
            p_ref = ref_tr.params.p[ref_tr.params.cur].cpu()
            n = min(p_dp.numel(), p_ref.numel())
            diff = (p_dp[:n] - p_ref[:n]).abs()
            frac_exact = float((diff <= 1e-6).double().mean())
            print(f"step {step}: max|dp-single| {float(diff.max()):.3g}, "
                  f"fraction within 1e-6: {frac_exact:.5f}")
            if float(diff.max()) > 2 * 3e-4 + 1e-6 or frac_exact < 0.99:
                ok = False
    flag = torch.tensor([1.0 if ok else 0.0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("DP PARITY OK" if flag.item() == 1.0 else "DP PARITY FAILED")
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1.0 else 1)


if __name__ == "__main__":
    main()
