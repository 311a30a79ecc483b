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
    a, b = partition_trajectories(lens, world, rank)
    dp_tr = Trainer(bundle(), TrainerConfig(), comm=DataParallel())
    ref_tr = Trainer(bundle(), TrainerConfig()) if rank == 0 else None
    ok = True
    for step in range(3):
        # imagined trajectories and a behavior lag make the record's counts non-trivial
        trajs = synthetic_trajectories(np.random.default_rng(100 + step), lens,
                                       np.arange(24) % 3 == 0, 7, 256, 40, imagined_every=3,
                                       behavior_version=max(0, step - 1))
        rec = dp_tr.train_step(dp_tr.build_train_batch(trajs[a:b]))
        if rank == 0:
            ref = ref_tr.train_step(ref_tr.build_train_batch(trajs))
            for k, v in ref.items():
                if isinstance(v, float):
                    good = abs(rec[k] - v) <= 1e-5 * max(1.0, abs(v))
                else:  # n_real, n_imagined, versions, excluded tokens: exact, global
                    good = rec[k] == v
                if not good:
                    print(f"step {step} record {k}: dp {rec[k]} vs single {v}")
                    ok = False
            pd, vd = dp_tr.params.to_host()
            pr, vr = ref_tr.params.to_host()
            diffs = np.concatenate([np.abs(x[k] - y[k]).ravel() for x, y in ((pd, pr), (vd, vr))
                                    for k in y])
            frac_exact = float(np.mean(diffs <= 1e-6))
            print(f"step {step}: max|dp-single| {diffs.max():.3g}, "
                  f"fraction within 1e-6: {frac_exact:.5f}")
            if diffs.max() > 2 * 3e-4 + 1e-6 or frac_exact < 0.99:
                ok = False
    # ZeRO-2 moments: sharded on the step path, assembled by the collective gather
    dp_tr.gather_moments()
    if rank == 0:
        for mine, want in zip(dp_tr.params.moments_to_host(), ref_tr.params.moments_to_host()):
            for grp_m, grp_w in zip(mine, want):
                for k in grp_w:
                    err = float(np.max(np.abs(grp_m[k] - grp_w[k])))
                    scale = float(np.max(np.abs(grp_w[k]))) + 1e-30
                    if err > 1e-3 * scale + 1e-9:
                        print(f"moment {k}: {err:.3g} vs scale {scale:.3g}")
                        ok = False
        n_mom = dp_tr.params.m[0].numel()
        print(f"moments per rank: {n_mom} of {dp_tr.layout.total}")
        ok = ok and n_mom * world == dp_tr.layout.total
    flag = torch.tensor([1.0 if ok else 0.0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("DP PARITY OK" if flag.item() == 1.0 else "DP PARITY FAILED")
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1.0 else 1)


if __name__ == "__main__":
    main()
