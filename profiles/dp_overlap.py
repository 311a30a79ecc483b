"""ZeRO-2 overlap timeline (run under torchrun, N GPUs): one cfg4 trainer step
(OpenVLA-7B-shaped heads, 64 x 128 transitions per GPU) with CUDA events on
the main stream (step start, each gradient bucket ready, step end) and on the
DataParallel side stream (each bucket's reduce-scatter + Adam + all-gather).
Rank 0 prints one JSON object: times in ms from the step start; `overlap` is
the fraction of side-stream time that ran before the backward finished.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        profiles/dp_overlap.py > gpurun_out/dp_overlap.json
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2603_18464_b200.dp import DataParallel  # noqa: E402
from paper_2603_18464_b200.params import BUCKETS  # noqa: E402
from paper_2603_18464_b200.trainer import Trainer, TrainerConfig  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    bench._WL["name"] = os.environ.get("WORKLOAD", "cfg4")
    comm = DataParallel()
    lens, done = bench.lengths_for(0, rank, 64 if bench._WL["name"] == "cfg4" else 4096, 520)
    n = len(lens)
    tr = Trainer(bench.make_bundle(0, 522), TrainerConfig(), comm=comm)
    inputs = bench.device_inputs(lens, done, rank, dev)
    bver = np.zeros(n, dtype=np.int64)

    def step():
        return tr.train_step(tr.build_from_device(inputs, n_real=n, behavior_version=bver))

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    comm.timeline = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step()
    e1.record()
    torch.cuda.synchronize()
    names = ["+".join(b[:2]) + ("..." if len(b) > 2 else "") for b in BUCKETS]
    rows, busy, before = [], 0.0, 0.0
    # the backward ends when the last bucket (layer 0) is ready
    bwd_end = max(e0.elapsed_time(ev) for _, ev, _, _ in comm.timeline)
    for b, ev, t0, t1 in comm.timeline:
        s, e = e0.elapsed_time(t0), e0.elapsed_time(t1)
        rows.append({"bucket": names[b], "floats": tr.layout.buckets[b][1] - tr.layout.buckets[b][0],
                     "ready_ms": e0.elapsed_time(ev), "comm_start_ms": s, "comm_end_ms": e})
        busy += e - s
        before += max(0.0, min(e, bwd_end) - s)
    out = {"world": world, "workload": bench._WL["name"], "step_ms": e0.elapsed_time(e1),
           "backward_end_ms": bwd_end, "buckets": rows,
           "comm_ms": busy, "overlap": before / busy if busy else 0.0}
    if rank == 0:
        print(json.dumps(out))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
