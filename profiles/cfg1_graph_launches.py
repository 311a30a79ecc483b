"""Kernel list of one cfg1 CUDA-graph replay (BASELINE configs[0]: 64 x 128).

    ncu --metrics gpu__time_duration.sum --csv --log-file out.csv \
        python profiles/cfg1_graph_launches.py
(ncu profiles graph nodes as individual kernels; the script replays 3 times.)
Without ncu it prints the replay time (CUDA events, 50 replays).
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_18464_b200.trainer import Trainer, TrainerConfig  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    with bench.workload("cfg1"):
        lens, done = bench.lengths_for(0, 0, 64, 128)
        n = len(lens)
        inputs = bench.device_inputs(lens, done, 17, dev)
        tr = Trainer(bench.make_bundle(0, 130), TrainerConfig())
        cap = tr.capture_step(inputs, n, np.zeros(n, dtype=np.int64))
        reps = int(os.environ.get("REPS", "3"))
        for _ in range(2):
            cap.run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            cap.run()
        e1.record()
        torch.cuda.synchronize()
        print(f"cfg1 graph replay: {e0.elapsed_time(e1) / reps:.3f} ms/step over {reps}")


if __name__ == "__main__":
    main()
