"""Segmented GAE (K1) throughput against the HBM roofline at the cfg2 sizes.

    python profiles/gae_bench.py [n_traj ...]

LIBERO-Long mixes of n trajectories (50 % done T ~ U[1, 520], 50 % truncated
at 520); bytes per launch = 20 N + 13 n (r, v reads, adv, ret and
frame-of writes, offsets + done per trajectory; the pooled statistics are
fused).  Inputs are re-made per size, timed with CUDA events over 20 launches.
"""

import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2603_18464_b200 import ops  # noqa: E402
from paper_2603_18464_b200.workload import libero_long_lengths  # noqa: E402


def main():
    dev = torch.device("cuda")
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    rows = []
    sizes = [int(a) for a in sys.argv[1:]] or [4096, 16384, 65536]
    for n in sizes:
        lens, done = libero_long_lengths(np.random.default_rng(n), n)
        off = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(lens, out=off[1:])
        N = int(off[-1])
        r = torch.randn(N, device=dev)
        v = torch.randn(N + n, device=dev)
        traj_off = torch.from_numpy(off).to(dev)
        dn = torch.from_numpy(done.astype(np.uint8)).to(dev)
        adv, ret = torch.empty_like(r), torch.empty_like(r)
        fo = torch.empty(N, dtype=torch.int32, device=dev)
        sums = torch.empty(4, dtype=torch.float64, device=dev)
        run = lambda: ops.gae_segmented(r, v, traj_off, dn, 0.99, 0.95, adv=adv, ret=ret,
                                        frame_of=fo, sums=sums)
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        byt = 20 * N + 13 * n
        rows.append({"n_traj": n, "transitions": N, "bytes": byt, "ms": ms,
                     "GBps": byt / ms / 1e6, "frac": byt / ms / 1e6 / peak})
    print(json.dumps({"kernel": "accel_gae_segmented", "peak_gbs": peak, "rows": rows}))


if __name__ == "__main__":
    main()
