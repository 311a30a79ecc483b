"""Trainer-step benchmark (driver contract).

One step = `Trainer.build_train_batch` + `Trainer.train_step` (revaluation,
segmented GAE, pooled normalization, behavior log-probs, policy + value
forward/backward with the fused GIPO token loss, Adam) over one synthetic
cfg2 batch per GPU:
  4096 LIBERO-Long-like ragged trajectories (50% successes, T ~ U[1,520],
  done; 50% truncations at T = 520), K = 7 action tokens x A = 256 bins,
  policy D = 64, obs 195, value head n_steps 522 / mlp 32, random init.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`value`  = transitions of all ranks / device-timed seconds (inputs resident in HBM).
`e2e`    = the same step through the public API from pinned HOST buffers, H2D of
           every input and the D2H of the record inside the timed region.
`--impl reference` times the float64 CPU restatement of the reference trainer
(oracle/, the reference itself is pure NumPy) on the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOAD_CFG4 = ("cfg4 trainer step: OpenVLA-7B-shaped policy/value heads (obs = hidden = 4096, "
                 "K=7, A=256 slim head, value mlp 32), 64 trajectories x 128 steps per GPU, GIPO "
                 "trust arm, revalue on")
METRIC = "trainer transitions/sec"
UNIT = "transitions/s"
WORKLOAD = ("cfg2 trainer step: LIBERO-Long ragged trajectories (50% success T~U[1,520] done, "
            "50% truncated T=520), K=7, A=256, D=64, obs 195, GIPO trust arm, revalue on")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n-traj", type=int, default=4096, help="trajectories per GPU")
    ap.add_argument("--horizon", type=int, default=520)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-traj", type=int, default=64, help="cpu_baseline sample size")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dz", default="recompute", choices=["store", "recompute"],
                    help="store: K4 writes dz rows; recompute: token scalars + frame-blocked "
                         "recomputing grouped sums")
    ap.add_argument("--block-chunks", type=int, default=64)
    ap.add_argument("--workload", default="cfg2", choices=["cfg2", "cfg4"],
                    help="cfg2: LIBERO-Long ragged batch, D = 64 (the headline); cfg4: "
                         "OpenVLA-7B-shaped heads O = D = 4096, 64 x 128 transitions per GPU")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the cfg1 / cfg4 / drop-in-call lines (extra keys)")
    return ap.parse_args()


_WL = {"name": "cfg2"}


class workload:
    """Temporarily switch the workload the helpers below describe."""

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        self.prev, _WL["name"] = _WL["name"], self.name

    def __exit__(self, *exc):
        _WL["name"] = self.prev
        return False


def dims():
    if _WL["name"] == "cfg4":  # OpenVLA-7B-shaped heads
        return dict(K=7, A=256, D=4096, O=4096, H=32)
    return dict(K=7, A=256, D=64, O=195, H=32)  # cfg1 and the cfg2 headline


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def sfu_rate(peaks: dict) -> float:
    """ex2 per second: 16 SFU ops per clock per SM (B200), 148 SMs, max SM clock."""
    return 16 * 148 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6


def trainer_roofline(N: int, n: int, peaks: dict, recompute: bool) -> dict:
    """T_roof = sum over the step's stages of max(bytes / BW, flops / F_peak,
    ex2 / SFU rate), with each stage's algorithmic bytes (fp32
    activations, i32 indices), for the GEMMs 3xTF32 tensor flops against half
    the measured bf16 dense rate, and for the softmax passes one ex2 per logit
    and pass on the SFU.  Passes a fused design avoids (the frame finiteness
    read, the tanh derivatives) are not counted.  recompute: the dz-free loss
    path (token scalars + frame-blocked recomputing grouped sums).  roofline
    time / achieved time is the trainer's fraction of roofline."""
    d = dims()
    K, A, D, O, H = d["K"], d["A"], d["D"], d["O"], d["H"]
    M, F = N * K, N + n
    bw = float(peaks["hbm_gbs"]) * 1e9
    tf32 = 0.5 * float(peaks.get("bf16_tflops_sustained", 1420.9)) * 1e12
    sfu = sfu_rate(peaks)
    gemm = [  # (rows, K, N): backbone, values (revaluation), head, value head, backward
        (F, O, D), (F, D, D), (F, D, H), (F, D, A), (F, A, D), (F, D, D), (F, H, D),
        (F, A, D), (F, D, D), (F, O, D), (F, H, D)]
    stages = {  # (bytes, tensor flops, SFU ex2)
        "token_logp": (M * (4 * A + 8), 0.0, M * A),
        "gae": (20 * N + 13 * n, 0.0, 0.0),
        "loss_fact": (M * (16 + 12) + N * (8 * A + 8) if recompute
                      else M * (4 * A + 12) + N * (8 * A + 8), 0.0, 2 * M * A),
        "grouped_sums": (F * 4 * A + 24 * M, 0.0, M * A) if recompute
        else (M * (4 * A + 4), 0.0, 0.0),
        "gemms": (sum(4 * r * (k + c) for r, k, c in gemm),
                  sum(3 * 2 * r * k * c for r, k, c in gemm), 0.0),
        "value_head": (4 * F * (2 * D + D) + 4 * 3 * F * H + 4 * F * (3 * D + 2) + 4 * F * (2 * D + 2),
                       0.0, 0.0),
    }
    st = {k: max(b / bw, f / tf32, x / sfu) for k, (b, f, x) in stages.items()}
    return {"t_roof_ms": sum(st.values()) * 1e3, "bytes": sum(v[0] for v in stages.values()),
            "tensor_flops": sum(v[1] for v in stages.values()),
            "sfu_ex2": sum(v[2] for v in stages.values()),
            "stages_ms": {k: 1e3 * v for k, v in st.items()},
            "loss_path": "dz-free (token scalars + frame-blocked recompute)" if recompute
            else "dz stored and re-read by the grouped sums",
            "peak_source": "MEASURED_PEAKS.json hbm_gbs; TF32 = bf16 dense sustained / 2; "
                           "SFU = 16 ex2/clk/SM x 148 SMs x sm_max_mhz"}


def make_bundle(seed: int, n_steps: int):
    from paper_2603_18464_b200.types import (ModelBundle, PolicyConfig, PolicyModel, ValueConfig,
                                             ValueHead)
    d = dims()
    rng = np.random.default_rng(np.random.SeedSequence([seed, 3]))
    pc = PolicyConfig(obs_dim=d["O"], hidden_dim=d["D"], chunk_len=d["K"], n_actions=d["A"],
                      vocab_size=32000, action_start=31744)
    vc = ValueConfig(hidden_dim=d["D"], n_steps=n_steps, mlp_hidden=d["H"])
    return ModelBundle(PolicyModel.init(rng, pc), ValueHead.init(rng, vc))


def lengths_for(seed: int, rank: int, n: int, horizon: int):
    if _WL["name"] in ("cfg1", "cfg4"):  # n (64) trajectories x 128 steps, done alternating
        return np.full(n, 128, dtype=np.int64), np.arange(n) % 2 == 0
    from paper_2603_18464_b200.workload import libero_long_lengths
    return libero_long_lengths(np.random.default_rng(np.random.SeedSequence([seed, rank, 11])), n,
                               horizon)


def device_inputs(lens, done, seed: int, device):
    """Synthetic packed batch generated directly in HBM (N(0,1) values, U[0,A) tokens)."""
    import torch
    d = dims()
    n = len(lens)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    N = int(off[-1])
    F = N + n
    steps = (np.arange(F) - np.repeat(off[:-1] + np.arange(n), lens + 1)).astype(np.int32)
    from paper_2603_18464_b200 import ops
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    f32 = torch.float32
    frames = ops.alloc_pitched(F, d["O"], device)  # aligned rows: the GEMMs stream via TMA
    frames.normal_(generator=g)
    return {
        "traj_off": torch.from_numpy(off).to(device),
        "frames": frames,
        "steps": torch.from_numpy(steps).to(device),
        "values": torch.randn(F, generator=g, device=device, dtype=f32),
        "tokens": torch.randint(0, d["A"], (N * d["K"],), generator=g, device=device,
                                dtype=torch.int32),
        "rewards": torch.randn(N, generator=g, device=device, dtype=f32),
        "mu": torch.randn(N * d["K"], d["A"], generator=g, device=device, dtype=f32),
        "done": torch.from_numpy(np.asarray(done, dtype=np.uint8)).to(device),
    }


class ClockSampler:
    """nvidia-smi clocks / throttle reasons at 50 ms intervals.  start() launches the
    poller early (its start-up takes ~0.1 s); the `with` block marks the timed
    region, and only samples stamped inside it (+ one interval) are summarised."""
    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        if self.proc is None:
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                     "-lms", "50", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                    stderr=subprocess.DEVNULL, text=True)
            except OSError:
                self.proc = None
        return self

    def __enter__(self):
        import datetime
        self.start()
        self.t0 = datetime.datetime.now()
        return self

    def __exit__(self, *exc):
        import datetime
        self.t1 = datetime.datetime.now()
        self.summary = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if self.proc is None:
            return False
        time.sleep(0.12)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        lo = self.t0 - datetime.timedelta(milliseconds=10)
        hi = self.t1 + datetime.timedelta(milliseconds=60)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f")
                if not lo <= ts <= hi:
                    continue
                sm.append(float(parts[2]))
                smax.append(float(parts[3]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[6:10]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if sm:
            self.summary = {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)),
                            "reasons": sorted(reasons), "samples": len(sm)}
        return False


def gae_sweep(dev, peak: float, sizes=(4096, 16384, 65536), reps: int = 20,
              frame_of: bool = False) -> dict:
    """cfg2 (BASELINE.json configs[1]): K1 over LIBERO-Long mixes of 4K-64K
    trajectories (up to 25.5 M transitions, 0.5 GB), device-resident inputs,
    CUDA events over `reps` back-to-back launches (inputs > L2 at 16K+)."""
    import torch

    from paper_2603_18464_b200 import ops
    from paper_2603_18464_b200.workload import libero_long_lengths

    rows = []
    for n, pure in [(n, False) for n in sizes] + [(sizes[-1], True)]:
        # (the last row: SURVEY 8(d)'s pure U[1, 520] length variant)
        lens, dn = libero_long_lengths(np.random.default_rng(n), n, pure_uniform=pure)
        off = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(lens, out=off[1:])
        N = int(off[-1])
        g = torch.Generator(device=dev).manual_seed(n)
        r = torch.randn(N, device=dev, generator=g)
        v = torch.randn(N + n, device=dev, generator=g)
        t_off = torch.from_numpy(off).to(dev)
        d_dev = torch.from_numpy(dn.astype(np.uint8)).to(dev)
        adv, ret = torch.empty_like(r), torch.empty_like(r)
        fo = torch.empty(N, dtype=torch.int32, device=dev)
        sums = torch.empty(4, dtype=torch.float64, device=dev)

        def run():
            ops.gae_segmented(r, v, t_off, d_dev, 0.99, 0.95, adv=adv, ret=ret,
                              frame_of=fo if frame_of else None, sums=sums)

        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        byt = 16 * N + 13 * n + (4 * N if frame_of else 0)  # SURVEY 8(d) (+ frame_of)
        rows.append({"trajectories": n, "lengths": "U[1,520]" if pure else "LIBERO-Long mix",
                     "transitions": N, "bytes_per_launch": byt,
                     "ms_per_launch": ms, "achieved": byt / ms / 1e6,
                     "frac": byt / ms / 1e6 / peak})
        del r, v, adv, ret, fo
    return {"kernel": "accel_gae_segmented (K1: warp per trajectory range + pooled-statistics "
                      "partials)", "unit": "GB/s", "peak": peak,
            "bytes": "16 N + 13 n (SURVEY 8(d): r, v in; adv, ret out; offsets, done, "
                     "bootstrap v)" + (" + 4 N frame_of" if frame_of else ""),
            "config": "cfg2: LIBERO-Long mix (50% done T~U[1,520], 50% truncated at 520)",
            "rows": rows}


def cpu_baseline(bundle, inputs_host, lens, done, n_cpu: int, n_steps: int, reps: int = 3,
                 threads: int | None = None):
    """The float64 oracle (reference restatement) on a bounded sample of the
    same batch, host cores: best of `reps` timed build_train_batch +
    train_step after one warm-up, OpenBLAS limited to `threads` (default all)."""
    from threadpoolctl import threadpool_limits

    from oracle.trainer_ref import OracleConfig, OracleTrainer
    from paper_2603_18464_b200.workload import PackedBatch, unpack_trajectories
    d = dims()
    n = min(n_cpu, len(lens))
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens[:n], out=off[1:])
    N = int(off[-1])
    F = N + n
    pb = PackedBatch(traj_off=off, frames=inputs_host["frames"][:F], steps=inputs_host["steps"][:F],
                     values=inputs_host["values"][:F],
                     tokens=inputs_host["tokens"][:N * d["K"]].reshape(N, d["K"]),
                     rewards=inputs_host["rewards"][:N],
                     mu=inputs_host["mu"][:N * d["K"]].reshape(N, d["K"], d["A"]),
                     done=np.asarray(done[:n], dtype=np.uint8), real=np.ones(n, np.uint8),
                     behavior_version=np.zeros(n, np.int64))
    trajs = unpack_trajectories(pb)
    cores = threads or os.cpu_count() or 1
    best = None
    with threadpool_limits(limits=cores):
        for _ in range(reps + 1):
            orc = OracleTrainer(bundle.policy.params.tensors, bundle.value.params.tensors,
                                d["A"], n_steps, OracleConfig())
            t0 = time.perf_counter()
            b = orc.build_train_batch(trajs)
            orc.train_step(b)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
    return {"value": N / best, "unit": UNIT, "cores": cores, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"{n} trajectories / {N} transitions of the same workload, oracle "
                      f"build_train_batch + train_step (float64 NumPy, OpenBLAS {cores} "
                      f"thread{'s' if cores > 1 else ''}), best of {reps} after 1 warm-up"}


def timed_steps(fn, steps: int, warmup: int) -> float:
    """ms per call of fn over `steps` calls after `warmup`, CUDA events."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def run_cfg1(dev, seed: int, steps: int, warmup: int, cpu: bool) -> dict:
    """BASELINE configs[0] (cfg1: 64 x 128, K = 7, A = 256, D = 64, obs 195) on
    one GPU, eager and as a CUDA-graph replay of the whole step
    (Trainer.capture_step), beside the float64 CPU oracle on the identical
    batch at 1 thread and at every host core (best of 3)."""
    import torch

    from paper_2603_18464_b200 import _lib
    from paper_2603_18464_b200.trainer import Trainer, TrainerConfig
    with workload("cfg1"):
        lens, done = lengths_for(seed, 0, 64, 128)
        n, N = len(lens), int(lens.sum())
        bundle = make_bundle(seed, 130)
        inputs = device_inputs(lens, done, seed + 17, dev)
        bver = np.zeros(n, dtype=np.int64)
        tr = Trainer(bundle, TrainerConfig())
        c0 = _lib.launch_count()
        tr.train_step(tr.build_from_device(inputs, n_real=n, behavior_version=bver))
        launches = _lib.launch_count() - c0
        ms_eager = timed_steps(
            lambda: tr.train_step(tr.build_from_device(inputs, n_real=n, behavior_version=bver)),
            steps, warmup)
        graphed = Trainer(make_bundle(seed, 130), TrainerConfig())
        cap = graphed.capture_step(inputs, n, bver)
        ms_graph = timed_steps(cap.run, steps, max(warmup, 2))
        out = {"workload": "cfg1: 64 trajectories x 128 steps (N = 8192, M = 57,344 tokens), "
                           "K=7, A=256, D=64, obs 195, GIPO trust arm, revalue on",
               "value": N / (ms_graph / 1e3), "unit": UNIT, "ms_per_step": ms_graph,
               "ms_per_step_eager": ms_eager, "value_eager": N / (ms_eager / 1e3),
               "libaccel_launches_per_step": int(launches), "cuda_graph": True,
               "host_syncs_per_step": 1}
        if cpu:
            host = {k: v.cpu().numpy() for k, v in inputs.items()}
            host["frames"] = np.ascontiguousarray(host["frames"])
            for thr in (1, None):
                c = cpu_baseline(bundle, host, lens, done, n, 130, reps=3, threads=thr)
                out["cpu_1thread" if thr == 1 else "cpu_all_cores"] = c
        return out


def run_cfg4(dev, seed: int, rank: int, steps: int, warmup: int, comm,
             strong: bool = False) -> dict:
    """BASELINE configs[3] (cfg4: OpenVLA-7B-shaped heads, O = D = 4096, 64 x 128
    transitions per GPU) -- ZeRO-2 data parallel under torchrun (weak scaling;
    strong=True: the 64 x 128 global batch split over the ranks); every GEMM on
    the wide tcgen05 kernel (csrc/tc_wide.cu)."""
    import torch
    import torch.distributed as dist

    from paper_2603_18464_b200.trainer import Trainer, TrainerConfig
    world = comm.world if comm is not None else 1
    with workload("cfg4"):
        lens, done = lengths_for(seed, rank, 64 // world if strong else 64, 128)
        n, N = len(lens), int(lens.sum())
        tr = Trainer(make_bundle(seed, 522), TrainerConfig(), comm=comm)
        inputs = device_inputs(lens, done, seed * 1000 + rank, dev)
        bver = np.zeros(n, dtype=np.int64)
        if comm is not None:
            dist.barrier()
        ms = timed_steps(
            lambda: tr.train_step(tr.build_from_device(inputs, n_real=n, behavior_version=bver)),
            steps, warmup)
        t = torch.tensor([ms, float(N)], dtype=torch.float64, device=dev)
        if comm is not None:
            mx = t[:1].clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            ms, tot = float(mx.item()), float(t[1].item())
        else:
            tot = float(N)
        del tr, inputs
        torch.cuda.empty_cache()
        return {"workload": WORKLOAD_CFG4 if not strong else
                WORKLOAD_CFG4.replace("64 trajectories x 128 steps per GPU",
                                      "64 x 128 global batch split over the GPUs"),
                "value": tot / (ms / 1e3), "unit": UNIT,
                "ms_per_step": ms, "n_gpus": world, "scaling": "strong" if strong else "weak",
                "parallelism": f"dp{world} (ZeRO-2)" if world > 1 else "single",
                "gemms": "accel_tc_gemm_wide (tf32 + bf16-pair tcgen05), no cuBLAS on the step"}


def e2e_api(tr, seed: int, n_traj: int = 256, reps: int = 3) -> dict:
    """The drop-in call itself: Trainer.build_train_batch(list[Trajectory]) +
    train_step on reference-style float64 Trajectory objects (a sample of the
    headline workload), wall clock per step -- the threaded pack into pinned
    staging, the H2D upload, the device build and step, the record readback."""
    from paper_2603_18464_b200.workload import synthetic_packed, unpack_trajectories
    d = dims()
    lens, done = lengths_for(seed + 7, 0, n_traj, 520)
    pb = synthetic_packed(seed + 7, lens, done, d["K"], d["A"], d["O"])
    trajs = unpack_trajectories(pb)  # float64 arrays, as the reference's Trajectory holds
    del pb
    N = int(lens.sum())
    tr.train_step(tr.build_train_batch(trajs))
    best, tot = None, 0.0
    for _ in range(reps):
        t0 = time.perf_counter()
        tr.train_step(tr.build_train_batch(trajs))
        dt = time.perf_counter() - t0
        tot += dt
        best = dt if best is None else min(best, dt)
    f64_bytes = sum(t.observations.nbytes + t.behavior_logits.nbytes + t.rewards.nbytes
                    + t.values.nbytes + t.tokens.nbytes + t.steps.nbytes for t in trajs)
    return {"value": N / (tot / reps), "unit": UNIT, "ms_per_step": 1e3 * tot / reps,
            "best_ms": 1e3 * best, "sample": f"{n_traj} trajectories / {N} transitions",
            "call": "Trainer.build_train_batch(list[Trajectory float64]) + Trainer.train_step",
            "host_input_bytes_f64": int(f64_bytes)}


def loss_sweep(dev, seed: int, sfu_peak: float, sizes=(16, 64, 256, 1024, 4096)) -> dict:
    """SURVEY 8(d) loss-kernel sweep: the dz-free loss kernel (K4) and the grouped
    recompute over token counts from ~50 K to ~11 M (cfg2 LIBERO-Long mixes of
    16 ... 4096 trajectories), in-step CUDA-event times (mean of 3 steps)."""
    import torch

    from paper_2603_18464_b200.trainer import Trainer, TrainerConfig
    d = dims()
    rows = []
    for nt in sizes:
        lens, done = lengths_for(seed + nt, 0, nt, 520)
        N = int(lens.sum())
        M = N * d["K"]
        tr = Trainer(make_bundle(seed, 522), TrainerConfig())
        inputs = device_inputs(lens, done, seed + 31 * nt, dev)
        bver = np.zeros(len(lens), dtype=np.int64)
        for _ in range(2):
            tr.train_step(tr.build_from_device(inputs, n_real=len(lens), behavior_version=bver))
        tr.profile_events = []
        for _ in range(3):
            tr.train_step(tr.build_from_device(inputs, n_real=len(lens), behavior_version=bver))
        torch.cuda.synchronize()
        kern = {}
        for name, a, b in tr.profile_events:
            kern.setdefault(name, []).append(a.elapsed_time(b))
        t_loss = float(np.mean(kern.get("token_loss", [float("nan")])))
        t_grp = float(np.mean(kern.get("group_sum", [float("nan")])))
        ex2 = 2 * M * d["A"]
        rows.append({"trajectories": nt, "transitions": N, "tokens": M,
                     "loss_ms": t_loss, "loss_tex2_s": ex2 / t_loss / 1e9,
                     "loss_sfu_frac": ex2 / t_loss / 1e9 / sfu_peak,
                     "recompute_ms": t_grp,
                     "recompute_sfu_frac": (M * d["A"]) / t_grp / 1e9 / sfu_peak})
        del tr, inputs
        torch.cuda.empty_cache()
    return {"kernels": "token_loss_fact2 (K4, dz-free) + fact_group_sum2 (grouped recompute)",
            "bound": "sfu (2 ex2 per logit in K4, 1 in the recompute); latency-bound in practice",
            "peak_tex2_s": sfu_peak, "rows": rows}


def run_reference(args, rank: int, world: int):
    """--impl reference: the CPU restatement of the reference trainer (rank 0)."""
    if rank != 0:
        return
    import torch  # noqa: F401  (device-free: generation on the host)
    d = dims()
    lens, done = lengths_for(args.seed, 0, args.n_traj, args.horizon)
    n_steps = 522 if args.workload == "cfg4" else args.horizon + 2
    bundle = make_bundle(args.seed, n_steps)
    from paper_2603_18464_b200.workload import synthetic_packed, unpack_trajectories
    from threadpoolctl import threadpool_limits

    from oracle.trainer_ref import OracleConfig, OracleTrainer
    n = min(16, args.n_traj)
    pb = synthetic_packed(args.seed, lens[:n], done[:n], d["K"], d["A"], d["O"])
    trajs = unpack_trajectories(pb)
    N = pb.n_transitions
    cores = os.cpu_count() or 1
    times = []
    with threadpool_limits(limits=cores):
        orc = OracleTrainer(bundle.policy.params.tensors, bundle.value.params.tensors, d["A"],
                            n_steps, OracleConfig())
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            b = orc.build_train_batch(trajs)
            orc.train_step(b)
            if i >= args.warmup:
                times.append(time.perf_counter() - t0)
    sec = float(np.sum(times)) / max(1, len(times))
    value = N / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded N(0,1) values/logits, U[0,A) tokens)",
        "config": {"workload": WORKLOAD, "sample_trajectories": n, "sample_transitions": N},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{n} trajectories / {N} transitions per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    _WL["name"] = args.workload
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_2603_18464_b200 import _lib, ops
    from paper_2603_18464_b200.trainer import Trainer, TrainerConfig

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    # keep stdout for the single JSON line: library banners (NCCL) go to stderr
    saved_stdout = os.dup(1)
    os.dup2(2, 1)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        from paper_2603_18464_b200.dp import DataParallel
        comm = DataParallel()
    d = dims()
    n_steps = 522 if args.workload == "cfg4" else args.horizon + 2
    lens, done = lengths_for(args.seed, rank, 64 if args.workload == "cfg4" else args.n_traj,
                             args.horizon)
    N = int(lens.sum())
    n = len(lens)
    M = N * d["K"]
    bundle = make_bundle(args.seed, n_steps)
    tr = Trainer(bundle, TrainerConfig(), comm=comm)
    tr.recompute_dz = args.dz == "recompute"
    tr.group_block_chunks = args.block_chunks
    inputs = device_inputs(lens, done, args.seed * 1000 + rank, dev)
    bver = np.zeros(n, dtype=np.int64)

    def step(inp):
        batch = tr.build_from_device(inp, n_real=n, behavior_version=bver)
        return tr.train_step(batch)

    clocks = ClockSampler(local).start()  # the poller is up before the timed region
    for _ in range(args.warmup):
        step(inputs)
    torch.cuda.synchronize()

    # ---- device-resident timed region -------------------------------------------
    tr.profile_events = []
    launches0 = _lib.launch_count()
    if comm is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with clocks:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            rec = step(inputs)
        e1.record()
        torch.cuda.synchronize()
    if comm is not None:
        dist.barrier()
    launches = _lib.launch_count() - launches0
    ms = e0.elapsed_time(e1) / args.steps
    kern = {}
    for name, a, b in tr.profile_events:
        kern.setdefault(name, []).append(a.elapsed_time(b))
    tr.profile_events = None
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    tot = torch.tensor([float(N)], dtype=torch.float64, device=dev)
    if comm is not None:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    ms = float(ms_t.item())
    value = float(tot.item()) / (ms / 1e3)

    # ---- e2e: public API from pinned host buffers --------------------------------
    e2e = None
    host = {k: v.cpu().pin_memory() if k != "traj_off" else v.cpu() for k, v in inputs.items()}
    if not args.no_e2e:
        # every step copies its own inputs from pinned host memory and reads its
        # record back; two device input sets and a copy stream let step i + 1's
        # upload run under step i's kernels (the copy is still inside the timed
        # region of every step -- the PCIe link is the bound)
        h2d = sum(v.numel() * v.element_size() for v in host.values())
        bufs, stagings = [], []
        for _ in range(2):
            b = {k: torch.empty_like(v, device=dev) for k, v in host.items()}
            stagings.append(b["frames"])  # contiguous landing buffer for the frame rows
            b["frames"] = ops.alloc_pitched(*host["frames"].shape, dev)
            bufs.append(b)
        copy_stream = torch.cuda.Stream(device=dev)

        def upload(i):
            with torch.cuda.stream(copy_stream):
                for k in host:
                    if k == "frames":  # contiguous DMA, then re-pitch on the device
                        stagings[i].copy_(host[k], non_blocking=True)
                        bufs[i][k].copy_(stagings[i])
                    else:
                        bufs[i][k].copy_(host[k], non_blocking=True)

        def run_pipelined(nsteps, start_event=None):
            ready = [torch.cuda.Event(), torch.cuda.Event()]
            free = [torch.cuda.Event(), torch.cuda.Event()]
            main = torch.cuda.current_stream()
            if start_event is not None:
                copy_stream.wait_event(start_event)
            upload(0)
            ready[0].record(copy_stream)
            for i in range(nsteps):
                b = i & 1
                if i + 1 < nsteps:  # the next step's inputs, once its buffer is free
                    if i >= 1:
                        copy_stream.wait_event(free[b ^ 1])
                    upload(b ^ 1)
                    ready[b ^ 1].record(copy_stream)
                main.wait_event(ready[b])
                step(bufs[b])
                free[b].record(main)

        run_pipelined(2)  # warm-up
        if comm is not None:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record()
        run_pipelined(args.steps, a0)
        a1.record()
        torch.cuda.synchronize()
        e_ms = torch.tensor([a0.elapsed_time(a1) / args.steps], dtype=torch.float64, device=dev)
        if comm is not None:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e_ms = float(e_ms.item())
        e2e = {"value": float(tot.item()) / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": (18 + 20) * 8, "ms_per_step": e_ms,
               "wall_ms_per_step": (time.perf_counter() - t0) * 1e3 / args.steps,
               "pipelined": "double-buffered inputs, uploads on a copy stream under the previous step"}
        del bufs, stagings

    extra = {}
    if not args.no_extra and args.workload == "cfg2":
        extra["e2e_api"] = e2e_api(tr, args.seed + rank)
        extra["cfg4"] = run_cfg4(dev, args.seed, rank, 10, 3, comm)
        if world > 1:  # cfg4 also at a fixed global batch
            extra["cfg4_strong"] = run_cfg4(dev, args.seed, rank, 10, 3, comm, strong=True)
        if rank == 0:
            extra["cfg1"] = run_cfg1(dev, args.seed, 50, 5, not args.no_cpu)
            import bench_imagine  # cfg3: the imagination step
            extra["cfg3"] = bench_imagine.run(4096, 16, 5, 16 if not args.no_cpu else 0)
        if comm is not None:
            dist.barrier()
    if rank != 0:
        if comm is not None:
            dist.destroy_process_group()
        return

    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {"hbm_gbs": 6650.0}
    tr_roof = trainer_roofline(N, n, peaks, tr.recompute_dz)
    peak = float(peaks["hbm_gbs"])
    A = d["A"]
    # factorized head (trainer default): per token dz write (4A) + token/lp_old/lp_new
    # (12); per transition the H2W row read and the g_frame row write (8A) + adv and
    # frame index (8).  DESIGN.md "Kernels / token_loss_fact".
    if not tr.factorized:
        loss_bytes = M * (8 * A + 12) + 4 * N
    elif tr.recompute_dz:  # 16 B of token scalars replace the 4A-byte dz row
        loss_bytes = M * (16 + 12) + N * (8 * A + 8)
    else:
        loss_bytes = M * (4 * A + 12) + N * (8 * A + 8)
    t_loss = float(np.mean(kern.get("token_loss", [float("nan")]))) / 1e3
    achieved = loss_bytes / t_loss / 1e9
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        tj = json.loads(tf.read_text())
        traffic = tj.get("token_loss_sc_dram_bytes_per_launch" if tr.recompute_dz
                         else "token_loss_dram_bytes_per_launch")
    t_grp = float(np.mean(kern.get("group_sum", [float("nan")]))) / 1e3
    ex2_loss = 2 * M * A  # one ex2 per logit in each of the loss kernel's two passes
    gae_bytes = 20 * N + 13 * n
    t_gae = float(np.mean(kern.get("gae", [float("nan")]))) / 1e3
    logp_bytes = M * (4 * A + 8)
    t_logp = float(np.mean(kern.get("token_logp", [float("nan")]))) / 1e3

    sweep = gae_sweep(dev, peak)
    lsweep = None
    if not args.no_extra:
        sm_mhz = (clocks.summary or {}).get("sm_max_mhz") or 1965.0
        lsweep = loss_sweep(dev, args.seed, 16 * 148 * sm_mhz * 1e6 / 1e12)
    cpu = cpu1 = None
    if not args.no_cpu:
        host_np = {k: v.numpy() for k, v in host.items()}
        cpu = cpu_baseline(bundle, host_np, lens, done, args.cpu_traj, n_steps, reps=3)
        cpu1 = cpu_baseline(bundle, host_np, lens, done, 16, n_steps, reps=3, threads=1)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded N(0,1) obs/values/rewards/behavior logits, U[0,A) tokens, "
                "random-init policy/value heads)",
        "config": {"workload": WORKLOAD if args.workload == "cfg2" else WORKLOAD_CFG4,
                   "trajectories_per_gpu": n, "transitions_per_gpu": N,
                   "tokens_per_gpu": M, "parallelism": f"dp{world}" if world > 1 else "single",
                   "l2": "inputs larger than L2 (behavior logits alone 11+ GB per GPU)"},
        "roofline": ({"kernel": "token_loss_fact2 (fused GIPO fwd+bwd, factorized head, "
                                "dz-free scalar mode)", "bound": "sfu",
                      "achieved": ex2_loss / t_loss / 1e12, "peak": sfu_rate(peaks) / 1e12,
                      "unit": "Tex2/s", "frac": ex2_loss / t_loss / sfu_rate(peaks),
                      "traffic": traffic, "ex2_per_launch": ex2_loss,
                      "ms_per_launch": t_loss * 1e3,
                      "peak_source": "16 MUFU ex2 / clk / SM x 148 SMs x sm_max_mhz (B200)",
                      "hbm": {"bytes_per_launch": loss_bytes, "achieved": achieved,
                              "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                              "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
                      "note": "dz-free loss path: the kernel writes 16 B of token scalars per "
                              "token instead of the 1 KB dz row, so its binding resource is the "
                              "SFU (2 ex2 per logit), not HBM (store mode, HBM-bound: "
                              "profiles/r1_bench_store_mode.json)"}
                     if tr.recompute_dz else
                     {"kernel": "token_loss_fact (fused GIPO fwd+bwd, factorized head)",
                      "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                      "frac": achieved / peak, "traffic": traffic,
                      "bytes_per_launch": loss_bytes, "ms_per_launch": t_loss * 1e3,
                      "peak_source": "MEASURED_PEAKS.json hbm_gbs"}),
        "roofline_group_recompute": {
            "kernel": "fact_group_sum2 (frame-blocked dz recompute + grouped sums)",
            "ms_per_launch": t_grp * 1e3,
            "bytes_per_launch": (N + n) * 4 * A + 24 * M,
            "achieved": ((N + n) * 4 * A + 24 * M) / t_grp / 1e9, "unit": "GB/s",
            "sfu_frac": M * A / t_grp / sfu_rate(peaks)} if tr.recompute_dz else None,
        "roofline_gae": {"bytes_per_launch": gae_bytes, "ms_per_launch": t_gae * 1e3,
                         "achieved": gae_bytes / t_gae / 1e9,
                         "frac": gae_bytes / t_gae / 1e9 / peak, "unit": "GB/s",
                         "note": "in-step size (32 MB, L2-resident, latency-bound); "
                                 "see gae_sweep for the cfg2 sizes"},
        "gae_sweep": sweep,
        "loss_sweep": lsweep,
        "trainer_roofline": dict(tr_roof, achieved_ms=ms, frac=tr_roof["t_roof_ms"] / ms),
        "roofline_token_logp": {"bytes_per_launch": logp_bytes, "ms_per_launch": t_logp * 1e3,
                                "achieved": logp_bytes / t_logp / 1e9,
                                "frac": logp_bytes / t_logp / 1e9 / peak, "unit": "GB/s"},
        "cpu_baseline": cpu,
        "cpu_baseline_1thread": cpu1,
        "e2e": e2e,
        **extra,
        "gpu_launches": int(launches),
        "clocks": clocks.summary,
        "last_record": {k: rec[k] for k in ("loss", "policy_loss", "value_loss", "entropy")},
    }
    sys.stdout.flush()
    os.dup2(saved_stdout, 1)
    print(json.dumps(line), flush=True)
    if comm is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
