"""Data-parallel (ZeRO-2) host logic on CPU with the gloo backend, world_size 2.

The GPU kernels are not involved: Adam is injected as a float64 torch
function so the ZeRO-2 plumbing (shard bounds, padding, reduce-scatter,
per-shard Adam with the policy/value group split, all-gather) is checked
against a single-process Adam over the summed gradients.  The end-to-end
multi-GPU parity check (R-rank step == one-process step on the concatenated
batch) is tests/dp_gpu_check.py, run by test_dp_gpu_two_ranks on >= 2 GPUs.
"""

from __future__ import annotations

import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def torch_adam(p_in, g, m_in, v_in, p_out, m_out, v_out, n0, hyp, skip, bad):
    """float64 restatement of accel_adam on CPU tensors (numerics.py:95-126);
    hyp = (group 0, group 1) host tuples."""
    g0, g1 = hyp
    if int(skip[0]):
        return
    n = p_in.numel()
    for lo, hi, hp in ((0, n0, g0), (n0, n, g1)):
        if hi <= lo:
            continue
        lr, b1, b2, eps, bc1, bc2 = hp
        gg = g[lo:hi].double()
        m = b1 * m_in[lo:hi].double() + (1 - b1) * gg
        v = b2 * v_in[lo:hi].double() + (1 - b2) * gg * gg
        w = p_in[lo:hi].double() - lr * (m / bc1) / (torch.sqrt(v / bc2) + eps)
        p_out[lo:hi] = w.float()
        m_out[lo:hi] = m.float()
        v_out[lo:hi] = v.float()


def _run_gloo(target, world: int, attempts: int = 3) -> dict:
    """Spawn `world` gloo ranks running target(rank, world, port, queue) and
    collect one (rank, ...) tuple per rank.  A rendezvous port picked by
    _free_port can be taken by another process before the ranks bind it, so a
    failed launch is retried on a fresh port."""
    import queue as _queue
    ctx = mp.get_context("spawn")
    last = None
    for _ in range(attempts):
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
        for p in procs:
            p.start()
        res = {}
        try:
            for _ in range(world):
                item = q.get(timeout=120)
                res[item[0]] = item[1:]
        except (_queue.Empty, OSError) as e:  # a rank died (e.g. a port race): retry
            last = e
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
        if len(res) == world and all(p.exitcode == 0 for p in procs):
            return res
        last = last or RuntimeError(f"exit codes {[p.exitcode for p in procs]}")
    raise AssertionError(f"gloo ranks failed after {attempts} attempts: {last}")


def _layout(world):
    from paper_2603_18464_b200.params import Dims, FlatLayout
    return FlatLayout(Dims(obs_dim=5, hidden=3, chunk_len=2, n_actions=3, n_steps=4,
                           mlp_hidden=2), pad_to=4 * world)


def _init_params(params, seed):
    gen = torch.Generator().manual_seed(seed)
    total = params.layout.total
    params.p[0].copy_(torch.randn(total, generator=gen))
    m0 = torch.randn(total, generator=gen).abs() * 1e-3
    v0 = torch.rand(total, generator=gen) * 1e-4
    return m0, v0


HYP = ((3e-4, 0.9, 0.999, 1e-8, 1 - 0.9, 1 - 0.999), (1e-3, 0.8, 0.99, 1e-8, 1 - 0.8, 1 - 0.99))


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_18464_b200.dp import DataParallel
        from paper_2603_18464_b200.params import DeviceParams
        dp = DataParallel(adam_fn=torch_adam)
        layout = _layout(world)
        params = DeviceParams(layout, "cpu", shard=(rank, world))
        m0, v0 = _init_params(params, seed=5)
        for (s_lo, s_hi, s_off, _) in params.shard_slices():  # this rank's moment slices
            params.m[0][s_off:s_off + s_hi - s_lo] = m0[s_lo:s_hi]
            params.v[0][s_off:s_off + s_hi - s_lo] = v0[s_lo:s_hi]
        grads = [torch.randn(layout.total, generator=torch.Generator().manual_seed(100 + r))
                 for r in range(world)]
        params.g.copy_(grads[rank])
        skip = torch.zeros(1, dtype=torch.int32)
        bad = torch.zeros(1, dtype=torch.int32)
        dp.begin_step(params, HYP, skip, bad)
        for b in (3, 2, 1, 0):  # buckets in backward order, as the trainer fires them
            dp.bucket_ready(b)
        dp.finish_step()
        params.flip()  # the trainer adopts the new generation
        try:
            params.moments_to_host()
            stale_raised = False
        except Exception:
            stale_raised = True
        dp.gather_moments(params)
        mp_, vp_ = params.moments_to_host()
        # C1: pooled statistics from per-rank sums
        x = torch.arange(10, dtype=torch.float64) * (rank + 1)
        sums = torch.tensor([x.sum().item(), (x * x).sum().item(), float(x.numel())],
                            dtype=torch.float64)
        dp.all_reduce_sum(sums)
        mx = torch.tensor([float(rank)], dtype=torch.float64)
        dp.all_reduce_max(mx)
        # C5: token sums and maxima in one collective
        ls = torch.tensor([1.5 * (rank + 1), -2.0 * rank], dtype=torch.float64)
        lm = torch.tensor([float(rank), -float(rank)], dtype=torch.float64)
        dp.all_reduce_sum_max(ls, lm)
        out_q.put((rank, params.p[1].clone(), sums, mx, dp.global_counts(7 + rank, 3),
                   params._moments_host[1][0].copy(), params._moments_host[1][1].copy(),
                   params.m[1].numel(), stale_raised, ls, lm))
    finally:
        dist.destroy_process_group()


def test_zero2_adam_and_collectives_gloo():
    """Bucketed ZeRO-2 on 2 gloo ranks == one Adam over the summed gradients;
    moments are held only for each rank's slices and are readable only after
    the collective gather at the current generation."""
    from paper_2603_18464_b200.params import DeviceParams
    world = 2
    res = _run_gloo(_worker, world)
    layout = _layout(world)
    ref = DeviceParams(layout, "cpu")
    m0, v0 = _init_params(ref, seed=5)
    ref.m[0].copy_(m0)
    ref.v[0].copy_(v0)
    g_sum = sum(torch.randn(layout.total, generator=torch.Generator().manual_seed(100 + r))
                for r in range(world))
    torch_adam(ref.p[0], g_sum, ref.m[0], ref.v[0], ref.p[1], ref.m[1], ref.v[1], layout.n_policy,
               HYP, torch.zeros(1, dtype=torch.int32), None)
    for r in range(world):
        torch.testing.assert_close(res[r][0], ref.p[1], rtol=0, atol=1e-7)
        torch.testing.assert_close(torch.from_numpy(res[r][4]), ref.m[1], rtol=0, atol=1e-7)
        torch.testing.assert_close(torch.from_numpy(res[r][5]), ref.v[1], rtol=0, atol=1e-9)
        assert res[r][6] == layout.total // world  # moments: this rank's slices only
        assert res[r][7]  # reading unsharded moments without the gather raises
        xs = [torch.arange(10, dtype=torch.float64) * (q_ + 1) for q_ in range(world)]
        allx = torch.cat(xs)
        assert res[r][1].tolist() == pytest.approx([allx.sum().item(), (allx * allx).sum().item(),
                                                    20.0])
        assert res[r][2].item() == world - 1
        assert res[r][3] == (7 + 8, (7 + 8) * 3)
        assert res[r][8].tolist() == [1.5 + 3.0, -2.0]
        assert res[r][9].tolist() == [1.0, 0.0]
    # every bucket is a whole number of 16-byte rank slices
    for lo, hi, _ in layout.buckets:
        assert (hi - lo) % (4 * world) == 0


def test_partition_trajectories_is_contiguous_and_balanced():
    from paper_2603_18464_b200.dp import partition_trajectories
    rng = np.random.default_rng(0)
    lens = rng.integers(1, 521, size=1000)
    for world in (1, 2, 4, 8):
        spans = [partition_trajectories(lens, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == 1000
        for a, b in zip(spans, spans[1:]):
            assert a[1] == b[0]
        loads = [int(lens[a:b].sum()) for a, b in spans]
        assert max(loads) - min(loads) <= 2 * 520


@pytest.mark.gpu
def test_dp_gpu_two_ranks():
    """R=2 ZeRO-2 step over NCCL == one-process step on the concatenated batch."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(ROOT / "tests" / "dp_gpu_check.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "DP PARITY OK" in res.stdout


def _bcast_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_18464_b200.params import Dims, FlatLayout
        from paper_2603_18464_b200.publish import POLICY, VersionedWeights, broadcast_policy
        from paper_2603_18464_b200.types import (ModelBundle, PolicyConfig, PolicyModel,
                                                 ValueConfig, ValueHead)
        rng = np.random.default_rng(0)  # same template on every rank
        pc = PolicyConfig(obs_dim=9, hidden_dim=8, chunk_len=3, n_actions=5, vocab_size=5,
                          action_start=0)
        tpl = ModelBundle(PolicyModel.init(rng, pc), ValueHead.init(rng, ValueConfig(8, 12, 4)))
        layout = FlatLayout(Dims.from_models(tpl.policy, tpl.value), pad_to=4)
        snap = None
        if rank == 0:
            flat = torch.from_numpy(np.random.default_rng(1).normal(size=layout.total)
                                    .astype(np.float32))
            snap = VersionedWeights(POLICY, 17, flat=flat, split=layout.split, template=tpl)
        got = broadcast_policy(snap, tpl, src=0)
        q.put((rank, got.version, {k: v.copy() for k, v in got.policy.params.tensors.items()},
               {k: v.copy() for k, v in got.value.params.tensors.items()}))
    finally:
        dist.destroy_process_group()


def test_policy_snapshot_broadcast_gloo():
    """a versioned snapshot reaches every rank intact."""
    res = _run_gloo(_bcast_worker, 2)
    assert res[0][0] == res[1][0] == 17
    for k in res[0][1]:
        np.testing.assert_array_equal(res[0][1][k], res[1][1][k])
    for k in res[0][2]:
        np.testing.assert_array_equal(res[0][2][k], res[1][2][k])
