"""ZeRO-2 data parallelism for the trainer step (one process per GPU).

The reference simulates data parallelism inside one process: advantage
statistics are summed over K logical shards (trainer.py:128-158, "a
simulated all-reduce") and the paper's trainer is ZeRO-2 over
NCCL.  Here every rank owns whole trajectories (the
batch is partitioned in rank order) and the step exchanges:

  C1  all_reduce(SUM) f64 {sum A, sum A^2, N, n_real, n_traj, sum lag}
      pooled normalization (Eqs. 5-7) and the global record counts
  C5  all_reduce(SUM) f64 token statistics, MAX of {ratio_max, -w_min}
      -> global included-token count m, entropy over N*K, value MSE over N
  C2  per gradient bucket (params.BUCKETS: value head, head, layer 1, layer 0,
      in the order the backward completes them): reduce_scatter(SUM) of the
      bucket into this rank's slice, Adam on the slice (this rank's parameter
      and moment shard -- the moments exist only for the slice), then
  C3  all_gather of the bucket's updated parameters.
  C2/C3 run on a side stream, each bucket as soon as its gradients are
  written, so the exchange of the value-head, head and layer-1 buckets
  overlaps the rest of the backward (the layer-0 bucket, last to finish,
  does not).  Adam there is speculative: it writes the next parameter
  generation, which the host adopts only if the step's record accepts it.

Results equal the single-process step over the concatenation of all ranks'
trajectories up to float summation order (tests/dp_gpu_check.py; the gloo
tests cover the sharding on CPU).  All collectives go through
torch.distributed (NCCL on B200s, gloo in the CPU tests).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


class DataParallel:
    def __init__(self, group=None, adam_fn=None, overlap: bool = True) -> None:
        if not dist.is_initialized():
            raise RuntimeError("DataParallel needs torch.distributed to be initialized")
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = dist.get_backend(group)
        self._adam_fn = adam_fn
        self.overlap = overlap and self.backend == "nccl"
        self._stream = None
        self._g_shard = None
        self._step = None
        self.timeline = None  # list -> (bucket, ready, start, end) CUDA events per bucket

    # -- small collectives ----------------------------------------------------------
    def all_reduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def all_reduce_max(self, t: torch.Tensor) -> torch.Tensor:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return t

    def all_reduce_sum_max(self, s: torch.Tensor, m: torch.Tensor) -> None:
        """s <- sum over ranks, m <- max over ranks (1-D float64), in ONE
        collective: both are gathered and every rank reduces the [world, n]
        rows in rank order (identical results on every rank)."""
        ns = s.numel()
        buf = torch.cat([s, m])
        if self.backend == "nccl":
            rows = torch.empty(self.world * buf.numel(), dtype=buf.dtype, device=buf.device)
            dist.all_gather_into_tensor(rows, buf, group=self.group)
            rows = rows.view(self.world, -1)
        else:
            parts = [torch.empty_like(buf) for _ in range(self.world)]
            dist.all_gather(parts, buf, group=self.group)
            rows = torch.stack(parts)
        s.copy_(rows[:, :ns].sum(0))
        m.copy_(rows[:, ns:].amax(0))

    def global_counts(self, n_local: int, k: int) -> tuple:
        t = torch.tensor([float(n_local)], dtype=torch.float64, device=self._device())
        self.all_reduce_sum(t)
        n = int(t.item())
        return n, n * k

    def _device(self):
        if self.backend == "nccl":
            return torch.device("cuda", torch.cuda.current_device())
        return torch.device("cpu")

    # -- ZeRO-2 sharding ------------------------------------------------------------
    def shard_bounds(self, total: int) -> tuple:
        """[lo, hi) of this rank's slice of a bucket of `total` (a multiple of world)."""
        if total % self.world:
            raise ValueError(f"bucket of {total} is not a multiple of world {self.world}")
        per = total // self.world
        return self.rank * per, (self.rank + 1) * per

    def reduce_scatter(self, flat: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        """Sum of the bucket `flat` over ranks, this rank's slice into `out` (C2)."""
        if self.backend == "gloo":  # gloo has no reduce_scatter_tensor on CPU
            lo, hi = self.shard_bounds(flat.numel())
            tmp = flat.clone()
            dist.all_reduce(tmp, op=dist.ReduceOp.SUM, group=self.group)
            out.copy_(tmp[lo:hi])
        else:
            dist.reduce_scatter_tensor(out, flat, op=dist.ReduceOp.SUM, group=self.group)
        return out

    def all_gather(self, shard: torch.Tensor, full: torch.Tensor) -> torch.Tensor:
        """C3: every rank's slice into `full` (rank-ordered).  NCCL runs in place
        when `shard` is this rank's slice of `full`."""
        if self.backend == "gloo":
            parts = [torch.empty_like(shard) for _ in range(self.world)]
            dist.all_gather(parts, shard.contiguous(), group=self.group)
            full.copy_(torch.cat(parts))
        else:
            dist.all_gather_into_tensor(full, shard, group=self.group)
        return full

    # -- the bucketed ZeRO-2 update -----------------------------------------------------
    def begin_step(self, params, hyp: tuple, skip, bad, adam_fn=None) -> None:
        """Arm the per-bucket exchange of one optimizer step (generation
        params.cur -> cur ^ 1).  hyp: the Adam hyperparameters handed to
        adam_fn(p_in, g, m_in, v_in, p_out, m_out, v_out, n_policy, hyp, skip,
        bad) (ops.adam_dev: a device f64[12]); skip: device int (Adam does
        nothing when set); bad: device counter of non-finite new parameters."""
        if params.world != self.world or params.rank != self.rank:
            raise ValueError("DeviceParams shard does not match the communicator")
        n_shard = params.layout.total // self.world
        if self._g_shard is None or self._g_shard.numel() != n_shard \
                or self._g_shard.device != params.g.device:
            self._g_shard = torch.empty(n_shard, dtype=params.g.dtype, device=params.g.device)
        if self.overlap and self._stream is None:
            self._stream = torch.cuda.Stream(device=params.g.device)
        self._step = (params, hyp, skip, bad, adam_fn or self._adam_fn, params.shard_slices(),
                      set())

    def _bucket(self, b: int) -> None:
        params, hyp, skip, bad, fn, slices, _ = self._step
        lo, hi, _ = params.layout.buckets[b]
        s_lo, s_hi, s_off, policy = slices[b]
        per = s_hi - s_lo
        cur, nxt = params.cur, params.cur ^ 1
        g = self._g_shard[s_off:s_off + per]
        self.reduce_scatter(params.g[lo:hi], g)
        ms = slice(s_off, s_off + per)
        fn(params.p[cur][s_lo:s_hi], g, params.m[cur][ms], params.v[cur][ms],
           params.p[nxt][s_lo:s_hi], params.m[nxt][ms], params.v[nxt][ms],
           per if policy else 0, hyp, skip, bad)
        self.all_gather(params.p[nxt][s_lo:s_hi], params.p[nxt][lo:hi])

    def bucket_ready(self, b: int, after=None) -> None:
        """Bucket b's local gradients are complete on the current stream (or at
        CUDA event `after`): reduce-scatter it, Adam on this rank's slice,
        all-gather the slice (on the side stream under NCCL, overlapping the
        caller's next kernels).  Collectives of one process group run in issue
        order, so a caller issues this where the exchange should queue."""
        done = self._step[6]
        if b in done:
            return
        done.add(b)
        if not self.overlap:
            self._bucket(b)
            return
        timed = self.timeline is not None
        if after is not None:
            ev = after
        else:
            ev = torch.cuda.Event(enable_timing=timed)
            ev.record()
        with torch.cuda.stream(self._stream):
            self._stream.wait_event(ev)
            if timed:
                t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0.record()
            self._bucket(b)
            if timed:
                t1.record()
                self.timeline.append((b, ev, t0, t1))

    def finish_step(self) -> None:
        """Every bucket exchanged; the current stream waits for the side stream."""
        params = self._step[0]
        for b in range(len(params.layout.buckets)):
            self.bucket_ready(b)
        if self.overlap:
            torch.cuda.current_stream().wait_stream(self._stream)
        self._step = None

    def adam(self, params, hyp: tuple, skip, bad, adam_fn=None) -> None:
        """The whole ZeRO-2 update at once: every bucket in order."""
        self.begin_step(params, hyp, skip, bad, adam_fn)
        self.finish_step()

    def gather_moments(self, params) -> None:
        """Collective: assemble every rank's moment slices into full host
        buffers (params.moments_to_host() then serves them at this generation)."""
        cur, total = params.cur, params.layout.total
        full = []
        for buf in (params.m[cur], params.v[cur]):
            host = np.zeros(total, dtype=np.float32)
            for b, (s_lo, s_hi, s_off, _) in enumerate(params.shard_slices()):
                lo, hi, _ = params.layout.buckets[b]
                gathered = torch.empty(hi - lo, dtype=buf.dtype, device=buf.device)
                self.all_gather(buf[s_off:s_off + (s_hi - s_lo)].clone(), gathered)
                host[lo:hi] = gathered.cpu().numpy()
            full.append(host)
        params.set_gathered_moments(*full)


def partition_trajectories(lengths, world: int, rank: int) -> tuple:
    """Contiguous, rank-ordered split of whole trajectories balanced by
    transition count: returns [start, stop) trajectory ids."""
    lens = np.asarray(lengths, dtype=np.int64)
    n = lens.shape[0]
    if n == 0:
        return 0, 0
    cum = np.concatenate([[0], np.cumsum(lens)])
    total = int(cum[-1])
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        cuts.append(int(np.searchsorted(cum, target, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.minimum(np.asarray(cuts), n))
    return int(cuts[rank]), int(cuts[rank + 1])
