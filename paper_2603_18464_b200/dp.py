"""ZeRO-2 data parallelism for the trainer step (one process per GPU).

The reference simulates data parallelism inside one process: advantage
statistics are summed over K logical shards (trainer.py:128-158, "a
simulated all-reduce") and the paper's trainer is ZeRO-2 over
NCCL.  Here every rank owns whole trajectories (the
batch is partitioned in rank order) and the step exchanges:

  C1  all_reduce(SUM) f64 {sum A, sum A^2, N}        pooled normalization (Eqs. 5-7)
  C5  all_reduce(SUM) f64 token statistics, MAX of {ratio_max, -w_min}
      -> global included-token count m, entropy over N*K, value MSE over N
  C2  reduce_scatter(SUM) of the flat fp32 gradient buffer (ZeRO-2)
      Adam on this rank's 1/R shard of parameters and moments
  C3  all_gather of the updated parameter shards

Results equal the single-process step over the concatenation of all ranks'
trajectories up to float summation order (see tests/test_dp.py).  All
collectives go through torch.distributed (NCCL on B200s, gloo in the CPU
tests); the NCCL calls are stream-ordered with the trainer's kernels.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


class DataParallel:
    def __init__(self, group=None, adam_fn=None) -> None:
        if not dist.is_initialized():
            raise RuntimeError("DataParallel needs torch.distributed to be initialized")
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = dist.get_backend(group)
        self._adam_fn = adam_fn
        self._shard_cache = {}

    # -- small collectives ----------------------------------------------------------
    def all_reduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def all_reduce_max(self, t: torch.Tensor) -> torch.Tensor:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return t

    def global_counts(self, n_local: int, k: int) -> tuple:
        t = torch.tensor([float(n_local)], dtype=torch.float64,
                         device=self._device())
        self.all_reduce_sum(t)
        n = int(t.item())
        return n, n * k

    def _device(self):
        if self.backend == "nccl":
            return torch.device("cuda", torch.cuda.current_device())
        return torch.device("cpu")

    # -- ZeRO-2 sharding ------------------------------------------------------------
    def shard_bounds(self, total: int) -> tuple:
        """[lo, hi) of this rank's shard; `total` must be a multiple of world."""
        if total % self.world:
            raise ValueError(f"flat buffer of {total} is not a multiple of world {self.world}")
        per = total // self.world
        return self.rank * per, (self.rank + 1) * per

    def reduce_scatter(self, flat: torch.Tensor) -> torch.Tensor:
        """Sum of `flat` over ranks, restricted to this rank's shard (ZeRO-2 C2)."""
        lo, hi = self.shard_bounds(flat.numel())
        key = (flat.numel(), flat.dtype, flat.device)
        out = self._shard_cache.get(key)
        if out is None:
            out = torch.empty(hi - lo, dtype=flat.dtype, device=flat.device)
            self._shard_cache[key] = out
        if self.backend == "gloo":  # gloo has no reduce_scatter_tensor on CPU
            tmp = flat.clone()
            dist.all_reduce(tmp, op=dist.ReduceOp.SUM, group=self.group)
            out.copy_(tmp[lo:hi])
        else:
            dist.reduce_scatter_tensor(out, flat, op=dist.ReduceOp.SUM, group=self.group)
        return out

    def all_gather(self, shard: torch.Tensor, full: torch.Tensor) -> torch.Tensor:
        """C3: every rank's shard into `full` (rank-ordered)."""
        if self.backend == "gloo":
            parts = [torch.empty_like(shard) for _ in range(self.world)]
            dist.all_gather(parts, shard.contiguous(), group=self.group)
            full.copy_(torch.cat(parts))
        else:
            dist.all_gather_into_tensor(full, shard.contiguous(), group=self.group)
        return full

    def adam(self, params, n_policy: int, hyp: tuple, skip, bad, adam_fn=None) -> None:
        """Reduce-scatter the gradients, Adam on this rank's shard (ping-pong
        generation cur -> nxt), all-gather the new parameters.  The Adam moments
        stay sharded (ZeRO-2: a rank only ever reads its own shard of them);
        `gather_moments` assembles them when a caller needs the full state."""
        fn = adam_fn or self._adam_fn
        cur, nxt = params.cur, params.cur ^ 1
        total = params.p[cur].numel()
        lo, hi = self.shard_bounds(total)
        g_shard = self.reduce_scatter(params.g)
        n0 = min(max(n_policy - lo, 0), hi - lo)
        fn(params.p[cur][lo:hi], g_shard, params.m[cur][lo:hi], params.v[cur][lo:hi],
           params.p[nxt][lo:hi], params.m[nxt][lo:hi], params.v[nxt][lo:hi], n0, hyp[0], hyp[1],
           skip, bad)
        self.all_gather(params.p[nxt][lo:hi].clone(), params.p[nxt])

    def gather_moments(self, params) -> None:
        """Collective: every rank's shard of the current Adam moments into the
        full buffers (for inspection / checkpointing; not on the step path)."""
        cur = params.cur
        lo, hi = self.shard_bounds(params.m[cur].numel())
        for buf in (params.m[cur], params.v[cur]):
            self.all_gather(buf[lo:hi].clone(), buf)


def partition_trajectories(lengths, world: int, rank: int) -> tuple:
    """Contiguous, rank-ordered split of whole trajectories balanced by
    transition count: returns [start, stop) trajectory ids."""
    import numpy as np
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
