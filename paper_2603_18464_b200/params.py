"""Device-resident parameters, gradients and Adam moments in one flat buffer.

Layout (fp32, each tensor 16-byte aligned): the policy tensors of the
reference `PolicyModel` (models.py:103-109) followed by the `ValueHead`
tensors (models.py:247-255).  One flat buffer lets a single kernel run Adam
over both parameter groups (two step counters, as the reference keeps two
`AdamState`s, trainer.py:312-315) and lets data-parallel ranks reduce all
gradients with one collective.

Parameters and moments are ping-ponged: Adam reads generation `cur` and
writes `1 - cur`; the host flips `cur` only after the step's record shows a
valid update, so a rejected step (dropped batch, non-finite gradients or
results) leaves the live parameters untouched, like the reference's pure
`adam_step` (numerics.py:95-126).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

POLICY_NAMES = ("w0", "b0", "w1", "b1", "e_prev", "e_pos", "w_head", "b_head")
VALUE_NAMES = ("w_attn", "b_attn", "e_step", "w0v", "b0v", "w1v", "b1v")


@dataclass(frozen=True)
class Dims:
    obs_dim: int      # O
    hidden: int       # D
    chunk_len: int    # K
    n_actions: int    # A
    n_steps: int      # S (value step table)
    mlp_hidden: int   # H

    def shapes(self) -> dict:
        O, D, K, A, S, H = (self.obs_dim, self.hidden, self.chunk_len, self.n_actions,
                            self.n_steps, self.mlp_hidden)
        return {
            "w0": (D, O), "b0": (D,), "w1": (D, D), "b1": (D,), "e_prev": (A + 1, D),
            "e_pos": (K, D), "w_head": (A, D), "b_head": (A,),
            "w_attn": (D,), "b_attn": (1,), "e_step": (S, D), "w0v": (H, D), "b0v": (H,),
            "w1v": (1, H), "b1v": (1,),
        }

    @classmethod
    def from_models(cls, policy, value) -> "Dims":
        pc, vc = policy.cfg, value.cfg
        if vc.hidden_dim != pc.hidden_dim:
            from .errors import DimensionError
            raise DimensionError(f"value hidden_dim {vc.hidden_dim} != policy {pc.hidden_dim}")
        return cls(pc.obs_dim, pc.hidden_dim, pc.chunk_len, pc.n_actions, vc.n_steps,
                   vc.mlp_hidden)


# Gradient buckets in flat order (ZeRO-2 reduce-scatter units), each complete
# at a distinct point of the backward: the value head first, then the head
# (e_prev, e_pos, w_head, b_head), then layer 1, then layer 0.
BUCKETS = (("w0", "b0"), ("w1", "b1"), ("e_prev", "e_pos", "w_head", "b_head"), VALUE_NAMES)


class FlatLayout:
    def __init__(self, dims: Dims, pad_to: int = 4) -> None:
        """pad_to: every bucket (BUCKETS) is padded to a multiple of it -- 4 *
        world under ZeRO-2, so each rank's slice of each bucket is equal and
        16-byte aligned (the reduce-scatter / all-gather unit)."""
        self.dims = dims
        self.pad_to = int(pad_to)
        shapes = dims.shapes()
        self.offsets, self.shapes = {}, {}
        self.buckets = []  # (lo, hi, is_policy)
        off = 0
        for names in BUCKETS:
            lo = off
            if names is VALUE_NAMES:
                self.n_policy = off
            for name in names:
                n = int(np.prod(shapes[name]))
                self.offsets[name] = off
                self.shapes[name] = shapes[name]
                off += (n + 3) // 4 * 4
            off = (off + self.pad_to - 1) // self.pad_to * self.pad_to
            self.buckets.append((lo, off, names is not VALUE_NAMES))
        self.total = off

    def bucket_of(self, name: str) -> int:
        return next(i for i, names in enumerate(BUCKETS) if name in names)

    def views(self, buf: torch.Tensor) -> dict:
        out = {}
        for name, off in self.offsets.items():
            n = int(np.prod(self.shapes[name]))
            out[name] = buf[off:off + n].view(self.shapes[name])
        return out

    def n_params(self, names) -> int:
        return int(sum(np.prod(self.shapes[k]) for k in names))

    def split(self, flat: np.ndarray) -> tuple:
        """Host flat buffer -> ({policy tensors}, {value tensors}) in float64."""
        out = ({}, {})
        for i, names in enumerate((POLICY_NAMES, VALUE_NAMES)):
            for k in names:
                off = self.offsets[k]
                n = int(np.prod(self.shapes[k]))
                out[i][k] = flat[off:off + n].astype(np.float64).reshape(self.shapes[k])
        return out


class DeviceParams:
    """Ping-pong parameter / moment buffers plus one gradient buffer.

    shard = (rank, world) (ZeRO-2): the Adam moments exist only for this
    rank's slice of every bucket, stored back to back in bucket order
    (`shard_slices`); parameters and gradients stay full (the forward and
    backward need all parameters; the gradients are reduce-scattered)."""

    def __init__(self, layout: FlatLayout, device, shard=None) -> None:
        self.layout = layout
        self.rank, self.world = shard if shard is not None else (0, 1)
        z = lambda n: torch.zeros(n, dtype=torch.float32, device=device)
        self.p = [z(layout.total), z(layout.total)]
        n_mom = layout.total // self.world
        self.m = [z(n_mom), z(n_mom)]
        self.v = [z(n_mom), z(n_mom)]
        self.g = z(layout.total)
        self.cur = 0
        self.generation = 0  # bumps on every flip (moments snapshots are tagged with it)
        self._moments_host = None
        self._views = [layout.views(self.p[0]), layout.views(self.p[1])]
        self.gv = layout.views(self.g)

    @property
    def sharded(self) -> bool:
        return self.world > 1

    def shard_slices(self) -> list:
        """Per bucket: (flat lo, flat hi, shard offset, is_policy) of this rank's slice."""
        out, s_off = [], 0
        for lo, hi, pol in self.layout.buckets:
            per = (hi - lo) // self.world
            out.append((lo + self.rank * per, lo + (self.rank + 1) * per, s_off, pol))
            s_off += per
        return out

    def rows(self, first: str, n_rows: int) -> torch.Tensor:
        """[n_rows, D] view of the current parameters starting at tensor `first`
        and running into the tensors after it (they are contiguous when each
        tensor's size is a multiple of 4 floats, as for e_prev -> e_pos)."""
        off = self.layout.offsets[first]
        d = self.layout.shapes[first][-1]
        names = list(self.layout.offsets)
        i, rows, parts, contiguous = names.index(first), 0, [], True
        while rows < n_rows:  # the tensors the rows run through
            name = names[i]
            r = int(np.prod(self.layout.shapes[name])) // d
            contiguous &= self.layout.offsets[name] == off + rows * d
            parts.append(self._views[self.cur][name].view(r, d))
            rows, i = rows + r, i + 1
        if contiguous:
            return self.p[self.cur][off:off + n_rows * d].view(n_rows, d)
        return torch.cat(parts)[:n_rows]  # padding between them: a small copy

    @property
    def pv(self) -> dict:
        return self._views[self.cur]

    def flip(self) -> None:
        self.cur ^= 1
        self.generation += 1

    def load(self, policy_tensors: dict, value_tensors: dict) -> None:
        host = np.zeros(self.layout.total, dtype=np.float32)
        for src, names in ((policy_tensors, POLICY_NAMES), (value_tensors, VALUE_NAMES)):
            for k in names:
                off = self.layout.offsets[k]
                arr = np.asarray(src[k], dtype=np.float32)
                if arr.shape != tuple(self.layout.shapes[k]):
                    from .errors import DimensionError
                    raise DimensionError(f"parameter {k!r}: shape {arr.shape} != "
                                         f"{self.layout.shapes[k]}")
                host[off:off + arr.size] = arr.ravel()
        self.p[self.cur].copy_(torch.from_numpy(host))

    def _split(self, flat: np.ndarray) -> tuple:
        return self.layout.split(flat)

    def to_host(self) -> tuple:
        return self._split(self.p[self.cur].cpu().numpy())

    def moments_to_host(self) -> tuple:
        """({policy m}, {value m}), ({policy v}, {value v}) in float64.  Under
        ZeRO-2 the moments are sharded: only a snapshot assembled by the
        collective `Trainer.gather_moments()` at the current generation is
        returned (a stale or missing one raises instead of mixing shards)."""
        if not self.sharded:
            return (self._split(self.m[self.cur].cpu().numpy()),
                    self._split(self.v[self.cur].cpu().numpy()))
        if self._moments_host is None or self._moments_host[0] != self.generation:
            from .errors import AccelError
            raise AccelError("Adam moments are sharded across data-parallel ranks: call the "
                             "collective Trainer.gather_moments() on every rank first")
        m, v = self._moments_host[1]
        return self._split(m), self._split(v)

    def set_gathered_moments(self, m_full: np.ndarray, v_full: np.ndarray) -> None:
        self._moments_host = (self.generation, (m_full, v_full))

    def grads_to_host(self) -> tuple:
        return self._split(self.g.cpu().numpy())


class AdamStateView:
    """Reference-shaped view of one Adam group (numerics.py:75-92)."""

    def __init__(self, owner, group: int, lr: float, beta1: float, beta2: float,
                 eps: float = 1e-8) -> None:
        self._owner = owner
        self._group = group
        self.step = 0
        self.lr, self.beta1, self.beta2, self.eps = lr, beta1, beta2, eps

    def hyper(self, t: int) -> tuple:
        """{lr, beta1, beta2, eps, 1 - beta1^t, 1 - beta2^t} for step t (host)."""
        return (self.lr, self.beta1, self.beta2, self.eps,
                1.0 - self.beta1 ** t, 1.0 - self.beta2 ** t)

    @property
    def m(self) -> dict:
        return self._owner.params.moments_to_host()[0][self._group]

    @property
    def v(self) -> dict:
        return self._owner.params.moments_to_host()[1][self._group]
