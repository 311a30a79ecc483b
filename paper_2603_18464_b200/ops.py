"""Torch-tensor front end of the C ABI (device pointers + the current stream).

Each function takes CUDA tensors, checks dtype/shape/contiguity on the host,
and launches through `_lib.call` on `torch.cuda.current_stream()` (so the
calls are capturable in CUDA graphs).  No function here has a CPU path.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .errors import AccelError, DimensionError

F32, F64, I32, I64, U8 = torch.float32, torch.float64, torch.int32, torch.int64, torch.uint8


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _check(t, name, dtype, shape=None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise AccelError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if t.dtype != dtype:
        raise DimensionError(f"{name}: dtype {t.dtype} != {dtype}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise DimensionError(f"{name}: shape {tuple(t.shape)} != {tuple(shape)}")
    if not t.is_contiguous():
        raise DimensionError(f"{name} must be contiguous")


class Workspace:
    """Grow-only scratch buffer reused across calls on one device."""

    def __init__(self) -> None:
        self._buf = None

    def get(self, nbytes: int) -> torch.Tensor:
        nbytes = max(int(nbytes), 16)
        if self._buf is None or self._buf.numel() < nbytes:
            self._buf = torch.empty(nbytes + (nbytes >> 3), dtype=U8, device="cuda")
        return self._buf


_WS: dict = {}


def workspace(tag: str) -> Workspace:
    return _WS.setdefault(tag, Workspace())


# ---------------------------------------------------------------------------
# (a) advantages


def gae_segmented(rewards, values_frames, traj_off, done, gamma, lam, *, adv=None, ret=None,
                  frame_of=None, sums=None, ws: Workspace | None = None):
    """Segmented GAE (trainer.py:79-101) over a CSR batch; see accel.h."""
    n_traj = traj_off.shape[0] - 1
    n = rewards.shape[0]
    _check(rewards, "rewards", F32, (n,))
    _check(values_frames, "values_frames", F32, (n + n_traj,))
    _check(traj_off, "traj_off", I64, (n_traj + 1,))
    _check(done, "done", U8, (n_traj,))
    adv = torch.empty_like(rewards) if adv is None else adv
    ret = torch.empty_like(rewards) if ret is None else ret
    sums = torch.empty(4, dtype=F64, device=rewards.device) if sums is None else sums
    if frame_of is not None:
        _check(frame_of, "frame_of", I32, (n,))
    nbytes = _lib.lib().accel_gae_workspace_size(n)
    buf = (ws or workspace("gae")).get(nbytes)
    _lib.call("accel_gae_segmented", _p(rewards), _p(values_frames), _p(traj_off), _p(done),
              n_traj, n, float(gamma), float(lam), _p(adv), _p(ret), _p(frame_of), _p(sums),
              _p(buf), buf.numel(), _stream())
    return adv, ret, sums


def normalize_finalize(sums, eps, stats=None):
    """Pooled mean/std/denominator + domain flags (trainer.py:135-150)."""
    _check(sums, "sums", F64)
    stats = torch.empty(4, dtype=F64, device=sums.device) if stats is None else stats
    _lib.call("accel_normalize_finalize", _p(sums), float(eps), _p(stats), _stream())
    return stats


def normalize_apply(adv, stats, out=None):
    _check(adv, "adv", F32)
    out = torch.empty_like(adv) if out is None else out
    _lib.call("accel_normalize_apply", _p(adv), adv.numel(), _p(stats), _p(out), _stream())
    return out
