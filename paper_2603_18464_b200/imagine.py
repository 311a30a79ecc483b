"""Batched world-model imagination on the GPU (north-star (c)).

`Imaginer(bundle, grid=(height, width)).imagine(starts, h_img)` runs
`RolloutWorker.imagine_episode` (rollout.py:295-362) for every start frame
in one kernel launch (`accel_imagine`): the per-step policy / obs-model /
reward-model requests (inference.py:146-159) never leave the device.
Returns reference `Trajectory` records (source "imagined") or None for
episodes the reference would discard (non-finite prediction,
rollout.py:315-331).

Randomness: `uniforms` [n, h_img + 1, K] reproduces the reference exactly
(the r-th policy request of episode e consumes uniforms[e, r]); without
it a Philox stream keyed by (seed, episode) is used.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import DimensionError
from .types import Trajectory

F64 = torch.float64


class Imaginer:
    def __init__(self, bundle, grid: tuple | None = None, threshold: float = 0.9,
                 version: int = 0) -> None:
        if not torch.cuda.is_available():
            from .errors import AccelError
            raise AccelError("imagination needs a CUDA device (there is no CPU path)")
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.grid = grid
        self.threshold = float(threshold)
        self.update(bundle, version)

    def update(self, bundle, version: int = 0) -> None:
        """(Re)upload the four parameter sets (float64, transposed)."""
        pol, val = bundle.policy, bundle.value
        obs_m, rew_m = bundle.obs_model, bundle.reward_model
        pc = pol.cfg
        p, v = pol.params.tensors, val.params.tensors
        o, r = obs_m.params.tensors, rew_m.params.tensors
        self.O, self.D, self.K, self.A = pc.obs_dim, pc.hidden_dim, pc.chunk_len, pc.n_actions
        self.S, self.HV = val.cfg.n_steps, val.cfg.mlp_hidden
        self.HO, self.HR = o["w0"].shape[0], r["w0"].shape[0]
        if o["w0"].shape[1] != self.O + self.K * self.A or o["w1"].shape[0] != self.O:
            raise DimensionError("obs model does not map [obs, onehot(chunk)] -> obs")
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(self.device)
        self._w = [
            t(p["w0"].T), t(p["b0"]), t(p["w1"].T), t(p["b1"]), t(p["e_prev"]), t(p["e_pos"]),
            t(p["w_head"].T), t(p["b_head"]),
            t(v["w_attn"]), t(v["b_attn"]), t(v["e_step"]), t(v["w0v"].T), t(v["b0v"]),
            t(v["w1v"].ravel()), t(v["b1v"]),
            t(o["w0"].T), t(o["b0"]), t(o["w1"].T), t(o["b1"]),
            t(r["w0"].T), t(r["b0"]), t(r["w1"].ravel()), t(r["b1"]),
        ]
        self.version = version

    def imagine(self, start_vecs, start_steps, h_img: int, uniforms=None, seed: int = 0) -> dict:
        """One batch; returns host numpy arrays keyed like the kernel outputs.

        The outputs come back as asynchronous copies into page-locked buffers
        (from torch's caching host allocator, so a returned array owns its
        buffer until it is dropped) with one synchronization for the batch."""
        out = self.imagine_device(start_vecs, start_steps, h_img, uniforms, seed)
        host = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in out.items()}
        for k, v in out.items():
            host[k].copy_(v, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return {k: v.numpy() for k, v in host.items()}

    def imagine_device(self, start_vecs, start_steps, h_img: int, uniforms=None,
                       seed: int = 0) -> dict:
        """Launch on the current stream; returns the device output tensors."""
        if isinstance(start_vecs, torch.Tensor):
            x = start_vecs.to(self.device, torch.float64).contiguous()
        else:
            x = torch.as_tensor(np.asarray(start_vecs, dtype=np.float64), device=self.device)
        n = x.shape[0]
        if x.shape != (n, self.O):
            raise DimensionError(f"start observations {tuple(x.shape)} != (n, {self.O})")
        if isinstance(start_steps, torch.Tensor):
            st = start_steps.to(self.device, torch.int32).contiguous()
        else:
            st = torch.as_tensor(np.asarray(start_steps, dtype=np.int32), device=self.device)
        u = None
        if uniforms is not None:
            u = torch.as_tensor(np.asarray(uniforms, dtype=np.float64), device=self.device)
            if u.shape != (n, h_img + 1, self.K):
                raise DimensionError(f"uniforms {tuple(u.shape)} != {(n, h_img + 1, self.K)}")
            u = u.contiguous()
        dev, H, O, K, A = self.device, h_img, self.O, self.K, self.A
        out = {
            "observations": torch.zeros(n, H + 1, O, dtype=F64, device=dev),
            "steps": torch.zeros(n, H + 1, dtype=torch.int32, device=dev),
            "tokens": torch.zeros(n, H, K, dtype=torch.int32, device=dev),
            "behavior_logits": torch.zeros(n, H, K, A, dtype=F64, device=dev),
            "values": torch.zeros(n, H, dtype=F64, device=dev),
            "rewards": torch.zeros(n, H, dtype=F64, device=dev),
            "bootstrap_value": torch.zeros(n, dtype=F64, device=dev),
            "t_len": torch.zeros(n, dtype=torch.int32, device=dev),
            "done": torch.zeros(n, dtype=torch.uint8, device=dev),
            "status": torch.zeros(n, dtype=torch.int32, device=dev),
        }
        gh, gw = self.grid if self.grid is not None else (0, 0)
        dims = (ctypes.c_int * 11)(O, self.D, K, A, self.S, self.HV, self.HO, self.HR, gh, gw,
                                   1 if self.grid is not None else 0)
        wptrs = (ctypes.c_void_p * len(self._w))(*[w.data_ptr() for w in self._w])
        P = lambda tns: None if tns is None else ctypes.c_void_p(tns.data_ptr())
        _lib.call("accel_imagine", wptrs, dims, int(H), self.threshold, ctypes.c_uint64(seed),
                  P(x), P(st), P(u), n, P(out["observations"]), P(out["steps"]),
                  P(out["tokens"]), P(out["behavior_logits"]), P(out["values"]),
                  P(out["rewards"]), P(out["bootstrap_value"]), P(out["t_len"]), P(out["done"]),
                  P(out["status"]), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        return out

    def imagine_trajectories(self, starts, h_img: int, uniforms=None, seed: int = 0) -> list:
        """starts: objects with .vec, .step, .task_id (env.Observation)."""
        res = self.imagine([s.vec for s in starts], [s.step for s in starts], h_img, uniforms,
                           seed)
        out = []
        for e, s in enumerate(starts):
            if res["status"][e] != 0:
                out.append(None)
                continue
            T = int(res["t_len"][e])
            out.append(Trajectory(
                task_id=int(s.task_id), source="imagined",
                observations=res["observations"][e, :T + 1], steps=res["steps"][e, :T + 1],
                tokens=res["tokens"][e, :T], rewards=res["rewards"][e, :T],
                behavior_logits=res["behavior_logits"][e, :T], values=res["values"][e, :T],
                bootstrap_value=float(res["bootstrap_value"][e]), done=bool(res["done"][e]),
                behavior_version=self.version,
                step_versions=np.full(T, self.version, dtype=np.int64)))
        return out
