"""Batched policy / world-model serving on the GPU.

Reference: `inference.run_batch` (inference.py:129-160) -- the evaluation of
one dynamic-window batch of requests under one weight snapshot, called by the
service's batcher (`_batcher`, inference.py:296-330; the firing rule
`should_trigger`, :69-74, is host control flow and stays the reference's).
Here the whole batch is one launch (`accel_serve`, csrc/imagine.cu): a warp
per request runs the policy's autoregressive chunk sampling and the state
value, the observation model, or the reward model, in float64 like the
reference.  Each policy request consumes the K uniforms of its own ticket
substream, `default_rng(SeedSequence([base_seed, ticket])).random(K)` (the
reference draws them one `rng.random()` per token), so a request's tokens
are bitwise independent of the batch it rides in, as the reference's
batched == solo property requires (tests/test_inference.py:148-170).
Weight snapshots are uploaded once per (kind, version) and cached.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import DimensionError, PayloadError
from .publish import OBS_MODEL, POLICY, REWARD_MODEL

F64, I32 = torch.float64, torch.int32
_KIND = {POLICY: 0, OBS_MODEL: 1, REWARD_MODEL: 2}


@dataclass(frozen=True)
class PolicyResponse:  # inference.py:86-91
    tokens: np.ndarray
    logits: np.ndarray
    value: float
    version: int


@dataclass(frozen=True)
class ObsResponse:  # inference.py:94-97
    next_obs: np.ndarray
    version: int


@dataclass(frozen=True)
class RewardResponse:  # inference.py:100-103
    probability: float
    version: int


def ticket_uniforms(base_seed: int, tickets, K: int) -> np.ndarray:
    """[n, K] uniforms: request i's substream SeedSequence([base_seed, ticket])."""
    return np.stack([np.random.default_rng(np.random.SeedSequence([base_seed, int(t)])).random(K)
                     for t in tickets]) if len(tickets) else np.zeros((0, K))


def _device_ticket_uniforms(base_seed: int, tickets, K: int, dev) -> torch.Tensor:
    """ticket_uniforms computed on the device (accel_ticket_uniforms: the same
    SeedSequence + PCG64 arithmetic, one thread per ticket); integers outside
    the kernel's 64-bit range take the host path."""
    n = len(tickets)
    if 0 <= int(base_seed) < 2 ** 64 and all(0 <= int(t) < 2 ** 63 for t in tickets):
        tk = torch.tensor([int(t) for t in tickets], dtype=torch.int64).to(dev)
        u = torch.empty(n, K, dtype=F64, device=dev)
        _lib.call("accel_ticket_uniforms", ctypes.c_uint64(int(base_seed)),
                  ctypes.c_void_p(tk.data_ptr()), n, int(K), ctypes.c_void_p(u.data_ptr()),
                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        return u
    return torch.from_numpy(ticket_uniforms(base_seed, tickets, K)).to(dev)


class DeviceServer:
    """Evaluates request batches on the device; drop-in for `run_batch`."""

    def __init__(self, device=None) -> None:
        if not torch.cuda.is_available():
            from .errors import AccelError
            raise AccelError("serving needs a CUDA device (there is no CPU path)")
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self._cache: dict = {}

    def _weights(self, weights):
        key = (weights.kind, int(weights.version), id(weights))
        hit = self._cache.get(weights.kind)
        if hit is not None and hit[0] == key:
            return hit[1], hit[2]
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(self.device)
        z = torch.zeros(1, dtype=F64, device=self.device)
        w = [z] * 23
        dims = [1] * 8
        flat, layout = getattr(weights, "flat", None), getattr(weights, "layout", None)
        if (weights.kind == POLICY and layout is not None and isinstance(flat, torch.Tensor)
                and flat.is_cuda and flat.device == self.device):
            # device-resident snapshot (Trainer.snapshot / broadcast_policy): the
            # serving layout (f64, [in][out]) is sliced, transposed and widened
            # from the flat fp32 buffer on the device -- no host round trip; the
            # values equal the host path's (the same fp32 parameters, widened)
            def dv(name, transpose=False, ravel=False):
                off = layout.offsets[name]
                shape = layout.shapes[name]
                x = flat[off:off + int(np.prod(shape))].view(shape)
                x = x.t() if transpose else x
                return (x.reshape(-1) if ravel else x).to(F64).contiguous()
            w[0:8] = [dv("w0", True), dv("b0"), dv("w1", True), dv("b1"), dv("e_prev"),
                      dv("e_pos"), dv("w_head", True), dv("b_head")]
            w[8:15] = [dv("w_attn"), dv("b_attn"), dv("e_step"), dv("w0v", True), dv("b0v"),
                       dv("w1v", ravel=True), dv("b1v")]
            d = layout.dims
            dims[:6] = [d.obs_dim, d.hidden, d.chunk_len, d.n_actions, d.n_steps, d.mlp_hidden]
        elif weights.kind == POLICY:
            pol, val = weights.policy, weights.value
            p, v = pol.params.tensors, val.params.tensors
            pc = pol.cfg
            w[0:8] = [t(p["w0"].T), t(p["b0"]), t(p["w1"].T), t(p["b1"]), t(p["e_prev"]),
                      t(p["e_pos"]), t(p["w_head"].T), t(p["b_head"])]
            w[8:15] = [t(v["w_attn"]), t(v["b_attn"]), t(v["e_step"]), t(v["w0v"].T),
                       t(v["b0v"]), t(v["w1v"].ravel()), t(v["b1v"])]
            dims[:6] = [pc.obs_dim, pc.hidden_dim, pc.chunk_len, pc.n_actions, val.cfg.n_steps,
                        val.cfg.mlp_hidden]
        elif weights.kind == OBS_MODEL:
            m = weights.obs_model
            o = m.params.tensors
            w[15:19] = [t(o["w0"].T), t(o["b0"]), t(o["w1"].T), t(o["b1"])]
            dims[0], dims[2], dims[3] = m.cfg.obs_dim, m.cfg.chunk_len, m.cfg.n_actions
            dims[6] = o["w0"].shape[0]
        elif weights.kind == REWARD_MODEL:
            m = weights.reward_model
            r = m.params.tensors
            w[19:23] = [t(r["w0"].T), t(r["b0"]), t(r["w1"].ravel()), t(r["b1"])]
            dims[0], dims[7] = r["w0"].shape[1], r["w0"].shape[0]
        else:
            raise PayloadError(f"unknown model kind {weights.kind!r}")
        self._cache[weights.kind] = (key, w, dims)
        return w, dims

    def run_batch(self, weights, requests, base_seed: int) -> list:
        """inference.run_batch: evaluate `requests` under one weight snapshot."""
        if not requests:
            raise PayloadError("run_batch on an empty request list")
        kinds = {r.kind for r in requests}
        if kinds != {weights.kind}:
            raise PayloadError(f"batch mixes kinds {sorted(kinds)} under weights {weights.kind!r}")
        w, dims = self._weights(weights)
        kind = _KIND[weights.kind]
        n, O, K, A = len(requests), dims[0], dims[2], dims[3]
        dev = self.device
        obs = np.stack([np.asarray(r.obs.vec, dtype=np.float64) for r in requests])
        if obs.shape != (n, O):
            raise DimensionError(f"observations {obs.shape} != ({n}, {O})")
        P = lambda x: None if x is None else ctypes.c_void_p(x.data_ptr())
        x = torch.from_numpy(obs).to(dev)
        steps = chunks = u = tok = lg = val = nxt = prob = None
        if kind == 0:
            st = np.array([int(r.obs.step) for r in requests], dtype=np.int64)
            if np.any(st < 0) or np.any(st >= dims[4]):  # ValueHead._check_steps (models.py:261-267)
                raise DimensionError(f"step index outside value-step table [0, {dims[4]})")
            steps = torch.from_numpy(st.astype(np.int32)).to(dev)
            u = _device_ticket_uniforms(base_seed, [r.ticket for r in requests], K, dev)
            tok = torch.empty(n, K, dtype=I32, device=dev)
            lg = torch.empty(n, K, A, dtype=F64, device=dev)
            val = torch.empty(n, dtype=F64, device=dev)
        elif kind == 1:
            ch = np.stack([np.asarray(r.chunk, dtype=np.int64) for r in requests])
            if ch.shape != (n, K):
                raise DimensionError(f"chunks {ch.shape} != ({n}, {K})")
            chunks = torch.from_numpy(ch.astype(np.int32)).to(dev)
            nxt = torch.empty(n, O, dtype=F64, device=dev)
        else:
            prob = torch.empty(n, dtype=F64, device=dev)
        wptrs = (ctypes.c_void_p * 23)(*[t.data_ptr() for t in w])
        _lib.call("accel_serve", wptrs, (ctypes.c_int * 8)(*dims), kind, P(x), P(steps),
                  P(chunks), P(u), n, P(tok), P(lg), P(val), P(nxt), P(prob),
                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        ver = int(weights.version)
        if kind == 0:
            tok, lg, val = tok.cpu().numpy().astype(np.int64), lg.cpu().numpy(), val.cpu().numpy()
            return [PolicyResponse(tok[i], lg[i], float(val[i]), ver) for i in range(n)]
        if kind == 1:
            nxt = nxt.cpu().numpy()
            return [ObsResponse(nxt[i], ver) for i in range(n)]
        prob = prob.cpu().numpy()
        return [RewardResponse(float(prob[i]), ver) for i in range(n)]
