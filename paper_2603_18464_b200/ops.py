"""Torch-tensor front end of the C ABI (device pointers + the current stream).

Each function takes CUDA tensors, checks dtype/shape/contiguity on the host,
and launches through `_lib.call` on `torch.cuda.current_stream()` (so the
calls are capturable in CUDA graphs).  No function here has a CPU path.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import AccelError, DimensionError

F32, F64, I32, I64, U8 = torch.float32, torch.float64, torch.int32, torch.int64, torch.uint8


def _p(t):
    """Pointer of a dense tensor (the kernel assumes its packed row-major layout):
    a strided view would be read or written as if it were packed, so refuse it."""
    if t is None:
        return None
    if not t.is_contiguous():
        raise DimensionError(f"dense operand expected, got strides {tuple(t.stride())} "
                             f"for shape {tuple(t.shape)}")
    return ctypes.c_void_p(t.data_ptr())


def _pp(t):
    """Pointer of a row-pitched operand (unit column stride; the wrapper passes
    its row pitch to the kernel)."""
    if t is None:
        return None
    if t.dim() == 2 and t.shape[0] > 1 and t.stride(1) != 1:
        raise DimensionError(f"pitched operand needs unit column stride, got {tuple(t.stride())}")
    return ctypes.c_void_p(t.data_ptr())


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


_RETAIN = []  # grown-out buffers kept alive once a CUDA graph may reference them


def retain_workspaces() -> None:
    """From now on a grow-only buffer that is replaced is kept alive instead of
    freed: a captured CUDA graph may still point into it (trainer.CapturedStep)."""
    if not _RETAIN:
        _RETAIN.append(None)


def retire(buf) -> None:
    if _RETAIN and buf is not None:
        _RETAIN.append(buf)


class Workspace:
    """Grow-only scratch buffer reused across calls on one device."""

    def __init__(self) -> None:
        self._buf = None

    def get(self, nbytes: int) -> torch.Tensor:
        nbytes = max(int(nbytes), 16)
        if self._buf is None or self._buf.numel() < nbytes:
            retire(self._buf)
            self._buf = torch.empty(nbytes + (nbytes >> 3), dtype=U8, device="cuda")
        return self._buf


_WS: dict = {}


def workspace(tag: str) -> Workspace:
    return _WS.setdefault(tag, Workspace())


def stream_workspace(tag: str, nbytes: int) -> torch.Tensor:
    """Grow-only scratch private to the current stream: launches on one stream
    are ordered, so reuse is safe; launches on different streams (the trainer
    runs the value-head backward beside the policy's) never share a buffer."""
    return workspace(f"{tag}@{torch.cuda.current_stream().cuda_stream}").get(nbytes)


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
    nbytes = _lib.lib().accel_gae_workspace_size(n_traj, n)
    buf = ws.get(nbytes) if ws is not None else stream_workspace("gae", nbytes)
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


# ---------------------------------------------------------------------------
# (b) token loss


def token_grid(M: int) -> int:
    return int(_lib.lib().accel_token_grid(int(M)))


def token_logp(mu, tokens, lp_out=None, bad_part=None):
    """Behavior log-probs (trainer.py:289-293); mu f32[M, A], tokens i32[M]."""
    M, A = mu.shape
    _check(mu, "mu", F32)
    _check(tokens, "tokens", I32)
    if tokens.numel() != M:
        raise DimensionError(f"tokens has {tokens.numel()} entries, expected {M}")
    lp_out = torch.empty(M, dtype=F32, device=mu.device) if lp_out is None else lp_out
    g = token_grid(M)
    bad_part = torch.empty(g, 2, dtype=F64, device=mu.device) if bad_part is None else bad_part
    _lib.call("accel_token_logp", _p(mu), _p(tokens), M, A, _p(lp_out), _p(bad_part), _stream())
    return lp_out, bad_part


def token_loss(logits, bias, tokens, lp_old, adv, K, algo, sigma, clip_eps, lambda_h, m_global,
               dlogits, lp_new, dbias_part, stat_part, max_part, fix_stats=None):
    """Fused GIPO/PPO + entropy forward/backward (see accel.h)."""
    M, A = logits.shape
    _lib.call("accel_token_loss", _p(logits), _p(bias), _p(tokens), _p(lp_old), _p(adv), M, int(K),
              A, int(algo), float(sigma), float(clip_eps), float(lambda_h), float(m_global),
              _p(fix_stats), _p(dlogits), _p(lp_new), _p(dbias_part), _p(stat_part),
              _p(max_part), _stream())


# ---------------------------------------------------------------------------
# policy glue


def bias_tanh(z, b):
    _lib.call("accel_bias_tanh", _p(z), _p(b), z.shape[0], z.shape[1], _stream())
    return z


def build_c(h2, frame_of, tokens, e_prev, e_pos, N, K, A, out):
    _lib.call("accel_build_c", _p(h2), _p(frame_of), _p(tokens), _p(e_prev), _p(e_pos), N, K, A,
              h2.shape[1], _p(out), _stream())
    return out


def rows_grid(rows: int) -> int:
    return int(_lib.lib().accel_rows_grid(int(rows)))


def warp_grid(rows: int) -> int:
    return int(_lib.lib().accel_warp_grid(int(rows)))


def dc_reduce(dc, h2, frame_of, N, K, D, dz2, pos_part, db1_part, grid):
    _lib.call("accel_dc_reduce", _p(dc), _p(h2), _p(frame_of), N, K, D, _p(dz2), _p(pos_part),
              _p(db1_part), int(grid), _stream())


def tanh_grad_colsum(g, h, col_part, grid):
    for t, nm in ((g, "g"), (h, "h")):
        if t.stride(1) != 1:
            raise DimensionError(f"tanh_grad_colsum: {nm} needs unit column stride")
    _lib.call("accel_tanh_grad_colsum", _pp(g), g.stride(0), _pp(h), h.stride(0), g.shape[0],
              g.shape[1], _pp(col_part), int(grid), _stream())


# ---------------------------------------------------------------------------
# deterministic grouping (np.add.at)


class Grouping:
    """A stable counting sort of R keys in [0, nkeys) (fixed per batch).

    cpb > 0: frame-blocked order -- rows are cut into blocks of cpb 4096-row
    chunks and sorted by (block, key), so a pass over the pieces in order
    touches one block of rows at a time (accel_group_by_key_blocked); the key
    sums then fold the blocks in order (accel_fold_blocked_pieces)."""

    def __init__(self, keys, nkeys: int, cpb: int = 0, rows=None, heavy_key: int = -1):
        """rows: also write the inverse permutation pos inside the scatter (see
        sort_rows).  heavy_key: a key expected to hold a large share of the rows
        (its key pass runs over more CTAs; -1: none)."""
        R = keys.numel()
        dev = keys.device
        lib = _lib.lib()
        self.R, self.nkeys, self.cpb = R, int(nkeys), int(cpb)
        self.heavy_key = int(heavy_key)
        self.nblocks = int(lib.accel_group_blocks(R, self.cpb)) if cpb > 0 else 1
        nk = self.nkeys * self.nblocks
        self.perm = torch.empty(max(R, 1), dtype=I32, device=dev)
        self.seg_off = torch.empty(nk + 1, dtype=I64, device=dev)
        self.piece_off = torch.empty(nk + 1, dtype=I64, device=dev)
        self.max_pieces = int(lib.accel_group_max_pieces_blocked(R, nkeys, self.cpb))
        self.piece_key = torch.empty(max(self.max_pieces, 1), dtype=I32, device=dev)
        nbytes = lib.accel_group_workspace_size_blocked(R, nkeys, self.cpb)
        buf = stream_workspace("group", nbytes)
        self.pos = None
        if rows:  # the inverse permutation, written coalesced by the scatter
            self.pos = torch.empty(max(R, 1), dtype=I32, device=dev)
        _lib.call("accel_group_by_key_blocked", _pp(keys), R, nkeys, self.cpb, _pp(self.perm),
                  _pp(self.seg_off), _pp(self.piece_off), _pp(self.piece_key), None, None, 1,
                  None, None, _pp(self.pos), _pp(buf), buf.numel(), _stream())

    def sort_rows(self, frame_of=None, tokens=None, K=None):
        """The inverse permutation pos (pos[perm[r]] = r, fixed per batch): where
        the loss kernel writes each token's scalars for the grouped recompute."""
        if self.pos is None:
            R = self.R
            self.pos = torch.empty(max(R, 1), dtype=I32, device=self.perm.device)
            scratch = torch.empty(2 * max(R, 1), dtype=I32, device=self.perm.device)
            _lib.call("accel_sorted_rows", _pp(self.perm), _pp(frame_of), _pp(tokens), R, int(K),
                      _pp(scratch[:max(R, 1)]), _pp(scratch[max(R, 1):]), _pp(self.pos), _stream())
        return self.pos

    def fact_rows_sum(self, h2w, epp, frame_of, tokens, tsc, K, out, piece_buf=None):
        """Grouped dz sums with dz recomputed from the loss pass's token scalars
        (accel_fact_group_sum, then the key pass)."""
        A = h2w.shape[1]
        if piece_buf is None:
            piece_buf = stream_workspace("group_pieces_f32", 4 * max(self.max_pieces, 1) * A)
        nk = self.nkeys * self.nblocks
        if self.cpb > 0:  # tsc holds the scalars at the sorted positions (sort_rows)
            _lib.call("accel_fact_group_sum2", _pp(h2w), _pp(epp), _pp(self.perm), _pp(frame_of),
                      _pp(tokens), int(K), _pp(tsc), _pp(self.seg_off), _pp(self.piece_off),
                      _pp(self.piece_key), nk, self.nkeys, A, self.max_pieces, _pp(piece_buf),
                      _stream())
        else:
            _lib.call("accel_fact_group_sum", _pp(h2w), _pp(epp), _pp(frame_of), _pp(tokens),
                      _pp(tsc), _pp(self.perm), _pp(self.seg_off), _pp(self.piece_off), nk, 0,
                      int(K), A, 256, self.max_pieces, _pp(piece_buf), _stream())
        self._key_pass(piece_buf, A, out)
        return out

    def rows_sum(self, vals, out, piece_buf=None):
        D = vals.shape[1]
        if piece_buf is None:
            piece_buf = stream_workspace("group_pieces_f32", 4 * max(self.max_pieces, 1) * D)
        if self.cpb > 0:
            raise DimensionError("rows_sum needs a plain (unblocked) grouping")
        _lib.call("accel_grouped_rows_sum", _pp(vals), self.R, D, _pp(self.perm), _pp(self.seg_off),
                  _pp(self.piece_off), _pp(self.piece_key), self.nkeys, self.max_pieces,
                  _pp(piece_buf), _pp(out), _stream())
        return out

    def _key_pass(self, piece_buf, D, out):
        if self.cpb > 0:
            wsb = stream_workspace("fold", _lib.lib().accel_fold_workspace_size(self.nkeys, D))
            _lib.call("accel_fold_blocked_pieces", _pp(piece_buf), _pp(self.piece_off), self.nkeys,
                      self.nblocks, D, self.heavy_key, _pp(out), _pp(wsb), _stream())
        else:
            _lib.call("accel_grouped_rows_sum", None, self.R, D, _pp(self.perm), _pp(self.seg_off),
                      _pp(self.piece_off), _pp(self.piece_key), self.nkeys, self.max_pieces,
                      _pp(piece_buf), _pp(out), _stream())


def prev_keys(tokens, N, K, A, with_pos=False, out=None):
    out = torch.empty(N * K, dtype=I32, device=tokens.device) if out is None else out
    _lib.call("accel_prev_keys", _p(tokens), N, K, A, int(bool(with_pos)), _p(out), _stream())
    return out


def fact_grid(N: int) -> int:
    return int(_lib.lib().accel_fact_grid(int(N)))


def fact_partials(N: int, K: int, A: int, scalar_out: bool) -> int:
    """Rows of the loss kernel's statistics partials (accel_fact_partials)."""
    return int(_lib.lib().accel_fact_partials(int(N), int(K), int(A), int(bool(scalar_out))))


def ep_plus(ep, pp, bias, K, out):
    A = ep.shape[1]
    _lib.call("accel_ep_plus", _p(ep), _p(pp), _p(bias), A, int(K), _p(out), _stream())
    return out


def token_loss_fact(h2w, epp, frame_of, tokens, lp_old, adv, N, K, algo, sigma, clip_eps,
                    lambda_h, m_global, dz, g_frame, lp_new, stat_part, max_part,
                    fix_stats=None, tsc=None, tsc_pos=None):
    """Factorized-head fused loss (see accel.h accel_token_loss_fact2); dz=None
    with tsc (f32[M, 4]) writes the per-token scalars instead of dz rows, at
    tsc_pos[t] (a frame-blocked grouping's sorted positions) when given."""
    A = h2w.shape[1]
    counters = stream_workspace("fact2_ctr", 8)  # main-pass / fix-up work counters
    _lib.call("accel_token_loss_fact2", _p(h2w), _p(epp), _p(frame_of), _p(tokens), _p(lp_old),
              _p(adv), int(N), int(K), A, int(algo), float(sigma), float(clip_eps),
              float(lambda_h), float(m_global), _p(fix_stats), _p(dz), _p(tsc), _p(tsc_pos),
              _p(g_frame), _p(lp_new), _p(stat_part), _p(max_part), _p(counters), _stream())


def pk_marginals(dpk, K, A, dprev, dpos):
    _lib.call("accel_pk_marginals", _p(dpk), int(K), int(A), _p(dprev), _p(dpos), _stream())


def step_keys(steps, frame_of, R, n_steps, bad_count, out=None):
    out = torch.empty(R, dtype=I32, device=steps.device) if out is None else out
    _lib.call("accel_step_keys", _p(steps), _p(frame_of), R, int(n_steps), _p(out), _p(bad_count),
              _stream())
    return out


# ---------------------------------------------------------------------------
# value head


def value_pool(h1, h2, row_frame, steps, R, n_steps, w_attn, b_attn, e_step, U, alpha, bad_part,
               grid):
    _lib.call("accel_value_pool", _p(h1), _p(h2), _p(row_frame), _p(steps), R, h1.shape[1],
              int(n_steps), _p(w_attn), _p(b_attn), _p(e_step), _p(U), _p(alpha), _p(bad_part),
              int(grid), _stream())


def value_head(zm, b0v, w1v, b1v, targets, lambda_v, n_global, values_out, part, dpart, grid,
               row_frame=None, rows=None, v_old=None, vclip=0.0):
    """rows R (default zm rows); row_frame: zm row of each of the R rows (the
    dzm rows are written back there); v_old (+ vclip > 0): value-clip loss."""
    R = zm.shape[0] if rows is None else int(rows)
    _lib.call("accel_value_head", _p(zm), _p(row_frame), _p(b0v), _p(w1v), _p(b1v), R,
              zm.shape[1], _p(targets), _p(v_old), float(vclip), float(lambda_v),
              float(n_global), _p(values_out), _p(part), _p(dpart), int(grid), _stream())


def value_attn_grad(dU, h1, h2, row_frame, alpha, de, part, grid):
    _lib.call("accel_value_attn_grad", _p(dU), _p(h1), _p(h2), _p(row_frame), _p(alpha),
              dU.shape[0], dU.shape[1], _p(de), _p(part), int(grid), _stream())


def value_attn_backward(dU, h1, h2, row_frame, alpha, bpart, wpart, grid, de=None):
    """value_attn_grad + value_attn_wgrad in one pass (de rows optional)."""
    _lib.call("accel_value_attn_backward", _p(dU), _p(h1), _p(h2), _p(row_frame), _p(alpha),
              dU.shape[0], dU.shape[1], _p(de), _p(bpart), _p(wpart), int(grid), _stream())


def value_attn_wgrad(de, h1, h2, row_frame, R, part, grid):
    _lib.call("accel_value_attn_wgrad", _p(de), _p(h1), _p(h2), _p(row_frame), R, h1.shape[1],
              _p(part), int(grid), _stream())


# ---------------------------------------------------------------------------
# reductions / record / optimizer


def reduce_segments(segs):
    """segs: list of (src_tensor, dst_tensor, parts, len, pitch) (<= 16)."""
    n = len(segs)
    if n == 0:
        return
    for src, dst, parts, ln, pitch in segs:  # the kernel writes len packed floats from dst
        if not dst.is_contiguous() or dst.numel() < ln:
            raise DimensionError(f"reduce_segments: dst must be packed with >= {ln} elements")
        need = (int(parts) - 1) * int(pitch) + int(ln) if parts else 0
        if src.storage_offset() + need > src.untyped_storage().nbytes() // src.element_size():
            raise DimensionError("reduce_segments: src parts exceed their storage")
    srcs = (ctypes.c_void_p * n)(*[s[0].data_ptr() for s in segs])
    dsts = (ctypes.c_void_p * n)(*[s[1].data_ptr() for s in segs])
    parts = (ctypes.c_int64 * n)(*[int(s[2]) for s in segs])
    lens = (ctypes.c_int64 * n)(*[int(s[3]) for s in segs])
    pitches = (ctypes.c_int64 * n)(*[int(s[4]) for s in segs])
    _lib.call("accel_reduce_segments", srcs, dsts, parts, lens, pitches, n, _stream())


def reduce_f64(part, parts, width, mode, out):
    nbytes = _lib.lib().accel_reduce_f64_scratch_size(int(parts), int(width))
    scratch = stream_workspace("reduce_f64", nbytes) if nbytes else None
    _lib.call("accel_reduce_f64", _p(part), int(parts), int(width), int(mode), _p(out),
              _p(scratch), _stream())
    return out


def segment_moments(x, off, out=None):
    n = off.numel() - 1
    out = torch.empty(n, 3, dtype=F64, device=x.device) if out is None else out
    _lib.call("accel_segment_moments", _p(x), _p(off), n, _p(out), _stream())
    return out


def count_nonfinite_rows(x, rows, R, count):
    _lib.call("accel_count_nonfinite_rows", _pp(x), _pp(rows), int(R), x.shape[1], x.stride(0),
              _pp(count),
              _stream())


def count_nonfinite(x, count):
    _lib.call("accel_count_nonfinite", _p(x), x.numel(), _p(count), _stream())


def step_finalize(loss_sums, loss_max, value_sums, bad_counts, attn_bad, algo, lambda_v, lambda_h,
                  n_tokens, n_transitions, record, skip):
    _lib.call("accel_step_finalize", _p(loss_sums), _p(loss_max), _p(value_sums), _p(bad_counts),
              _p(attn_bad), int(algo), float(lambda_v), float(lambda_h), float(n_tokens),
              float(n_transitions), _p(record), _p(skip), _stream())


def adam_dev(p_in, g, m_in, v_in, p_out, m_out, v_out, n0, hyper, skip, bad):
    """hyper: DEVICE f64[12], {lr, beta1, beta2, eps, 1-beta1^t, 1-beta2^t} of the
    two groups, read at run time (graph-replayable)."""
    _check(hyper, "hyper", F64, (12,))
    _lib.call("accel_adam_dev", _p(p_in), _p(g), _p(m_in), _p(v_in), _p(p_out), _p(m_out),
              _p(v_out), p_in.numel(), int(n0), _p(hyper), _p(skip), _p(bad), _stream())


def adam(p_in, g, m_in, v_in, p_out, m_out, v_out, n0, group0, group1, skip, bad):
    """group0/group1: HOST sequences {lr, beta1, beta2, eps, 1-beta1^t, 1-beta2^t}."""
    n = p_in.numel()
    h0 = (ctypes.c_double * 6)(*[float(x) for x in group0])
    h1 = (ctypes.c_double * 6)(*[float(x) for x in group1])
    _lib.call("accel_adam", _p(p_in), _p(g), _p(m_in), _p(v_in), _p(p_out), _p(m_out), _p(v_out),
              n, int(n0), h0, h1, _p(skip), _p(bad), _stream())


# ---------------------------------------------------------------------------
# tensor-core GEMM (tcgen05, 3xTF32)


def pitched(x):
    """x (2-D fp32) with 16-byte aligned rows: x itself when its row pitch is a
    multiple of 4 floats, else a copy with the pitch rounded up (the tensor-core
    GEMMs stream operands through TMA, which needs aligned rows).  Producers on
    the hot path allocate pitched storage up front (`alloc_pitched`)."""
    if x.stride(1) == 1 and x.stride(0) % 4 == 0 and x.data_ptr() % 16 == 0:
        return x
    out = alloc_pitched(x.shape[0], x.shape[1], x.device)
    out.copy_(x)
    return out


def copy_2d(dst, src):
    """dst[:] = src for 2-D tensors with unit column stride and any row pitch,
    one strided DMA (host <-> device)."""
    if dst.shape != src.shape or dst.stride(1) != 1 or src.stride(1) != 1:
        raise DimensionError("copy_2d: shapes/strides")
    es = dst.element_size()
    _lib.call("accel_copy_2d", _pp(dst), dst.stride(0) * es, _pp(src), src.stride(0) * es,
              dst.shape[1] * es, dst.shape[0], _stream())
    return dst


def upload_pitched(a, device, dtype=F32, staging=None):
    """Host array/tensor [rows, cols] -> pitched device storage (aligned rows):
    one contiguous H2D copy (full DMA rate; a row-strided DMA of short rows is
    several times slower) into `staging` (or a temporary), then a device-side
    re-pitch."""
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
    t = t.to(dtype).contiguous()
    out = alloc_pitched(t.shape[0], t.shape[1], device, dtype)
    if out.is_contiguous():
        return out.copy_(t, non_blocking=True)
    tmp = torch.empty(t.shape, dtype=dtype, device=device) if staging is None else staging
    tmp.copy_(t, non_blocking=True)
    return out.copy_(tmp)


def alloc_pitched(rows, cols, device, dtype=F32):
    """[rows, cols] view of a [rows, round_up(cols, 4)] buffer (aligned rows)."""
    pitch = -(-int(cols) // 4) * 4
    return torch.empty(rows, pitch, dtype=dtype, device=device)[:, :cols]


def tc_rows_supported(K: int, N: int) -> bool:
    """Shapes the tensor-core row transform takes (resident split weight):
    K, N <= 256.  Wider products (cfg4's D = 4096) use cuBLAS fp32 (TF32 off)."""
    return K <= 256 and N <= 256


# ---- wide products (cfg4: O = D = 4096): streamed tcgen05 tf32 + bf16-pair GEMM ----


def _pair_shape(rows: int, cols: int, row_pair: bool) -> tuple:
    c8 = -(-int(cols) // 8) * 8
    if row_pair:
        return (2 * (-(-int(rows) // 8) * 8), c8)
    return (int(rows), 2 * c8)


def tf32_pairs(x, row_pair: bool, lo_first: bool, out=None):
    """bf16 pair operand of fp32 x (accel_tf32_pairs): per 8-group along K,
    [bf16(hi) | bf16(lo)] ([lo | hi] with lo_first), hi = trunc19(x).  K runs
    along the columns (row_pair False, K-major use) or the rows (MN-major use)."""
    rows, cols = x.shape
    if x.stride(1) != 1:
        raise DimensionError("tf32_pairs: unit column stride required")
    shape = _pair_shape(rows, cols, row_pair)
    out = torch.empty(shape, dtype=torch.bfloat16, device=x.device) if out is None else out
    _lib.call("accel_tf32_pairs", _pp(x), rows, cols, x.stride(0), _pp(out), out.stride(0),
              int(row_pair), int(lo_first), _stream())
    return out


def _pairs_ws(tag: str, x, row_pair: bool, lo_first: bool):
    shape = _pair_shape(x.shape[0], x.shape[1], row_pair)
    n = shape[0] * shape[1]
    buf = stream_workspace("pair." + tag, 2 * n)
    return tf32_pairs(x, row_pair, lo_first, buf[:2 * n].view(torch.bfloat16).view(shape))


def wide_tiles(M: int, N: int, b_mn: bool) -> int:
    return int(_lib.lib().accel_tc_wide_tiles(int(M), int(N), int(bool(b_mn))))


def wide_gemm(a, b, out, *, a_mn: bool, b_mn: bool, epi: int = 0, bias=None, h=None,
              col_part=None, kslices: int = 1, tag: str = ""):
    """out = A . B^T on the streamed tensor-core kernel (accel_tc_gemm_wide):
    a is A [M, K] (a_mn False) or A^T stored [K, M]; b is B [N, K] (b_mn False)
    or B^T stored [K, N].  epi 0 store, 1 tanh(. + bias), 2 (.)(1 - h^2) with
    col_part[m_tiles, N] column sums, 3 split-K partial slices out[kslices, M, N]."""
    M = a.shape[1] if a_mn else a.shape[0]
    K = a.shape[0] if a_mn else a.shape[1]
    N = b.shape[1] if b_mn else b.shape[0]
    if (b.shape[0] if b_mn else b.shape[1]) != K:
        raise DimensionError(f"wide_gemm: inner dims {K} and {tuple(b.shape)}")
    a, b = pitched(a), pitched(b)
    ap = _pairs_ws(tag + "a", a, a_mn, False)
    bp = _pairs_ws(tag + "b", b, b_mn, True)
    ldc = N if epi == 3 else out.stride(0)
    _lib.call("accel_tc_gemm_wide", _pp(a), _pp(ap), _pp(b), _pp(bp), _pp(out), _pp(bias), _pp(h),
              _pp(col_part), M, N, K, a.stride(0), ap.stride(0), b.stride(0), bp.stride(0), ldc,
              h.stride(0) if h is not None else 0, int(a_mn), int(b_mn), int(epi), int(kslices),
              _stream())
    return out


def _wide_rows(x, b, out, b_mn: bool, bias=None, tanh=False):
    """out = act(x . B^T + bias) for wide shapes; few output tiles -> split-K
    partial slices summed in fixed order (deterministic)."""
    M, N = x.shape[0], out.shape[1]
    tiles = wide_tiles(M, N, b_mn)
    sms = tc_sm_count()
    if tanh:
        if bias is None:
            raise DimensionError("tanh epilogue needs the bias")
        return wide_gemm(x, b, out, a_mn=False, b_mn=b_mn, epi=1, bias=bias, tag="rows")
    ks = _wide_split(tiles, x.shape[1]) if tiles < sms // 2 and out.is_contiguous() else 1
    if ks > 1:
        part = stream_workspace("wide_part", 4 * ks * M * N)[:4 * ks * M * N].view(F32)
        wide_gemm(x, b, part, a_mn=False, b_mn=b_mn, epi=3, kslices=ks, tag="rows")
        reduce_segments([(part, out, ks, M * N, M * N)])
    else:
        wide_gemm(x, b, out, a_mn=False, b_mn=b_mn, epi=0, tag="rows")
    if bias is not None:
        out.add_(bias)
    return out


SMALL_FMAS = 1 << 26  # products up to 64 M FMAs with a short output run the SIMT kernel


def _small(M, N, K) -> bool:
    return M <= 512 and M * N * K <= SMALL_FMAS


def small_gemm(a, b, out, a_trans: bool, b_trans: bool):
    """out[M, N] = op(a) op(b)^T (accel_small_gemm): a is [M, K] or (a_trans) [K, M],
    b is [N, K] or (b_trans) [K, N]; unit column strides, any row pitch."""
    M = a.shape[1] if a_trans else a.shape[0]
    K = a.shape[0] if a_trans else a.shape[1]
    N = b.shape[1] if b_trans else b.shape[0]
    for t, nm in ((a, "a"), (b, "b"), (out, "out")):
        if t.stride(1) != 1:
            raise DimensionError(f"small_gemm: {nm} needs unit column stride")
    nws = int(_lib.lib().accel_small_gemm_ws_floats(M, N, K))
    ws = stream_workspace("small_gemm", 4 * nws) if nws else None
    _lib.call("accel_small_gemm", _pp(a), _pp(b), _pp(out), M, N, K, a.stride(0), b.stride(0),
              out.stride(0), int(a_trans), int(b_trans), _pp(ws), nws, _stream())
    return out


def tc_linear(x, w, out=None, bias=None, tanh=False, accumulate=False):
    """out[M, N] = act(x[M, K] . w[N, K]^T + bias) (+ out): y = x W^T as in models.py."""
    M, K = x.shape
    N = w.shape[0]
    out = torch.empty(M, N, dtype=F32, device=x.device) if out is None else out
    if bias is None and not tanh and not accumulate and _small(M, N, K):
        return small_gemm(x, w, out, False, False)
    if not tc_rows_supported(K, N):
        if accumulate:
            raise DimensionError("wide products do not accumulate")
        return _wide_rows(x, w, out, False, bias, tanh)
    x = pitched(x)
    _lib.call("accel_tc_gemm", _pp(x), _pp(w), _pp(out), _pp(bias), M, K, N, x.stride(0),
              w.stride(0), out.stride(0), 0, 0, int(tanh), int(accumulate), 1, _stream())
    return out


def tc_linear_checked(x, w, out, nonfinite, bias=None, tanh=False):
    """tc_linear that also adds the count of non-finite elements of x to
    `nonfinite` (i32/u32 device scalar)."""
    M, K = x.shape
    N = w.shape[0]
    if not tc_rows_supported(K, N):
        count_nonfinite_rows(x, None, M, nonfinite)  # counts rows, same decision
        return _wide_rows(x, w, out, False, bias, tanh)
    x = pitched(x)
    _lib.call("accel_tc_linear_checked", _pp(x), _pp(w), _pp(out), _pp(bias), M, K, N, x.stride(0),
              w.stride(0), out.stride(0), int(tanh), _pp(nonfinite), _stream())
    return out


def tc_matmul_nn(x, w, out=None, accumulate=False):
    """out[M, N] = x[M, K] . w[K, N] (w row-major, i.e. B given transposed)."""
    M, K = x.shape
    N = w.shape[1]
    out = torch.empty(M, N, dtype=F32, device=x.device) if out is None else out
    if not accumulate and _small(M, N, K):
        return small_gemm(x, w, out, False, True)
    if not tc_rows_supported(K, N):
        if accumulate:
            raise DimensionError("wide products do not accumulate")
        return _wide_rows(x, w, out, True)
    x = pitched(x)
    _lib.call("accel_tc_gemm", _pp(x), _pp(w), _pp(out), None, M, K, N, x.stride(0), w.stride(0),
              out.stride(0), 0, 1, 0, int(accumulate), 1, _stream())
    return out


def tc_rows_grid(M: int) -> int:
    return int(_lib.lib().accel_tc_rows_grid(int(M)))


def _aligned_rows(t) -> bool:
    return t.stride(1) == 1 and t.stride(0) % 4 == 0 and t.data_ptr() % 16 == 0


def tc_matmul_nn_dtanh(x, w, h, out, part_fn):
    """out = (x . w) * (1 - h^2) with per-CTA column sums of out; returns
    (out, col_part, n_parts).  part_fn(n) -> f32[n, N] buffer.  Falls back to
    the unfused product + accel_tanh_grad_colsum at unaligned widths."""
    x = pitched(x)
    M, K = x.shape
    N = w.shape[1]
    # fused for short K (the resident [W_hi; W_lo] leaves room for two H staging
    # boxes per epilogue warp) and, with H read by the epilogue lanes straight from
    # global memory, for narrow N (<= 64, whole 32-column chunks) up to K = 256
    if not tc_rows_supported(K, N):  # wide: the tanh derivative rides in the epilogue
        n = -(-M // 128)
        part = part_fn(n)
        wide_gemm(x, w, out, a_mn=False, b_mn=True, epi=2, h=pitched(h), col_part=part,
                  tag="dtanh")
        return out, part, n
    if (N <= 256 and (K <= 128 or (N <= 64 and N % 32 == 0)) and _aligned_rows(out)
            and _aligned_rows(h)):
        n = tc_rows_grid(M)
        part = part_fn(n)
        _lib.call("accel_tc_gemm_dtanh", _pp(x), _pp(w), _pp(out), _pp(h), _pp(part), M, K, N,
                  x.stride(0), w.stride(0), out.stride(0), h.stride(0), 1, _stream())
        return out, part, n
    tc_matmul_nn(x, w, out)
    n = rows_grid(M)
    part = part_fn(n)
    tanh_grad_colsum(out, h, part, n)
    return out, part, n


def tc_sm_count() -> int:
    return int(_lib.lib().accel_tc_sm_count())


def _wide_split(tiles: int, K: int) -> int:
    """Split-K slices filling the SMs, at most one per 16-k block (the kernel
    gives every slice at least one block)."""
    return max(1, min(tc_sm_count() // max(tiles, 1), -(-int(K) // 16)))


def wide_kslices(n: int, k: int, rows: int) -> int:
    """k slices of a wide weight gradient dW[n, k] = dy[rows, n]^T x[rows, k]."""
    return _wide_split(wide_tiles(n, k, True), rows)


def tc_wgrad(dy, x, out, kslices=None, partial=None):
    """out[n, k] = dy[F, n]^T . x[F, k] (reduction over the F rows): `kslices`
    persistent CTAs each produce two fp32 partials, reduced in fixed order
    (deterministic)."""
    F, n = dy.shape
    k = x.shape[1]
    if _small(n, k, F):
        return small_gemm(dy, x, out, True, True)
    dst = out if out.is_contiguous() else torch.empty(n, k, dtype=F32, device=dy.device)
    if n > 256 or k > 256:
        ks = wide_kslices(n, k, F)
        part = torch.empty(ks, n, k, dtype=F32, device=dy.device)
        wide_gemm(dy, x, part, a_mn=True, b_mn=True, epi=3, kslices=ks, tag="wgrad")
        reduce_segments([(part, dst, ks, n * k, n * k)])
        return out if dst is out else out.copy_(dst)
    dy, x = pitched(dy), pitched(x)
    if kslices is None:
        kslices = max(1, min(tc_sm_count(), -(-F // 32)))
    if partial is None:
        partial = torch.empty(2 * kslices, n, k, dtype=F32, device=dy.device)
    _lib.call("accel_tc_gemm", _pp(dy), _pp(x), _p(partial), None, n, F, k, dy.stride(0),
              x.stride(0), k, 1, 1, 0, 0, int(kslices), _stream())
    reduce_segments([(partial, dst, 2 * kslices, n * k, n * k)])
    return out if dst is out else out.copy_(dst)


# ---------------------------------------------------------------------------
# world-model training sub-steps (trainer.py:469-535), float64


def wm_mlp2_grad(x, target, din, dh, dout, kind, params, grads, loss, nonfinite):
    """Forward + backward of a 2-layer tanh MLP on the device (accel.h)."""
    n = x.shape[0]
    _check(x, "x", F64, (n, din))
    _check(params, "params", F64)
    nbytes = _lib.lib().accel_wm_workspace_size(n, dh, dout)
    buf = stream_workspace("wm", nbytes)
    _lib.call("accel_wm_mlp2_grad", _p(x), _p(target), n, din, dh, dout, int(kind), _p(params),
              _p(grads), _p(loss), _p(nonfinite), _p(buf), buf.numel(), _stream())


def wm_adam(params, grads, m, v, lr, beta1, beta2, eps, t, bad):
    _lib.call("accel_wm_adam", _p(params), _p(grads), _p(m), _p(v), params.numel(), float(lr),
              float(beta1), float(beta2), float(eps), int(t), _p(bad), _stream())
