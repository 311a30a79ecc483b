"""ctypes binding of libaccel.so (the C ABI in include/accel.h).

There is no fallback: if the library is missing or no CUDA device is
present, every op raises AccelError.  Build with
`python -m paper_2603_18464_b200.build`.
"""

from __future__ import annotations

import ctypes
from ctypes import c_double, c_int, c_int64, c_size_t, c_uint64, c_void_p
from pathlib import Path

from .errors import AccelError, raise_for_status

LIB_PATH = Path(__file__).resolve().parent / "libaccel.so"

P = c_void_p
# name -> (restype, argtypes)
_SIGNATURES = {
    "accel_last_error": (ctypes.c_char_p, []),
    "accel_launch_count": (ctypes.c_ulonglong, []),
    "accel_version": (c_int, []),
    "accel_build_id": (ctypes.c_char_p, []),
    "accel_copy_2d": (c_int, [P, c_size_t, P, c_size_t, c_size_t, c_size_t, P]),
    "accel_gae_workspace_size": (c_size_t, [c_int64, c_int64]),
    "accel_gae_segmented": (c_int, [P, P, P, P, c_int64, c_int64, c_double, c_double,
                                    P, P, P, P, P, c_size_t, P]),
    "accel_normalize_finalize": (c_int, [P, c_double, P, P]),
    "accel_normalize_apply": (c_int, [P, c_int64, P, P, P]),
    "accel_token_grid": (c_int, [c_int64]),
    "accel_token_logp": (c_int, [P, P, c_int64, c_int, P, P, P]),
    "accel_token_loss": (c_int, [P, P, P, P, P, c_int64, c_int, c_int, c_int, c_double,
                                 c_double, c_double, c_double, P, P, P, P, P, P, P]),
    "accel_bias_tanh": (c_int, [P, P, c_int64, c_int, P]),
    "accel_build_c": (c_int, [P, P, P, P, P, c_int64, c_int, c_int, c_int, P, P]),
    "accel_rows_grid": (c_int, [c_int64]),
    "accel_dc_reduce": (c_int, [P, P, P, c_int64, c_int, c_int, P, P, P, c_int, P]),
    "accel_tanh_grad_colsum": (c_int, [P, c_int64, P, c_int64, c_int64, c_int, P, c_int, P]),
    "accel_prev_keys": (c_int, [P, c_int64, c_int, c_int, c_int, P, P]),
    "accel_fact_grid": (c_int, [c_int64]),
    "accel_fact_partials": (c_int64, [c_int64, c_int, c_int, c_int]),
    "accel_ep_plus": (c_int, [P, P, P, c_int, c_int, P, P]),
    "accel_token_loss_fact2": (c_int, [P, P, P, P, P, P, c_int64, c_int, c_int, c_int,
                                       c_double, c_double, c_double, c_double, P, P, P, P, P, P,
                                       P, P, P, P]),
    "accel_fact_group_sum": (c_int, [P, P, P, P, P, P, P, P, c_int, c_int, c_int, c_int, c_int,
                                     c_int64, P, P]),
    "accel_pk_marginals": (c_int, [P, c_int, c_int, P, P, P]),
    "accel_step_keys": (c_int, [P, P, c_int64, c_int, P, P, P]),
    "accel_group_workspace_size": (c_size_t, [c_int64, c_int]),
    "accel_group_max_pieces": (c_int64, [c_int64, c_int]),
    "accel_group_by_key": (c_int, [P, c_int64, c_int, P, P, P, P, c_size_t, P]),
    "accel_group_workspace_size_blocked": (c_size_t, [c_int64, c_int, c_int64]),
    "accel_group_max_pieces_blocked": (c_int64, [c_int64, c_int, c_int64]),
    "accel_group_blocks": (c_int64, [c_int64, c_int64]),
    "accel_group_by_key_blocked": (c_int, [P, c_int64, c_int, c_int64, P, P, P, P, P, P, c_int,
                                           P, P, P, P, c_size_t, P]),
    "accel_fold_workspace_size": (c_size_t, [c_int, c_int]),
    "accel_fact_group_sum2": (c_int, [P, P, P, P, P, c_int, P, P, P, P, c_int, c_int, c_int,
                                      c_int64, P, P]),
    "accel_wm_workspace_size": (c_size_t, [c_int64, c_int, c_int]),
    "accel_wm_mlp2_grad": (c_int, [P, P, c_int64, c_int, c_int, c_int, c_int, P, P, P, P, P,
                                   c_size_t, P]),
    "accel_wm_adam": (c_int, [P, P, P, P, c_int64, c_double, c_double, c_double, c_double,
                              c_int64, P, P]),
    "accel_serve": (c_int, [P, P, c_int, P, P, P, P, c_int64, P, P, P, P, P, P]),
    "accel_split_tf32": (c_int, [P, c_int64, P, P, P]),
    "accel_sorted_rows": (c_int, [P, P, P, c_int64, c_int, P, P, P, P]),
    "accel_fold_blocked_pieces": (c_int, [P, P, c_int, c_int, c_int, c_int, P, P, P]),
    "accel_grouped_rows_sum": (c_int, [P, c_int64, c_int, P, P, P, P, c_int, c_int64, P, P, P]),
    "accel_warp_grid": (c_int, [c_int64]),
    "accel_value_pool": (c_int, [P, P, P, P, c_int64, c_int, c_int, P, P, P, P, P, P, c_int,
                                 P]),
    "accel_value_head": (c_int, [P, P, P, P, P, c_int64, c_int, P, P, c_double, c_double,
                                 c_double, P, P, P, c_int, P]),
    "accel_value_attn_grad": (c_int, [P, P, P, P, P, c_int64, c_int, P, P, c_int, P]),
    "accel_value_attn_wgrad": (c_int, [P, P, P, P, c_int64, c_int, P, c_int, P]),
    "accel_value_attn_backward": (c_int, [P, P, P, P, P, c_int64, c_int, P, P, P, c_int, P]),
    "accel_reduce_segments": (c_int, [P, P, P, P, P, c_int, P]),
    "accel_segment_moments": (c_int, [P, P, c_int64, P, P]),
    "accel_count_nonfinite_rows": (c_int, [P, P, c_int64, c_int, c_int64, P, P]),
    "accel_reduce_f64": (c_int, [P, c_int64, c_int, c_int, P, P, P]),
    "accel_reduce_f64_scratch_size": (c_size_t, [c_int64, c_int]),
    "accel_step_finalize": (c_int, [P, P, P, P, P, c_int, c_double, c_double, c_double,
                                    c_double, P, P, P]),
    "accel_count_nonfinite": (c_int, [P, c_int64, P, P]),
    "accel_adam": (c_int, [P, P, P, P, P, P, P, c_int64, c_int64, P, P, P, P, P]),
    "accel_adam_dev": (c_int, [P, P, P, P, P, P, P, c_int64, c_int64, P, P, P, P]),
    "accel_tc_sm_count": (c_int, []),
    "accel_tc_gemm_wide": (c_int, [P, P, P, P, P, P, P, P, c_int64, c_int64, c_int64, c_int64,
                                   c_int64, c_int64, c_int64, c_int64, c_int64, c_int, c_int,
                                   c_int, c_int, P]),
    "accel_tc_wide_tiles": (c_int, [c_int64, c_int64, c_int]),
    "accel_small_gemm": (c_int, [P, P, P, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64,
                                 c_int, c_int, P, c_int64, P]),
    "accel_small_gemm_ws_floats": (c_int64, [c_int64, c_int64, c_int64]),
    "accel_ticket_uniforms": (c_int, [ctypes.c_uint64, P, c_int64, c_int, P, P]),
    "accel_ticket_uniforms_host": (c_int, [ctypes.c_uint64, P, c_int64, c_int, P]),
    "accel_tc_wide_set_chunk": (None, [c_int]),
    "accel_tc_wide_set_multicast": (None, [c_int]),
    "accel_tf32_pairs": (c_int, [P, c_int64, c_int64, c_int64, P, c_int64, c_int, c_int, P]),
    "accel_tc_rows_grid": (c_int, [c_int64]),
    "accel_tc_linear_checked": (c_int, [P, P, P, P, c_int64, c_int64, c_int, c_int64, c_int64,
                                        c_int64, c_int, P, P]),
    "accel_tc_gemm_dtanh": (c_int, [P, P, P, P, P, c_int64, c_int64, c_int, c_int64, c_int64,
                                    c_int64, c_int64, c_int, P]),
    "accel_tc_gemm": (c_int, [P, P, P, P, c_int64, c_int64, c_int, c_int64, c_int64, c_int64,
                              c_int, c_int, c_int, c_int, c_int, P]),
    "accel_imagine_smem_bytes": (c_size_t, [c_int, c_int, c_int, c_int, c_int, c_int]),
    "accel_imagine": (c_int, [P, P, c_int, c_double, c_uint64, P, P, P, c_int64, P, P, P, P, P,
                              P, P, P, P, P, P]),
}

_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise AccelError(f"{LIB_PATH} not built; run `python -m paper_2603_18464_b200.build`")
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _check_build(handle)
        _lib = handle
    return _lib


def _check_build(handle) -> None:
    """The library must be built from the sources beside it (build.py's id);
    a stale libaccel.so raises instead of running old kernels."""
    from . import build as _build
    if not _build.CSRC.exists():  # an installed copy without sources: nothing to compare
        return
    have = handle.accel_build_id().decode()
    want = _build.build_id()
    if have != want:
        raise AccelError(f"{LIB_PATH} is stale (built from {have}, sources are {want}); "
                         "run `python -m paper_2603_18464_b200.build`")


def build_id() -> str:
    return lib().accel_build_id().decode()


def call(name: str, *args) -> None:
    """Invoke an int-status entry point; map a non-zero status to the
    reference exception types (include/accel.h conventions)."""
    handle = lib()
    status = getattr(handle, name)(*args)
    if status:
        raise_for_status(status, handle.accel_last_error().decode(errors="replace"))


def launch_count() -> int:
    return int(lib().accel_launch_count())


def exported_symbols() -> list:
    return sorted(_SIGNATURES)


def c_u64(x: int) -> c_uint64:
    return c_uint64(x)
