"""TEST INFRASTRUCTURE — ctypes loader for the C restatement (gae_ref.c).

Built by `build_c_oracle()` (called from `__graft_entry__.build()`) into
oracle/_build/liboracle.so with gcc; the .so travels to the GPU box.
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "gae_ref.c"
LIB = HERE / "_build" / "liboracle.so"


def build_c_oracle() -> Path:
    LIB.parent.mkdir(exist_ok=True)
    if not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-o", str(LIB), str(SRC)], check=True)
    return LIB


_lib = None


def _handle():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build_c_oracle()
        _lib = ctypes.CDLL(str(LIB))
        p = ctypes.c_void_p
        _lib.oracle_gae_csr.argtypes = [p, p, p, p, ctypes.c_int64, ctypes.c_double,
                                        ctypes.c_double, p, p]
        _lib.oracle_sums.argtypes = [p, ctypes.c_int64, p, p]
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def gae_csr(rewards, values_frames, traj_off, done, gamma, lam):
    r = np.ascontiguousarray(rewards, dtype=np.float64)
    v = np.ascontiguousarray(values_frames, dtype=np.float64)
    off = np.ascontiguousarray(traj_off, dtype=np.int64)
    d = np.ascontiguousarray(done, dtype=np.uint8)
    adv = np.empty_like(r)
    ret = np.empty_like(r)
    _handle().oracle_gae_csr(_ptr(r), _ptr(v), _ptr(off), _ptr(d), off.shape[0] - 1,
                             float(gamma), float(lam), _ptr(adv), _ptr(ret))
    return adv, ret


def sums(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    s, q = ctypes.c_double(), ctypes.c_double()
    _handle().oracle_sums(_ptr(x), x.shape[0], ctypes.byref(s), ctypes.byref(q))
    return s.value, q.value
