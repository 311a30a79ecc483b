"""Build libaccel.so (all csrc/*.cu) in-tree for sm_100a with nvcc.

`python -m paper_2603_18464_b200.build` or `__graft_entry__.build()`.
Objects go to paper_2603_18464_b200/_build/, the shared library next to
this file so it travels with the repo snapshot to the GPU box.

Provenance: the build id is a hash of every source (csrc/*.cu, *.cuh,
include/*.h) and the compiler flags.  It is compiled into the library
(`accel_build_id()`) and recorded with each object's own key in
_build/manifest.json; an object is recompiled when its key changes (content,
not mtimes), and `_lib.lib()` refuses a library whose id does not match the
sources beside it (a stale .so never runs silently).
"""

from __future__ import annotations

import hashlib
import json
import os
import shlex
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libaccel.so"
MANIFEST = BUILD / "manifest.json"
INCLUDE = PKG.parent / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# ACCEL_NVCC_DEFS: extra -D tuning defines (part of the build id), e.g. for sweeps
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
         "--expt-relaxed-constexpr", "-I", str(INCLUDE)] + \
    shlex.split(os.environ.get("ACCEL_NVCC_DEFS", ""))


def _flags_key() -> bytes:
    """The compiler flags without machine-specific paths (the repo moves)."""
    return " ".join(ARCH + [f for f in FLAGS if f != str(INCLUDE)]).encode()


def _sha(*parts: bytes) -> str:
    h = hashlib.sha256()
    for p in parts:
        h.update(p)
        h.update(b"\0")
    return h.hexdigest()[:16]


def _deps_hash() -> str:
    files = sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))
    return _sha(*(f.name.encode() + f.read_bytes() for f in files))


def build_id() -> str:
    """Hash of every source and the flags: what the library must report."""
    srcs = sorted(CSRC.glob("*.cu"))
    return _sha(_deps_hash().encode(), _flags_key(),
                *(f.name.encode() + f.read_bytes() for f in srcs))


def _key(src: Path, deps: str, bid: str) -> str:
    extra = bid.encode() if src.name == "abi.cu" else b""
    return _sha(src.read_bytes(), deps.encode(), _flags_key(), extra)


def _compile(src: Path, key: str, old: dict, bid: str, verbose: bool):
    obj = BUILD / (src.stem + ".o")
    if obj.exists() and old.get(src.name) == key:
        return obj, False
    cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
    if src.name == "abi.cu":
        cmd.insert(1, f'-DACCEL_BUILD_ID="{bid}"')
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr:
        sys.stderr.write(res.stderr)
    return obj, True


def build(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    sources = sorted(CSRC.glob("*.cu"))
    deps, bid = _deps_hash(), build_id()
    old = {}
    if MANIFEST.exists() and not force:
        try:
            old = json.loads(MANIFEST.read_text()).get("objects", {})
        except (OSError, ValueError):
            old = {}
    keys = {s.name: _key(s, deps, bid) for s in sources}
    with ThreadPoolExecutor(max_workers=min(8, len(sources))) as ex:
        done = list(ex.map(lambda s: _compile(s, keys[s.name], old, bid, verbose), sources))
    compiled = [s.name for s, (_, new) in zip(sources, done) if new]
    prev_lib = None
    if MANIFEST.exists():
        try:
            prev_lib = json.loads(MANIFEST.read_text()).get("build_id")
        except (OSError, ValueError):
            prev_lib = None
    if compiled or not LIB.exists() or prev_lib != bid or force:
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *(str(o) for o, _ in done),
               "-lcudart_static", "-Xcompiler", "-fPIC"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc link failed:\n{res.stdout}\n{res.stderr}")
        linked = True
    else:
        linked = False
    MANIFEST.write_text(json.dumps({"build_id": bid, "objects": keys, "compiled": compiled,
                                    "linked": linked, "nvcc_flags": ARCH + FLAGS}, indent=1))
    print(f"libaccel build {bid}: compiled {len(compiled)}/{len(sources)} "
          f"({', '.join(compiled) or 'up to date'}), linked={linked}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    path = build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(path)
