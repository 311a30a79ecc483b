"""cfg4 GEMM micro-benchmark: the streamed tf32 + bf16-pair tcgen05 kernel
(accel_tc_gemm_wide) on the OpenVLA-7B-shaped products (F = 8256 frame rows,
O = D = 4096) against cuBLAS (TF32 x1 and the 3xTF32 it replaced).

    python profiles/wide_bench.py > gpurun_out/wide_bench.json
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_18464_b200 import ops  # noqa: E402


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    F, D = 8256, 4096
    dev = "cuda"
    x = torch.randn(F, D, device=dev)
    w = torch.randn(D, D, device=dev) / 64
    b = torch.randn(D, device=dev)
    h = torch.tanh(torch.randn(F, D, device=dev))
    out = torch.empty(F, D, device=dev)
    rows = []
    flops = 2.0 * F * D * D

    def case(name, run, pairs):
        ms = timed(run)
        mp = timed(pairs)
        rows.append({"product": name, "ms_gemm": ms, "ms_pairs": mp,
                     "tflops_fp32_eq": flops / ms / 1e9})

    ap = ops._pairs_ws("ba", x, False, False)
    bp = ops._pairs_ws("bb", w, False, True)
    bpn = ops._pairs_ws("bn", w, True, True)
    apm = ops._pairs_ws("bam", x, True, False)
    hpm = ops._pairs_ws("bhm", h, True, True)
    part = torch.empty(-(-F // 128), D, device=dev)
    wg = torch.empty(D, D, device=dev)

    def call(a, apair, bb, bpair, c, epi, a_mn, b_mn, M, N, K, bias=None, H=None, cp=None):
        from paper_2603_18464_b200 import _lib
        _lib.call("accel_tc_gemm_wide", ops._p(a), ops._p(apair), ops._p(bb), ops._p(bpair),
                  ops._p(c), ops._p(bias), ops._p(H), ops._p(cp), M, N, K, a.stride(0),
                  apair.stride(0), bb.stride(0), bpair.stride(0), c.stride(0),
                  H.stride(0) if H is not None else 0, a_mn, b_mn, epi, 1, ops._stream())

    from paper_2603_18464_b200 import _lib
    chunk = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    mcast = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    _lib.lib().accel_tc_wide_set_chunk(chunk)
    _lib.lib().accel_tc_wide_set_multicast(mcast)
    case("fwd x.W^T + b, tanh (K-major x K-major)",
         lambda: call(x, ap, w, bp, out, 1, 0, 0, F, D, D, bias=b),
         lambda: (ops.tf32_pairs(x, False, False, ap), ops.tf32_pairs(w, False, True, bp)))
    case("bwd (dz . W)(1 - h^2) + col sums (K-major x MN-major)",
         lambda: call(x, ap, w, bpn, out, 2, 0, 1, F, D, D, H=h, cp=part),
         lambda: (ops.tf32_pairs(x, False, False, ap), ops.tf32_pairs(w, True, True, bpn)))
    case("wgrad dz^T h (MN-major x MN-major, K = F)",
         lambda: call(x, apm, h, hpm, wg, 0, 1, 1, D, D, F),
         lambda: (ops.tf32_pairs(x, True, False, apm), ops.tf32_pairs(h, True, True, hpm)))
    torch.backends.cuda.matmul.allow_tf32 = True
    t1 = timed(lambda: torch.mm(x, w.t(), out=out))
    t3 = timed(lambda: (torch.mm(x, w.t(), out=out), out.addmm_(x, w.t()), out.addmm_(x, w.t())))
    torch.backends.cuda.matmul.allow_tf32 = False
    t32 = timed(lambda: torch.mm(x, w.t(), out=out), reps=3)
    print(json.dumps({"shape": {"F": F, "D": D}, "chunk_kblocks": chunk, "multicast": mcast,
                      "rows": rows,
                      "cublas_tf32_x1_ms": t1, "cublas_3xtf32_ms": t3, "cublas_fp32_ms": t32,
                      "tf32_dense_peak_tflops_at_1965mhz": 148 * 4096 * 1.965e9 / 1e12}))


if __name__ == "__main__":
    main()
