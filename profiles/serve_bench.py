"""Serving throughput: DeviceServer.run_batch (inference.py:129-160) on policy
requests at the default harness dims (O = 195, K = 4, A = 7, D = 64).

    python profiles/serve_bench.py [batch ...]

Prints per batch size: the device-only launch time (accel_serve, CUDA events),
the end-to-end run_batch time (host requests in, response objects out) and the
float64 per-request restatement of the reference (oracle/imagine_ref.py) on
one core for a 256-request sample.
"""

import json
import sys
import time
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import imagine_ref  # noqa: E402
from paper_2603_18464_b200.publish import POLICY, VersionedWeights  # noqa: E402
from paper_2603_18464_b200.serve import DeviceServer, ticket_uniforms  # noqa: E402
from paper_2603_18464_b200.types import (ModelBundle, PolicyConfig, PolicyModel,  # noqa: E402
                                         ValueConfig, ValueHead)


def main():
    rng = np.random.default_rng(0)
    O, K, A, D = 195, 4, 7, 64
    pc = PolicyConfig(obs_dim=O, hidden_dim=D, chunk_len=K, n_actions=A, vocab_size=32,
                      action_start=16)
    b = ModelBundle(PolicyModel.init(rng, pc), ValueHead.init(rng, ValueConfig(D, 60, 32)))
    w = VersionedWeights(POLICY, 0, policy=b.policy, value=b.value)
    srv = DeviceServer()
    rows = []
    for n in [int(a) for a in sys.argv[1:]] or [64, 1024, 4096]:
        vecs = rng.normal(size=(n, O))
        reqs = [SimpleNamespace(ticket=i, kind=POLICY, obs=SimpleNamespace(vec=vecs[i], step=i % 60),
                                chunk=None) for i in range(n)]
        srv.run_batch(w, reqs, 0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            srv.run_batch(w, reqs, 0)
        e2e = (time.perf_counter() - t0) / 5
        # device-only: the launch on resident inputs
        from paper_2603_18464_b200 import _lib
        import ctypes
        wts, dims = srv._weights(w)
        dev = srv.device
        x = torch.from_numpy(vecs).to(dev)
        st = torch.tensor([i % 60 for i in range(n)], dtype=torch.int32, device=dev)
        u = torch.from_numpy(ticket_uniforms(0, range(n), K)).to(dev)
        tok = torch.empty(n, K, dtype=torch.int32, device=dev)
        lg = torch.empty(n, K, A, dtype=torch.float64, device=dev)
        val = torch.empty(n, dtype=torch.float64, device=dev)
        P = lambda t: ctypes.c_void_p(t.data_ptr())
        wp = (ctypes.c_void_p * 23)(*[t.data_ptr() for t in wts])
        call = lambda: _lib.call("accel_serve", wp, (ctypes.c_int * 8)(*dims), 0, P(x), P(st), None,
                                 P(u), n, P(tok), P(lg), P(val), None, None,
                                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        call()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            call()
        e1.record()
        torch.cuda.synchronize()
        dev_ms = e0.elapsed_time(e1) / 20
        rows.append({"batch": n, "device_ms": dev_ms, "device_requests_per_s": n / dev_ms * 1e3,
                     "e2e_ms": e2e * 1e3, "e2e_requests_per_s": n / e2e})
    # float64 per-request restatement on one core (the reference's algorithm)
    p, vp = b.policy.params.tensors, b.value.params.tensors
    m = 256
    vecs = rng.normal(size=(m, O))
    u = ticket_uniforms(0, range(m), K)
    t0 = time.perf_counter()
    for i in range(m):
        imagine_ref.sample_chunk(p, A, vecs[i], u[i])
        imagine_ref.state_value(p, vp, vecs[i], i % 60)
    cpu = m / (time.perf_counter() - t0)
    print(json.dumps({"kernel": "accel_serve (policy)", "rows": rows,
                      "cpu_port_requests_per_s": cpu, "cpu_cores": 1,
                      "cpu_sample": f"{m} requests, oracle/imagine_ref float64"}))


if __name__ == "__main__":
    main()
