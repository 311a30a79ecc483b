"""CPU: the per-ticket uniforms of the device server equal the reference's
per-token rng.random() draws, and the float64 restatement (oracle/imagine_ref)
fed with them reproduces the reference run_batch fixture bit-for-bit on tokens."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import imagine_ref
from paper_2603_18464_b200.serve import ticket_uniforms
from serve_fixture import ServeGolden


def test_ticket_uniforms_are_the_reference_draw_sequence():
    u = ticket_uniforms(7, [3, 10**9 + 1, 42], 5)
    for row, t in zip(u, [3, 10**9 + 1, 42]):
        rng = np.random.default_rng(np.random.SeedSequence([7, t]))  # inference.py:147
        np.testing.assert_array_equal(row, [rng.random() for _ in range(5)])


def test_oracle_reproduces_reference_run_batch():
    g = ServeGolden()
    m, z = g.meta, g.z
    p, vp = g.params("pol_"), g.params("val_")
    u = ticket_uniforms(m["base_seed"], z["tickets"], m["K"])
    for i in range(len(z["tickets"])):
        toks, lg = imagine_ref.sample_chunk(p, m["A"], z["vecs"][i], u[i])
        np.testing.assert_array_equal(toks, z["tokens"][i])
        np.testing.assert_allclose(lg, z["logits"][i], rtol=0, atol=1e-12)
        v = imagine_ref.state_value(p, vp, z["vecs"][i], int(z["steps"][i]))
        assert abs(v - z["values"][i]) <= 1e-12


@pytest.mark.parametrize("base_seed", [0, 7, 123, 2 ** 32 - 1, 2 ** 32, 2 ** 40 + 5, 2 ** 63 + 11])
def test_kernel_ticket_draws_equal_numpy(base_seed):
    """accel_ticket_uniforms' arithmetic (the host twin of the serving kernel):
    SeedSequence([base_seed, ticket]) + PCG64 + random() restated per ticket,
    bitwise equal to numpy's draws, incl. zero and multi-word integers."""
    import ctypes

    from paper_2603_18464_b200 import _lib
    if not _lib.LIB_PATH.exists():
        pytest.skip("libaccel.so not built")
    rng = np.random.default_rng(base_seed % 1000)
    t = np.array([0, 1, 2, 3, 10 ** 9 + 1, 2 ** 32 - 1, 2 ** 32, 2 ** 33 + 7, 2 ** 62]
                 + rng.integers(0, 2 ** 40, size=40).tolist(), dtype=np.int64)
    for K in (1, 4, 7):
        out = np.empty((len(t), K))
        rc = _lib.lib().accel_ticket_uniforms_host(
            ctypes.c_uint64(base_seed), t.ctypes.data_as(ctypes.c_void_p), len(t), K,
            out.ctypes.data_as(ctypes.c_void_p))
        assert rc == 0
        np.testing.assert_array_equal(out, ticket_uniforms(base_seed, t.tolist(), K))
