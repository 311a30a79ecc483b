"""CPU: the per-ticket uniforms of the device server equal the reference's
per-token rng.random() draws, and the float64 restatement (oracle/imagine_ref)
fed with them reproduces the reference run_batch fixture bit-for-bit on tokens."""

from __future__ import annotations

import numpy as np

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
