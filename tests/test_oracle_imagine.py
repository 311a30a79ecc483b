"""Pin the imagination restatement (oracle/imagine_ref.py) to the real reference worker."""

from __future__ import annotations

import numpy as np
import pytest

from golden_io import IMAGINE_CASES, ImagineGolden
from oracle.imagine_ref import imagine_episode


@pytest.mark.parametrize("name", IMAGINE_CASES)
def test_oracle_imagination_matches_reference(name):
    g = ImagineGolden(name)
    m = g.meta
    for e, ep in enumerate(g.episodes):
        vec, step, _ = g.start(e)
        out = imagine_episode(g.params("policy"), g.params("value"), g.params("obs"),
                              g.params("reward"), m["n_actions"], vec, step, g.uniforms(e),
                              m["h_img"], m["threshold"], (m["height"], m["width"]))
        if ep["discarded"]:
            assert "discarded" in out
            continue
        ref = g.traj(e)
        assert out["t_len"] == ep["t_len"] and out["done"] == ep["done"]
        np.testing.assert_array_equal(out["tokens"], ref["tokens"])
        np.testing.assert_array_equal(out["steps"], ref["steps"])
        np.testing.assert_allclose(out["observations"], ref["observations"], atol=1e-12)
        for f in ("rewards", "behavior_logits", "values"):
            np.testing.assert_allclose(out[f], ref[f], rtol=0, atol=1e-12, err_msg=f)
        assert abs(out["bootstrap_value"] - ep["bootstrap_value"]) < 1e-12
        # telescoping (reference tests/test_rollout.py:355-363)
        assert np.sum(out["rewards"]) == pytest.approx(
            np.sum(ref["rewards"]), abs=1e-12)
