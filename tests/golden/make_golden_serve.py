"""Golden fixtures for batched serving, made by the REAL reference's
`inference.run_batch` (inference.py:129-160) in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_serve.py

Policy, obs-model and reward-model batches (default harness dims: 8x8 grid,
O = 195, K = 4, A = 7, D = 64) with arbitrary tickets and base seed; the
fixture stores the requests (observation vectors, steps, chunks, tickets), the
weights and every response.  The GPU box reads only the .npz.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from asyncrl.env import Observation  # noqa: E402
from asyncrl.inference import (InferenceRequest, OBS_MODEL, POLICY, REWARD_MODEL,  # noqa: E402
                               VersionedWeights, run_batch)
from asyncrl.models import (ModelBundle, ObsModel, ObsModelConfig, PolicyConfig,  # noqa: E402
                            PolicyModel, RewardModel, ValueConfig, ValueHead)

OUT = Path(__file__).resolve().parent


def main() -> None:
    rng = np.random.default_rng(11)
    O, K, A, D = 195, 4, 7, 64
    pc = PolicyConfig(obs_dim=O, hidden_dim=D, chunk_len=K, n_actions=A, vocab_size=32,
                      action_start=16)
    bundle = ModelBundle(PolicyModel.init(rng, pc), ValueHead.init(rng, ValueConfig(D, 60, 32)),
                         ObsModel.init(rng, ObsModelConfig(obs_dim=O, chunk_len=K, n_actions=A)),
                         RewardModel.init(rng, O))
    n = 37
    vecs = np.zeros((n, O))
    for i in range(n):  # one-hot grid planes + task one-hot, like the suite's observations
        for c in range(3):
            vecs[i, c * 64 + rng.integers(64)] = 1.0
        vecs[i, 192 + rng.integers(3)] = 1.0
    vecs[:5] += rng.normal(scale=0.3, size=(5, O))  # off-grid inputs too
    steps = rng.integers(0, 60, size=n)
    tickets = rng.integers(0, 10**9, size=n)
    chunks = rng.integers(0, A, size=(n, K))
    base_seed = 1234
    out = {"vecs": vecs, "steps": steps, "tickets": tickets, "chunks": chunks}
    for pre, params in (("pol_", bundle.policy.params), ("val_", bundle.value.params),
                        ("obs_", bundle.obs_model.params), ("rew_", bundle.reward_model.params)):
        out.update({pre + k: v for k, v in params.tensors.items()})
    for kind in (POLICY, OBS_MODEL, REWARD_MODEL):
        w = VersionedWeights.from_bundle(kind, 3, bundle)
        reqs = [InferenceRequest(int(tickets[i]), kind, Observation(vecs[i], int(steps[i]), 0),
                                 chunks[i] if kind == OBS_MODEL else None, 0.0, None)
                for i in range(n)]
        res = run_batch(w, reqs, base_seed)
        if kind == POLICY:
            out["tokens"] = np.stack([r.tokens for r in res])
            out["logits"] = np.stack([r.logits for r in res])
            out["values"] = np.array([r.value for r in res])
        elif kind == OBS_MODEL:
            out["next_obs"] = np.stack([r.next_obs for r in res])
        else:
            out["probs"] = np.array([r.probability for r in res])
    np.savez_compressed(OUT / "serve_default_dims.npz", **out)
    (OUT / "serve_default_dims.json").write_text(json.dumps(
        {"O": O, "K": K, "A": A, "D": D, "vocab": 32, "action_start": 16, "n_steps": 60,
         "mlp_hidden": 32, "obs_hidden": 96, "reward_hidden": 64, "base_seed": base_seed,
         "version": 3}, indent=1))
    print("tokens[:3]", out["tokens"][:3].tolist(), "values[:3]", out["values"][:3].tolist())


if __name__ == "__main__":
    main()
