"""Loader for the world-model sub-step fixtures (tests/golden/wm_*.npz)."""

from __future__ import annotations

import json
from pathlib import Path
from types import SimpleNamespace

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
WM_CASES = ["subsampled", "full"]


class WmGolden:
    def __init__(self, name: str) -> None:
        self.meta = json.loads((GOLDEN / f"wm_{name}.json").read_text())
        self.z = np.load(GOLDEN / f"wm_{name}.npz")

    def params(self, prefix: str) -> dict:
        return {k[len(prefix):]: self.z[k] for k in self.z.files if k.startswith(prefix)}

    def trajectories(self):
        return [SimpleNamespace(observations=self.z[f"traj{i}_obs"],
                                tokens=self.z[f"traj{i}_tokens"],
                                rewards=self.z[f"traj{i}_rewards"])
                for i in range(len(self.meta["lens"]))]

    def after(self, step: int) -> dict:
        return self.params(f"step{step}_")
