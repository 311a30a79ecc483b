"""Loader for the batched-serving fixture (tests/golden/make_golden_serve.py)."""

from __future__ import annotations

import json
from pathlib import Path
from types import SimpleNamespace

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


class ServeGolden:
    def __init__(self, name: str = "default_dims") -> None:
        self.meta = json.loads((GOLDEN / f"serve_{name}.json").read_text())
        self.z = np.load(GOLDEN / f"serve_{name}.npz")

    def params(self, prefix: str) -> dict:
        return {k[len(prefix):]: self.z[k] for k in self.z.files if k.startswith(prefix)}

    def requests(self, kind: str):
        z = self.z
        return [SimpleNamespace(ticket=int(z["tickets"][i]), kind=kind,
                                obs=SimpleNamespace(vec=z["vecs"][i], step=int(z["steps"][i])),
                                chunk=z["chunks"][i])
                for i in range(len(z["tickets"]))]
