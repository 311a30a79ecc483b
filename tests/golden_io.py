"""Readers for the golden fixtures written by tests/golden/make_golden.py."""

from __future__ import annotations

import json

import numpy as np

from conftest import GOLDEN
from paper_2603_18464_b200.types import Trajectory
from paper_2603_18464_b200.workload import PackedBatch

CASES = ("trainer_trust_revalue", "trainer_clip_stored", "trainer_cfg1_dims")


class Golden:
    def __init__(self, name: str) -> None:
        self.name = name
        self.z = dict(np.load(GOLDEN / f"{name}.npz"))
        self.meta = json.loads((GOLDEN / f"{name}.json").read_text())

    @property
    def cfg(self) -> dict:
        return self.meta["cfg"]

    def params(self, tag: str, which: str) -> dict:
        pre = f"{tag}{which}."
        return {k[len(pre):]: v for k, v in self.z.items() if k.startswith(pre)}

    def init_policy(self) -> dict:
        return self.params("init.", "policy")

    def init_value(self) -> dict:
        return self.params("init.", "value")

    def after(self, step: int, which: str) -> dict:
        return self.params(f"s{step}.after.", which)

    def packed(self, step: int) -> PackedBatch:
        g = lambda k: self.z[f"s{step}.{k}"]
        return PackedBatch(
            traj_off=g("traj_off"), frames=g("frames").astype(np.float32),
            steps=g("steps").astype(np.int32), values=g("values").astype(np.float32),
            tokens=g("tokens").astype(np.int32), rewards=g("rewards").astype(np.float32),
            mu=g("mu").astype(np.float32), done=g("done"), real=g("real"),
            behavior_version=g("bver"))

    def trajectories(self, step: int) -> list:
        g = lambda k: self.z[f"s{step}.{k}"]
        off = g("traj_off")
        out = []
        for s in range(off.shape[0] - 1):
            a, b = int(off[s]), int(off[s + 1])
            out.append(Trajectory(
                task_id=0, source="real" if g("real")[s] else "imagined",
                observations=g("frames")[a + s:b + s + 1], steps=g("steps")[a + s:b + s + 1],
                tokens=g("tokens")[a:b], rewards=g("rewards")[a:b],
                behavior_logits=g("mu")[a:b], values=g("values")[a + s:b + s],
                bootstrap_value=float(g("values")[b + s]), done=bool(g("done")[s]),
                behavior_version=int(g("bver")[s])))
        return out

    def batch(self, step: int) -> dict:
        pre = f"s{step}.batch."
        return {k[len(pre):]: v for k, v in self.z.items() if k.startswith(pre)}

    def record(self, step: int) -> dict:
        return self.meta["records"][step]

    def batch_meta(self, step: int) -> dict:
        return self.meta["batch_meta"][step]


IMAGINE_CASES = ("imagine_small", "imagine_default_dims", "imagine_done_hat", "imagine_nan_obs")


class ImagineGolden:
    def __init__(self, name: str) -> None:
        self.name = name
        self.z = dict(np.load(GOLDEN / f"{name}.npz"))
        self.meta = json.loads((GOLDEN / f"{name}.json").read_text())

    def params(self, which: str) -> dict:
        pre = which + "."
        return {k[len(pre):]: v for k, v in self.z.items() if k.startswith(pre)}

    @property
    def episodes(self) -> list:
        return self.meta["episodes"]

    def start(self, e: int):
        ep = self.episodes[e]
        return self.z[f"e{e}.start_vec"], ep["start_step"], ep["task_id"]

    def uniforms(self, e: int):
        return self.z[f"e{e}.uniforms"]

    def traj(self, e: int) -> dict:
        pre = f"e{e}."
        return {k[len(pre):]: v for k, v in self.z.items() if k.startswith(pre)}
