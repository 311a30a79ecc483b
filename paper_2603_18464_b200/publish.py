"""Versioned weight snapshots handed to the inference side.

Reference: `Trainer.publish_policy` deep-clones the whole bundle on every
step (trainer.py:328-334) and wraps it in `VersionedWeights`
(inference.py:107-126).  Here a snapshot is one device-to-device copy of the
flat parameter buffer (~0.2 MB at D=64); host model objects are built only if
a consumer reads `.policy` / `.value`, so publication never forces a
device-to-host copy onto the optimizer's critical path.
"""

from __future__ import annotations

POLICY = "policy"
OBS_MODEL = "obs_model"
REWARD_MODEL = "reward_model"


class VersionedWeights:
    """Duck-types inference.VersionedWeights (kind, version, policy, value, ...)."""

    def __init__(self, kind: str, version: int, flat=None, owner=None, policy=None, value=None,
                 obs_model=None, reward_model=None) -> None:
        self.kind = kind
        self.version = version
        self.flat = flat          # device snapshot of the flat parameter buffer
        self._owner = owner
        self._policy = policy
        self._value = value
        self.obs_model = obs_model
        self.reward_model = reward_model

    @classmethod
    def from_device(cls, kind: str, version: int, trainer) -> "VersionedWeights":
        flat = trainer.params.p[trainer.params.cur].clone()
        return cls(kind, version, flat=flat, owner=trainer)

    def _materialize(self) -> None:
        if self._policy is not None or self._owner is None:
            return
        tr = self._owner
        host = self.flat.cpu().numpy()
        pol, val = tr.params._split(host)
        b = tr._bundle
        self._policy = b.policy.with_params(type(b.policy.params)(pol, self.version))
        self._value = b.value.with_params(type(b.value.params)(val, self.version))

    @property
    def policy(self):
        self._materialize()
        return self._policy

    @property
    def value(self):
        self._materialize()
        return self._value
