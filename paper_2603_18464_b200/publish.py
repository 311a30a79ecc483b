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
                 obs_model=None, reward_model=None, split=None, template=None,
                 layout=None) -> None:
        self.kind = kind
        self.version = version
        self.flat = flat          # device snapshot of the flat parameter buffer
        self.layout = layout      # params.FlatLayout of `flat` (device consumers slice it)
        self._owner = owner
        self._split = split       # host flat -> (policy, value) tensors (receivers)
        self._template = template  # bundle whose model classes / configs the views reuse
        self._policy = policy
        self._value = value
        self.obs_model = obs_model
        self.reward_model = reward_model

    @classmethod
    def from_device(cls, kind: str, version: int, trainer) -> "VersionedWeights":
        flat = trainer.params.p[trainer.params.cur].clone()
        return cls(kind, version, flat=flat, owner=trainer, layout=trainer.layout)

    def _materialize(self) -> None:
        if self._policy is not None or (self._owner is None and self._split is None):
            return
        host = self.flat.cpu().numpy()
        if self._owner is not None:
            pol, val = self._owner.params._split(host)
            b = self._owner._bundle
        else:
            pol, val = self._split(host)
            b = self._template
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


def broadcast_policy(snapshot, template, src: int = 0, group=None, device=None,
                     pad_to: int = 4):
    """Ship a policy snapshot from the trainer rank to every rank of `group`
    (reference: publish_policy's deep clone handed to
    InferenceService.update_weights in-process, trainer.py:328-334,
    inference.py:237-257).  Collective: every rank calls it; `src` passes its
    `VersionedWeights` (from Trainer.snapshot()), the others None.  One int64
    header {version, numel} and the flat float32 buffer travel over
    torch.distributed (NCCL over NVLink on B200s: ~0.2 MB at D = 64, no host
    copy); receivers get a VersionedWeights whose .policy / .value views are
    built from `template` (a bundle with the same configs) on first access.
    `pad_to` must match the trainer's layout (4 * data-parallel world)."""
    import torch
    import torch.distributed as dist

    from .params import Dims, FlatLayout

    rank = dist.get_rank(group)
    layout = FlatLayout(Dims.from_models(template.policy, template.value), pad_to=pad_to)
    if device is None:
        device = (torch.device("cuda", torch.cuda.current_device())
                  if dist.get_backend(group) == "nccl" else torch.device("cpu"))
    if rank == src:
        flat = snapshot.flat.to(device)
        hdr = torch.tensor([int(snapshot.version), flat.numel()], dtype=torch.int64, device=device)
    else:
        hdr = torch.zeros(2, dtype=torch.int64, device=device)
    dist.broadcast(hdr, src=dist.get_global_rank(group, src) if group is not None else src,
                   group=group)
    version, numel = int(hdr[0].item()), int(hdr[1].item())
    if numel != layout.total:
        from .errors import DimensionError
        raise DimensionError(f"snapshot has {numel} entries, the template layout {layout.total}")
    if rank != src:
        flat = torch.empty(numel, dtype=torch.float32, device=device)
    dist.broadcast(flat, src=dist.get_global_rank(group, src) if group is not None else src,
                   group=group)
    if rank == src:
        return snapshot
    return VersionedWeights(POLICY, version, flat=flat, split=layout.split, template=template,
                            layout=layout)
