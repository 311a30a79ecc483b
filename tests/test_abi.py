"""The C ABI library loads without a GPU and exports every symbol include/accel.h declares."""

from __future__ import annotations

import re

import pytest

from conftest import ROOT


def header_symbols() -> set:
    text = (ROOT / "include" / "accel.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(accel_\w+)\s*\(", text))


def test_library_exports_every_header_symbol():
    from paper_2603_18464_b200 import _lib

    if not _lib.LIB_PATH.exists():
        pytest.skip("libaccel.so not built (run __graft_entry__.build())")
    handle = _lib.lib()  # loads; no CUDA device needed
    missing = [s for s in sorted(header_symbols()) if not hasattr(handle, s)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    from paper_2603_18464_b200 import _lib

    assert header_symbols() == set(_lib.exported_symbols())


def test_status_codes_map_to_reference_exceptions():
    from paper_2603_18464_b200.errors import (AccelError, DimensionError, DomainError,
                                              NonFiniteError, raise_for_status)

    for status, exc in ((1, DomainError), (2, DimensionError), (3, NonFiniteError),
                        (4, AccelError)):
        with pytest.raises(exc, match="boom"):
            raise_for_status(status, "boom")
    raise_for_status(0, "")


def test_host_validation_without_device():
    """Config validation mirrors trainer.py:44-72 / :282-286 and needs no GPU."""
    from paper_2603_18464_b200.errors import DomainError
    from paper_2603_18464_b200.trainer import GaeConfig, LossConfig, TrainerConfig

    for bad in (lambda: GaeConfig(gamma=0.0), lambda: GaeConfig(lam=1.5),
                lambda: LossConfig(algorithm="ppo"), lambda: LossConfig(sigma=0.0),
                lambda: LossConfig(clip_eps=1.0), lambda: LossConfig(lambda_v=-0.1),
                lambda: TrainerConfig(k_shards=0)):
        with pytest.raises(DomainError):
            bad()


def test_packing_roundtrip_and_layout(rng):
    import numpy as np

    from paper_2603_18464_b200.workload import (pack_trajectories, synthetic_trajectories,
                                                unpack_trajectories)

    trajs = synthetic_trajectories(rng, [3, 1, 5], [True, False, True], 2, 7, 6)
    pb = pack_trajectories(trajs)
    assert pb.traj_off.tolist() == [0, 3, 4, 9]
    assert pb.n_frames == 12 and pb.frames.shape == (12, 6)
    np.testing.assert_array_equal(pb.frame_rows(), [0, 1, 2, 4, 6, 7, 8, 9, 10])
    assert pb.transition_frame_mask().sum() == 9
    back = unpack_trajectories(pb)
    for a, b in zip(trajs, back):
        np.testing.assert_array_equal(a.tokens, b.tokens)
        np.testing.assert_allclose(a.rewards, b.rewards, rtol=1e-6)
        assert a.done == b.done and a.t_len == b.t_len


def test_library_matches_its_sources(monkeypatch):
    """Build provenance: the loaded library reports the hash of the sources it
    was built from, and a library whose id does not match them is refused."""
    from paper_2603_18464_b200 import _lib, build
    from paper_2603_18464_b200.errors import AccelError
    assert _lib.build_id() == build.build_id()
    handle = _lib.lib()
    monkeypatch.setattr(build, "build_id", lambda: "0000000000000000")
    with pytest.raises(AccelError, match="stale"):
        _lib._check_build(handle)
