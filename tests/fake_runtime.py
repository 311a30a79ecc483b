"""A minimal stand-in for the reference runtime's effects (runtime.py: Get,
Sleep, CLOSED, TIMEOUT, Channel) and ReplayBuffer.sample, so the Trainer.run
generator can be driven on the GPU box, where the reference is absent."""

from __future__ import annotations

CLOSED = object()
TIMEOUT = object()


class Get:
    def __init__(self, chan, timeout=None):
        self.chan, self.timeout = chan, timeout


class Sleep:
    def __init__(self, dt):
        self.dt = dt


class Channel:
    def __init__(self, items):
        self.items = list(items)


class StopFlag:
    is_set = False


class ReplayBuffer:
    """sample(n, rng): n uniform picks with replacement, None below n items
    (buffers.py:74-86)."""

    def __init__(self, items):
        self.items = list(items)

    def sample(self, n, rng):
        if n == 0:
            return []
        if len(self.items) < n:
            return None
        return [self.items[i] for i in rng.integers(0, len(self.items), size=n)]


def drive(gen):
    """Run a Trainer.run generator to completion."""
    try:
        eff = next(gen)
        while True:
            if isinstance(eff, Get):
                out = eff.chan.items.pop(0) if eff.chan.items else CLOSED
            else:
                out = None
            eff = gen.send(out)
    except StopIteration:
        pass
