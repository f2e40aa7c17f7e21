"""Counter-based random streams.

Device paths never use this: every draw on the GPU is Philox4x32-10 keyed
by the 64-bit seed with counter (pixel, sample, segment, call)
(csrc/mf_transport.cuh), so results depend only on those keys -- never on
scheduling, tile size, pass size or GPU count.  RandomStream keeps the
reference's host-side stream API (rng.py:61-109: SplitMix64 over a Weyl
sequence keyed by (seed, stream)) for callers that draw uniforms on the
host, e.g. phase_sample(wo, medium, frame, rng)."""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

_U = np.uint64
_PHI = _U(0x9E3779B97F4A7C15)
_M1 = _U(0xBF58476D1CE4E5B9)
_M2 = _U(0x94D049BB133111EB)


def _mix(z):
    z = (z ^ (z >> _U(30))) * _M1
    z = (z ^ (z >> _U(27))) * _M2
    return z ^ (z >> _U(31))


@dataclass
class RandomStream:
    seed: int
    stream: int = 0
    counter: int = 0
    _base: np.uint64 = field(init=False, repr=False)

    def __post_init__(self):
        with np.errstate(over="ignore"):
            s = np.asarray(self.seed, dtype=np.uint64)
            k = np.asarray(self.stream, dtype=np.uint64)
            self._base = _mix(_mix(s * _PHI + _U(1)) ^ (k * _M2 + _U(1)))

    def uniform(self, shape=None):
        n = 1 if shape is None else int(np.prod(shape))
        ctr = np.arange(self.counter, self.counter + n, dtype=np.uint64)
        self.counter += n
        with np.errstate(over="ignore"):
            raw = _mix(self._base + ctr * _PHI)
        u = (raw >> _U(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
        return float(u[0]) if shape is None else u.reshape(shape)

    def derive(self, index):
        with np.errstate(over="ignore"):
            child = int(_mix(np.asarray(self.stream, dtype=np.uint64) * _PHI
                             ^ np.asarray(index, dtype=np.uint64) * _M1 + _U(1)))
        return RandomStream(self.seed, child)


def draw_uniforms(rng, shape):
    """Uniforms in [0, 1) from a RandomStream or a numpy Generator."""
    if isinstance(rng, np.random.Generator):
        return rng.random(shape)
    return np.asarray(rng.uniform(shape), dtype=np.float64)
