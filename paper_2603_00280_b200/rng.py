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

    def normal(self, shape=None):
        """Box-Muller over two uniforms per pair (rng.py:87-97)."""
        n = 1 if shape is None else int(np.prod(shape))
        m = (n + 1) // 2
        u1 = self.uniform((m,))
        u2 = self.uniform((m,))
        r = np.sqrt(-2.0 * np.log1p(-u1))
        z = np.concatenate([r * np.cos(6.283185307179586 * u2),
                            r * np.sin(6.283185307179586 * u2)])[:n]
        return float(z[0]) if shape is None else z.reshape(shape)

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


class BatchRng:
    """Per-ray counter-based streams of a wavefront (transport.py:52-67):
    `base` (uint64 per ray, e.g. stream_base / derive_bases) and `counter`
    (uint64 per ray).  The device does not consume SplitMix64 draws one by
    one: a call that walks / traces ray i keys ray i's Philox stream by
    philox_keys(base_i, counter_i) and then advances counter_i by one, so
    results depend only on (base, counter) -- never on batching or launch
    geometry -- and successive calls draw independent streams.  Parity with
    the reference's SplitMix64 draws is statistical."""

    def __init__(self, base, counter):
        self.base = np.asarray(base, dtype=np.uint64)
        self.counter = np.array(counter, dtype=np.uint64)

    def draw(self, mask=None):
        """Host-side uniforms, bit-identical to the reference's BatchRng."""
        with np.errstate(over="ignore"):
            raw = _mix(self.base + self.counter * _PHI)
        u = (raw >> _U(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
        self.counter = self.counter + (np.uint64(1) if mask is None
                                       else np.asarray(mask, dtype=np.uint64))
        return u


def stream_base(seed, stream):
    """Base state of stream (seed, stream) (rng.py:24-29)."""
    with np.errstate(over="ignore"):
        s = np.asarray(seed, dtype=np.uint64)
        k = np.asarray(stream, dtype=np.uint64)
        return _mix(_mix(s * _PHI + _U(1)) ^ (k * _M2 + _U(1)))


def derive_bases(seed, stream, indices):
    """Base states of the child streams RandomStream(seed, stream).derive(i)
    (rng.py:48-58)."""
    with np.errstate(over="ignore"):
        child = _mix(np.asarray(stream, dtype=np.uint64) * _PHI
                     ^ np.asarray(indices, dtype=np.uint64) * _M1 + _U(1))
    return stream_base(seed, child)


# Philox key of the device streams of BatchRng rays (any fixed 64-bit value)
BATCH_SEED = 0x6D61_6372_6F66_6163


def philox_keys(base, counter, n):
    """(pixel, sample) uint32 Philox counter words of n rays keyed by
    (base, counter): one SplitMix64 avalanche of both, split in halves."""
    b = np.broadcast_to(np.asarray(base, dtype=np.uint64), (n,))
    c = np.broadcast_to(np.asarray(counter, dtype=np.uint64), (n,))
    with np.errstate(over="ignore"):
        h = _mix(b ^ _mix(c * _PHI + _U(0x632BE59BD9B4E019)))
    lo = (h & _U(0xFFFFFFFF)).astype(np.uint32)
    hi = (h >> _U(32)).astype(np.uint32)
    return lo, hi
