"""Stream identity for the counter-based generator.

The reference keys SplitMix64 streams by (seed, stream) (rng.py:61-109).
On the device every draw is Philox4x32-10 keyed by the 64-bit seed with
counter (pixel, sample, segment, call) (csrc/mf_transport.cuh), so results
depend only on those keys -- never on scheduling, tile size, pass size or
GPU count.  RandomStream keeps the reference's (seed, stream) identity for
API compatibility (transmittance_estimate, trace_path)."""

from __future__ import annotations

from dataclasses import dataclass


@dataclass
class RandomStream:
    seed: int
    stream: int = 0
    counter: int = 0

    def derive(self, index):
        """Child stream keyed by index (rng.py:100-109, different hash)."""
        child = (self.stream * 0x9E3779B97F4A7C15 ^ (index * 0xBF58476D1CE4E5B9 + 1)) & (2**64 - 1)
        return RandomStream(self.seed, child)
