"""SplitMix64, scalar and counter-vectorised.

The reference seeds every generator with SplitMix64
(/root/reference/pkg/src/tiered_spgemm/rng.py:17-58).  SplitMix64 is a
counter generator in disguise: the k-th output (k >= 1) of a stream seeded
with s is ``mix(s + k * GAMMA)``.  ``stream`` evaluates any window of that
sequence with numpy uint64 arithmetic, so the R-MAT builder can draw its
billions of variates in bulk and still equal, value for value, what a
``PortableRng(seed)`` consumer would have drawn in order.
"""

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_MASK = (1 << 64) - 1


def _mix_scalar(z: int) -> int:
    z = ((z ^ (z >> 30)) * _M1) & _MASK
    z = ((z ^ (z >> 27)) * _M2) & _MASK
    return z ^ (z >> 31)


class PortableRng:
    """Sequential SplitMix64 with the reference's helper draws."""

    def __init__(self, seed: int):
        self._state = int(seed) & _MASK

    def next_u64(self) -> int:
        self._state = (self._state + GAMMA) & _MASK
        return _mix_scalar(self._state)

    def below(self, n: int) -> int:
        if n <= 0:
            raise ValueError("bound must be positive")
        reject_at = (1 << 64) - ((1 << 64) % n)
        while True:
            v = self.next_u64()
            if v < reject_at:
                return v % n

    def uniform_open_closed(self) -> float:
        return ((self.next_u64() >> 11) + 1) * (2.0 ** -53)

    def sample_without_replacement(self, n: int, k: int) -> list:
        if k > n:
            raise ValueError("cannot draw %d distinct values from %d" % (k, n))
        moved = {}
        picks = []
        for j in range(k):
            r = j + self.below(n - j)
            picks.append(moved.get(r, r))
            moved[r] = moved.get(j, j)
        return picks


def stream(seed: int, start: int, count: int) -> np.ndarray:
    """Outputs start+1 .. start+count of PortableRng(seed) as uint64."""
    k = np.arange(start + 1, start + 1 + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(int(seed) & _MASK) + k * np.uint64(GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
        z = z ^ (z >> np.uint64(31))
    return z


def unit_interval(u64: np.ndarray) -> np.ndarray:
    """uint64 draws to doubles in [0, 1) with 53 bits."""
    return (u64 >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
