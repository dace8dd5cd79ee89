"""Counter-based SplitMix64 streams (numpy, vectorised).

A stream is a 64-bit key; draw i of the stream is ``mix64(key + (i+1)*GOLDEN)``
(mod 2^64).  Streams are keyed by (config seed, layer index, purpose tag), so
every purpose draws from its own independent sequence and the result of a
recipe does not depend on chunk sizes or on the order purposes are drawn.
"""
import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_MASK = (1 << 64) - 1


def mix64(z):
    """SplitMix64 finaliser on a uint64 numpy array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def _mix_int(x: int) -> int:
    return int(mix64(np.array([x & _MASK], dtype=np.uint64))[0])


# purpose tags (any distinct constants)
TAGS = {
    "base": 1, "keep": 2, "unique": 3, "perm": 4, "graph": 5, "sample": 6,
}


def stream_key(seed: int, layer: int, tag: str) -> int:
    t = TAGS[tag]
    k = _mix_int(seed * 0x632BE59BD9B4E019 + 0x1234567)
    k = _mix_int(k ^ ((layer + 1) * 0xD1B54A32D192ED03))
    k = _mix_int(k ^ (t * 0x8CB92BA72F3D8DD7))
    return k


class Stream:
    """Counter-based generator: ``next_u64(n)`` returns the next n draws."""

    def __init__(self, key: int):
        self.key = np.uint64(key & _MASK)
        self.ctr = 0

    def next_u64(self, n: int) -> np.ndarray:
        i = np.arange(self.ctr + 1, self.ctr + 1 + n, dtype=np.uint64)
        self.ctr += n
        with np.errstate(over="ignore"):
            return mix64(self.key + i * GOLDEN)

    def next_uniform(self, n: int) -> np.ndarray:
        """Uniform doubles in [0,1): (x >> 11) * 2^-53."""
        x = self.next_u64(n)
        return (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)

    def next_below(self, n: int, bound: int) -> np.ndarray:
        """Integers in [0, bound) as ((x >> 32) * bound) >> 32 (bound < 2^32)."""
        assert 0 < bound < (1 << 32)
        x = self.next_u64(n) >> np.uint64(32)
        with np.errstate(over="ignore"):
            return ((x * np.uint64(bound)) >> np.uint64(32)).astype(np.int64)
