"""splitmix64 counter-based streams (pkg/src/picmc/rng.py:56-116).

Host restatement used by plasma loading; the device twin lives in
csrc/init.cu.  A draw is a pure function of (key, counter), so the
population a GPU shard loads is independent of how cells are sharded.
"""

import numpy as np

STREAM_INIT = 1      # rng.py:37 purpose tags
STREAM_COLLIDE = 2
STREAM_BENCH = 3

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
_C1 = 0xBF58476D1CE4E5B9
_C2 = 0x94D049BB133111EB
INV53 = 2.0 ** -53


def mix64(z: int) -> int:
    """splitmix64 finalizer (scalar)."""
    z &= M64
    z = ((z ^ (z >> 30)) * _C1) & M64
    z = ((z ^ (z >> 27)) * _C2) & M64
    return z ^ (z >> 31)


def mix64_vec(z) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_C1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_C2)
        return z ^ (z >> np.uint64(31))


def derive(key: int, n: int) -> int:
    return mix64((key + (n + 1) * GOLDEN) & M64)


def derive_vec(key, n) -> np.ndarray:
    key = np.asarray(key, dtype=np.uint64)
    n = np.asarray(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64_vec(key + (n + np.uint64(1)) * np.uint64(GOLDEN))


def stream(seed: int, *path: int) -> int:
    key = mix64(seed & M64)
    for p in path:
        key = derive(key, p)
    return key


def uniforms(key, counters) -> np.ndarray:
    return (derive_vec(key, counters) >> np.uint64(11)).astype(np.float64) * INV53


def uniforms_open(key, counters) -> np.ndarray:
    bits = derive_vec(key, counters) >> np.uint64(11)
    return (bits.astype(np.float64) + 0.5) * INV53
