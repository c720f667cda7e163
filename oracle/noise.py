"""Counter-based sampling noise, restated on the CPU for the checker.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product path.

The GPU kernels (paper_1611_09482_b200/csrc/noise.cuh) and this module
compute the same 32-bit integer hash, so noise is bit-identical on both
sides; only the final float transform (log) can differ in the last ulp, which
the parity tests treat as a logged near-tie ("Sampling
parity"). BASELINE's "shared seeded Gumbel/uniform noise table" for cfg4
would be 100 GB if materialised, so the table is this pure function of
(seed, global stream id, step, class) instead.
"""

from __future__ import annotations

import numpy as np

_M1 = np.uint32(0x7FEB352D)
_M2 = np.uint32(0x846CA68B)
SEED_SALT = 0x243F6A88
UNIFORM_CLASS = 0xFFFFFFFF  # class slot used for the per-step inverse-CDF uniform


def mix32(x: np.ndarray) -> np.ndarray:
    """lowbias32 integer finaliser on uint32 arrays (wrapping multiply)."""
    x = np.asarray(x, dtype=np.uint32).copy()
    with np.errstate(over="ignore"):
        x ^= x >> np.uint32(16)
        x *= _M1
        x ^= x >> np.uint32(15)
        x *= _M2
        x ^= x >> np.uint32(16)
    return x


def hash_bits(seed: int, stream, step, cls) -> np.ndarray:
    """32-bit hash of (seed, stream, step, class); arguments broadcast."""
    h = mix32(np.uint32((seed ^ SEED_SALT) & 0xFFFFFFFF))
    h = mix32(h ^ np.asarray(stream, dtype=np.uint32))
    h = mix32(h ^ np.asarray(step, dtype=np.uint32))
    return mix32(h ^ np.asarray(cls, dtype=np.uint32))


def uniform(seed: int, stream, step, cls) -> np.ndarray:
    """u in (0, 1): ((h >> 8) + 0.5) * 2**-24, exactly representable in float32."""
    h = hash_bits(seed, stream, step, cls)
    return ((h >> np.uint32(8)).astype(np.float64) + 0.5) * 2.0**-24


def gumbel(seed: int, streams: np.ndarray, step: int, classes: int) -> np.ndarray:
    """Gumbel noise g = -log(-log u), shape (len(streams), classes), float64."""
    s = np.asarray(streams, dtype=np.uint32)[:, None]
    c = np.arange(classes, dtype=np.uint32)[None, :]
    u = uniform(seed, s, np.uint32(step), c)
    return -np.log(-np.log(u))


def step_uniform(seed: int, streams: np.ndarray, step: int) -> np.ndarray:
    """The per-(stream, step) uniform of inverse-CDF sampling, shape (len(streams),)."""
    return uniform(seed, np.asarray(streams, dtype=np.uint32), np.uint32(step),
                   np.uint32(UNIFORM_CLASS))
