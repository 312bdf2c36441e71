"""Counter-based synthetic inputs, bit-identical on host and device.

``rand(seed, i) = mix64(i * 0x9E3779B97F4A7C15 + mix64(seed ^ 0x5851F42D4C957F2D))``
(== ``ixo_rand`` in oracle/ixoracle.c and ``ixg_gen_uniform`` on the device),
so a 2^28-element input can be generated on the GPU (no PCIe) and any slice
of it regenerated on the host to check results.
"""

from __future__ import annotations

import numpy as np

from .pred import mix64

_G = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def _mix_np(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _C1
    z = (z ^ (z >> np.uint64(27))) * _C2
    return z ^ (z >> np.uint64(31))


def seed_mix(seed: int) -> int:
    return mix64((seed ^ 0x5851F42D4C957F2D) & ((1 << 64) - 1))


def rand_u64(seed: int, n: int, offset: int = 0) -> np.ndarray:
    i = np.arange(offset, offset + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix_np(i * _G + np.uint64(seed_mix(seed)))


def uniform(seed: int, n: int, lo: int, hi: int, dtype=np.int64, offset: int = 0) -> np.ndarray:
    """lo + rand(seed, offset+i) mod (hi - lo + 1), like ixg_gen_uniform."""
    u = rand_u64(seed, n, offset)
    span = (hi - lo + 1) & ((1 << 64) - 1)
    with np.errstate(over="ignore"):
        if span == 0:
            v = u
        else:
            v = np.uint64(lo & ((1 << 64) - 1)) + u % np.uint64(span)
    return v.view(np.int64).astype(dtype)


def segment_shape(seed: int, m: int, k: int, empty_every: int = 97) -> np.ndarray:
    """m segment lengths summing to exactly k (BASELINE C2):
    uniform weights in [0, 2k/m] rescaled to sum k, with every
    ``empty_every``-th segment forced empty (>= 1 % empty segments)."""
    if m == 0:
        return np.zeros(0, dtype=np.int64)
    avg = max(1, (2 * k) // max(m, 1))
    w = uniform(seed, m, 0, avg, np.int64).astype(np.float64)
    if empty_every and m > 1:
        w[: m - 1 : empty_every] = 0.0  # never the last one: it absorbs rounding
    w[m - 1] = max(w[m - 1], 1.0)
    cum = np.floor(np.cumsum(w) * (k / w.sum())).astype(np.int64)
    cum[-1] = k
    cum = np.maximum.accumulate(np.minimum(cum, k))
    shape = np.diff(np.concatenate([[0], cum]))
    assert shape.sum() == k and (shape >= 0).all()
    return shape
