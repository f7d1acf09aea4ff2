"""numpy restatements used by the tests (test infrastructure only)."""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1


def splitmix64(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def channel_sign(seed: int, c: np.ndarray) -> np.ndarray:
    z = splitmix64(np.uint64(seed ^ 0x5BD1E9955BD1E995) ^ c.astype(np.uint64))
    return np.where(z & np.uint64(1), np.float32(1.0), np.float32(-1.0)).astype(np.float32)


def gen_values(seed, tensor, first, count, d, seq_len, outlier_channels=0, outlier_scale=1.0,
               hh_stride=0, hh_boost=0.0) -> np.ndarray:
    """CPU restatement of csrc/generate.cu (K0); returns float16 values."""
    base = (seed * 0x9E3779B97F4A7C15 + (tensor + 1) * 0xD1B54A32D192ED03) & M64
    i = np.uint64(first) + np.arange(count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = splitmix64(np.uint64(base) + i)
    s = sum(((z >> np.uint64(16 * j)) & np.uint64(0xFFFF)).astype(np.int64) for j in range(4))
    x = (s - 131070).astype(np.float32) * (np.float32(1.0) / np.float32(37836.5))
    c = (i % np.uint64(d)).astype(np.int64)
    if tensor == 0:
        m = c < outlier_channels
        x[m] = x[m] * np.float32(outlier_scale)
        if hh_stride > 0:
            t = (i // np.uint64(d)) % np.uint64(seq_len)
            m = (t % np.uint64(hh_stride)) == 0
            x[m] = x[m] + np.float32(hh_boost) * channel_sign(seed, c[m])
    elif tensor == 2 and hh_stride > 0:
        x = x + np.float32(0.5) * channel_sign(seed, c)
    return x.astype(np.float16)
