"""ORACLE TEST INFRASTRUCTURE — counter-based RNG shared with the executor.

splitmix64 / mix_seed restate the reference's proj/src/util.hpp:9-23 (the
reference derives independent seeds the same way).  init_normal and tokens
restate csrc/kernels.h (Irwin-Hall(4) N(0, 0.02) weights; uniform tokens),
vectorised over uint64 numpy arrays (wrapping arithmetic), bit-exact with the
device generators.
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = np.uint64(0x9E3779B97F4A7C15)
C1 = np.uint64(0xBF58476D1CE4E5B9)
C2 = np.uint64(0x94D049BB133111EB)
TOKEN_TAG = 0x746F6B656E73
INIT_SCALE = np.float32(float.fromhex("0x1.1bc77ap-21"))


def splitmix64(x):
    """util.hpp:10-15, on uint64 arrays."""
    with np.errstate(over="ignore"):
        x = np.asarray(x, dtype=np.uint64) + GOLDEN
        x = (x ^ (x >> np.uint64(30))) * C1
        x = (x ^ (x >> np.uint64(27))) * C2
        return x ^ (x >> np.uint64(31))


def splitmix64_int(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def mix_seed(seed: int, a: int, b: int = 0, c: int = 0) -> int:
    """util.hpp:17-23."""
    h = splitmix64_int((seed ^ 0x8E12FCA87B5D03E1) & M64)
    h = splitmix64_int(h ^ (a & M64))
    h = splitmix64_int(h ^ (b & M64))
    h = splitmix64_int(h ^ (c & M64))
    return h


def init_normal(tensor_seed: int, offset: int, n: int) -> np.ndarray:
    """Element idx of a tensor: (sum of the four 16-bit lanes of
    splitmix64(seed + idx) - 131070) * 0x1.1bc77ap-21 (std 0.02), fp32."""
    idx = np.arange(offset, offset + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = splitmix64(idx + np.uint64(tensor_seed & M64))
    m = np.uint64(0xFFFF)
    s = ((h & m).astype(np.int64) + ((h >> np.uint64(16)) & m).astype(np.int64)
         + ((h >> np.uint64(32)) & m).astype(np.int64) + ((h >> np.uint64(48)) & m).astype(np.int64)
         - 131070)
    return s.astype(np.float32) * INIT_SCALE


def tokens(seed: int, step: int, sample0: int, n_samples: int, S: int, vocab: int) -> np.ndarray:
    """[n_samples, S+1] int32: splitmix64(mix_seed(seed, TAG, step, sample) + pos) % vocab."""
    out = np.empty((n_samples, S + 1), np.int32)
    pos = np.arange(S + 1, dtype=np.uint64)
    for i in range(n_samples):
        base = np.uint64(mix_seed(seed, TOKEN_TAG, step, sample0 + i))
        with np.errstate(over="ignore"):
            out[i] = (splitmix64(pos + base) % np.uint64(vocab)).astype(np.int32)
    return out
