"""Counter-based PRF for deterministic table initialisation (TEST INFRASTRUCTURE).

SPEC S:48-51 ("keyed deterministic pseudo-random function") and S:252-260
(init_row: values[j] = prf_uniform(seed, "emb", (key, j), -1/sqrt(d), +1/sqrt(d))).
The concrete function is the reading SURVEY §8(c) Q15 proposes (DESIGN.md
reading R-PRF):

    h1 = splitmix64(seed + GOLDEN * (key + 1))          (mod 2^64)
    h  = splitmix64(h1 xor (j * MIX_J))
    uniform: u = (h >> 40) * 2^-24;  v = fp32(lo + scale*u)  with
             lo = fp32(-1/sqrt(d)), scale = fp32(2/sqrt(d))  (one rounding,
             i.e. the value a fused multiply-add produces)
    dyadic : v = ((h >> 60) - 8) * 2^-8                (parity regime P1)

Both the CUDA library and this module implement it independently.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
MIX_J = np.uint64(0xD1B54A32D192ED03)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def prf_words(seed: int, keys: np.ndarray, d: int) -> np.ndarray:
    """64-bit PRF words h[key, j] for j in [0, d)."""
    keys = np.asarray(keys, dtype=np.int64).astype(np.uint64)
    with np.errstate(over="ignore"):
        h1 = splitmix64(np.uint64(seed) + GOLDEN * (keys + np.uint64(1)))
        j = np.arange(d, dtype=np.uint64) * MIX_J
        return splitmix64(h1[:, None] ^ j[None, :])


def init_rows(seed: int, keys: np.ndarray, d: int, mode: str = "uniform") -> np.ndarray:
    """init_row of S:252-260 for every key: float32 [len(keys), d]."""
    h = prf_words(seed, keys, d)
    if mode == "uniform":
        lo = np.float32(-1.0 / np.sqrt(d))
        scale = np.float32(2.0 / np.sqrt(d))
        u = (h >> np.uint64(40)).astype(np.float64) * 2.0 ** -24
        # scale*u has <= 48 significant bits and lo's exponent is within a few
        # binades, so the fp64 expression is exact; one rounding to fp32 = fma
        return (np.float64(lo) + np.float64(scale) * u).astype(np.float32)
    if mode == "dyadic":
        r = (h >> np.uint64(60)).astype(np.int64) - 8
        return (r.astype(np.float64) * 2.0 ** -8).astype(np.float32)
    raise ValueError(mode)
