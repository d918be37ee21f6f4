"""Seeded synthetic INPUT generators shared by tests, bench.py and smoke().

Holds none of the method's arithmetic (no covariance, no factorization, no
likelihood): only random numbers and site patterns that are handed, as inputs,
to both the CUDA path and the oracle (task rule: random numbers the method
draws are passed in as inputs). Recipes are stated in DESIGN.md "Inputs".

  normals(n, seed)        e ~ N(0,1) by Box-Muller on a SplitMix64 stream
                          (Alg. 1 l.6, "Normal random generation of a vector e",
                          P:645; DESIGN R4).
  collinear_sites(n, h)   x_i = i*h, y_i = 0 (exact binary distances) for the
                          AR(1)/Kac-Murdock-Szego closed-form pin.
  spread_sites(n, gap)    sites `gap` apart on a line (Sigma = theta1*I exactly
                          once exp underflows).
"""
from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
STREAM_NORMALS = 0x4E4F524D414C5345  # "NORMALSE"
STREAM_HOLDOUT = 0x484F4C444F555431  # "HOLDOUT1"


def _mix(v: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser on a uint64 array (wrap-around arithmetic)."""
    with np.errstate(over="ignore"):
        v = v + np.uint64(0x9E3779B97F4A7C15)
        v = (v ^ (v >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        v = (v ^ (v >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return v ^ (v >> np.uint64(31))


def draws(seed: int, stream: int, count: int, start: int = 0) -> np.ndarray:
    """draw(seed, stream, i) = mix(mix(seed ^ stream) + i), i in [start, start+count)."""
    base = _mix(np.array([(seed ^ stream) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0]
    i = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix(base + i)


def normals(n: int, seed: int) -> np.ndarray:
    """n standard normal variates (Box-Muller on pairs of 53-bit uniforms)."""
    m = (n + 1) // 2
    b = draws(seed, STREAM_NORMALS, 2 * m)
    u1 = ((b[0::2] >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0**-53  # (0, 1]
    u2 = (b[1::2] >> np.uint64(11)).astype(np.float64) * 2.0**-53          # [0, 1)
    r = np.sqrt(-2.0 * np.log(u1))
    e = np.empty(2 * m, np.float64)
    e[0::2] = r * np.cos(2.0 * np.pi * u2)
    e[1::2] = r * np.sin(2.0 * np.pi * u2)
    return e[:n].copy()


def holdout_mask(n: int, m: int, seed: int) -> np.ndarray:
    """Boolean mask selecting the m sites with the smallest hold-out keys."""
    k = draws(seed, STREAM_HOLDOUT, n)
    idx = np.argsort(k, kind="stable")[:m]
    mask = np.zeros(n, bool)
    mask[idx] = True
    return mask


def collinear_sites(n: int, h: float = 2.0**-12):
    x = np.arange(n, dtype=np.float64) * h
    return x, np.zeros(n, np.float64)


def spread_sites(n: int, gap: float):
    x = np.arange(n, dtype=np.float64) * gap
    return x, np.zeros(n, np.float64)
