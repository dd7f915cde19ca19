"""Seeded synthetic inputs shared by the oracle tests, the GPU tests, smoke() and bench.py.

This module holds NONE of the method's arithmetic (no distances, no schedules, no
passes, no clamping).  It only draws the random numbers the method consumes, so that
the CPU oracle and the CUDA path are fed byte-identical host arrays:

* seed positions: i.i.d. uniform over the N x N pixel grid ("uniform
  distribution for the seeds", "seeds are randomly distributed with a
  uniform distribution");
* displacements: per axis, a uniform integer in [-d, d] ("seeds move up to
  d_max discrete units in any direction, randomly chosen with a uniform distribution";
  DESIGN.md reading R-10).  Clamping to the grid is the method's job, not this module's.

Generator: SplitMix64 as a counter-based hash of (rng_seed, stream, index), then the
multiply-shift map of the high 32 bits onto [0, n) (bias < n / 2**32, i.e. < 2**-16 for
n <= 65536).  Stream 0 draws seeds, stream 1 + f draws the displacements of frame f.
Everything is vectorised numpy on uint64 with wrap-around arithmetic.
"""
from __future__ import annotations

import numpy as np

__all__ = ["splitmix64", "uniform_below", "uniform_seeds", "displacements", "RNG_SEED"]

RNG_SEED = 2209  # default key: the paper's arXiv number prefix

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_STREAM_MUL = np.uint64(0xD1B54A32D192ED03)


def splitmix64(z: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser applied elementwise to uint64 counters (wrapping)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def _stream_key(rng_seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        k = np.uint64(rng_seed & 0xFFFFFFFFFFFFFFFF) ^ (np.uint64(stream + 1) * _STREAM_MUL)
    return splitmix64(np.array([k], dtype=np.uint64))[0]


def uniform_below(n: int, rng_seed: int, stream: int, count: int) -> np.ndarray:
    """`count` draws in [0, n) for counters 0..count-1 of (rng_seed, stream). uint64 out."""
    if n <= 0:
        raise ValueError("n must be positive")
    key = _stream_key(rng_seed, stream)
    with np.errstate(over="ignore"):
        ctr = np.arange(count, dtype=np.uint64) + key
    u = splitmix64(ctr) >> np.uint64(32)  # high 32 bits
    return (u * np.uint64(n)) >> np.uint64(32)


def uniform_seeds(N: int, s: int, rng_seed: int = RNG_SEED) -> np.ndarray:
    """s seed positions, uniform over [0,N)^2, as a flat uint16 array x0,y0,x1,y1,...

    At N = 65536 the pixel (65535, 65535) is reserved as the EMPTY sentinel (DESIGN.md
    reading R-4); a draw that lands there is replaced by (65534, 65535).  This is a
    property of the label encoding, not of the method, and it is the only adjustment.
    """
    if not (2 <= N <= 65536):
        raise ValueError("N must be in [2, 65536]")
    if not (1 <= s <= N * N):
        raise ValueError("need 1 <= s <= N*N")
    d = uniform_below(N, rng_seed, 0, 2 * s)
    xy = d.astype(np.uint16)
    if N == 65536:
        x = xy[0::2]
        y = xy[1::2]
        bad = (x == 65535) & (y == 65535)
        x[bad] = 65534
    return xy


def displacements(s: int, d: int, frame: int, rng_seed: int = RNG_SEED) -> np.ndarray:
    """Frame `frame`'s per-seed displacement, per axis uniform in [-d, d].

    Flat int16 array dx0,dy0,dx1,dy1,...  (d <= 32767).
    """
    if not (0 <= d <= 32767):
        raise ValueError("d must be in [0, 32767]")
    u = uniform_below(2 * d + 1, rng_seed, 1 + frame, 2 * s).astype(np.int64) - d
    return u.astype(np.int16)
