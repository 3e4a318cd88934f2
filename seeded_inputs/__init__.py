"""Seeded synthetic input generators shared by the oracle and the CUDA path.

This module is the ONLY code both sides may share (task rule ③). It holds no
arithmetic of the closest point method: no closest points, no interpolation,
no operators, no surfaces.  It only turns (seed, lattice coordinate) into
pseudo-random numbers with a counter-based generator, so that either side can
draw the value belonging to any grid node without knowing the other side's
node ordering.

Generator: SplitMix64 (Steele, Lea, Flood 2014) chained over the key
(seed, stream, i, j, k), with i, j, k taken as two's-complement 64-bit words.
uniform01 = (z >> 11) * 2**-53, i.e. 53 random mantissa bits in [0, 1).
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _splitmix64(z: np.ndarray) -> np.ndarray:
    z = z + _GOLDEN
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def _key(seed: int, stream: int, ijk: np.ndarray) -> np.ndarray:
    ijk = np.asarray(ijk, dtype=np.int64)
    if ijk.ndim != 2 or ijk.shape[1] != 3:
        raise ValueError("ijk must have shape (n, 3)")
    with np.errstate(over="ignore"):
        z = _splitmix64(np.full(ijk.shape[0], np.uint64(seed & 0xFFFFFFFFFFFFFFFF)))
        z = _splitmix64(z ^ np.uint64(stream & 0xFFFFFFFFFFFFFFFF))
        for c in range(3):
            z = _splitmix64(z ^ ijk[:, c].view(np.uint64))
    return z


def uniform01(seed: int, ijk: np.ndarray, stream: int = 0) -> np.ndarray:
    """U[0,1) per lattice node (n,3) int array -> (n,) float64."""
    z = _key(seed, stream, ijk)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform_pm1(seed: int, ijk: np.ndarray, stream: int = 0) -> np.ndarray:
    """U[-1,1) per lattice node (config 1: 'u drawn uniform[-1,1] (seed 0)')."""
    return 2.0 * uniform01(seed, ijk, stream) - 1.0


def normal(seed: int, ijk: np.ndarray, stream: int = 0) -> np.ndarray:
    """N(0,1) per lattice node by Box-Muller on two independent streams."""
    u1 = uniform01(seed, ijk, 2 * stream + 1)
    u2 = uniform01(seed, ijk, 2 * stream + 2)
    u1 = np.where(u1 <= 0.0, 2.0 ** -53, u1)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def smooth_modulation_coeffs(seed: int, n: int = 8) -> np.ndarray:
    """Coefficients of the 'random smooth modulation from seed 1' (config 2).

    Returns an (n, 4) array of (a, kx, ky, kz) used as
    m(x) = 1 + sum_q a_q * sin(kx_q x + ky_q y + kz_q z) evaluated on the
    closest point by each side itself.  Amplitudes sum to at most 0.5.
    """
    rng = np.random.Generator(np.random.Philox(seed))
    a = rng.uniform(-1.0, 1.0, n)
    a *= 0.5 / np.sum(np.abs(a))
    k = rng.integers(-3, 4, size=(n, 3)).astype(np.float64)
    return np.concatenate([a[:, None], k], axis=1)


__all__ = ["uniform01", "uniform_pm1", "normal", "smooth_modulation_coeffs"]
