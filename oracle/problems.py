"""Right-hand sides and inputs of BASELINE.json's configs — oracle side.

Each side (oracle, CUDA) evaluates f on its own closest points; only the
seeded random draws come from `seeded_inputs` (rule ③).
  config 0: sphere h=0.1, c=1,  f = (c + 12) Y_3^2(cp(x)),  GMRES(30)
  config 1: sphere h=1/200, c=10, f = (c + 42) Y_6^3(cp(x)), GMRES(50); applies on U[-1,1] seed 0
  config 2: torus R=1 r=0.4 h=1/400, c=1, f = cos(3 th) sin(2 ph) m(cp) (reading R10)
  config 3: sphere h=1/800, c=0.1, f = Y_10^5(cp(x)) + 1e-3 N(0,1) seed 2
"""
from __future__ import annotations

import numpy as np

import seeded_inputs

from .band import Band, lattice_points
from .sph import real_sph


def cp_of(band: Band, ijk: np.ndarray) -> np.ndarray:
    cp, _ = band.surface.cp(lattice_points(ijk, band.h))
    return cp


def rhs_sph(band: Band, c: float, l: int, m: int, ijk=None) -> np.ndarray:
    """f = (c + l(l+1)) Y_l^m(cp(x)) on the active nodes (or the given nodes)."""
    ijk = band.active if ijk is None else ijk
    return (c + l * (l + 1)) * real_sph(l, m, cp_of(band, ijk))


def exact_sph(band: Band, l: int, m: int, ijk=None) -> np.ndarray:
    ijk = band.active if ijk is None else ijk
    return real_sph(l, m, cp_of(band, ijk))


def torus_angles(cp: np.ndarray, R: float):
    """ph = toroidal angle atan2(y, x); th = poloidal angle atan2(z, rho - R)."""
    ph = np.arctan2(cp[:, 1], cp[:, 0])
    rho = np.sqrt(cp[:, 0] ** 2 + cp[:, 1] ** 2)
    th = np.arctan2(cp[:, 2], rho - R)
    return th, ph


def rhs_torus(band: Band, seed: int = 1, ijk=None) -> np.ndarray:
    """f = cos(3 th) sin(2 ph) (1 + sum_q a_q sin(k_q . cp))  (config 2, reading R10)."""
    ijk = band.active if ijk is None else ijk
    cp = cp_of(band, ijk)
    th, ph = torus_angles(cp, band.surface.R)
    co = seeded_inputs.smooth_modulation_coeffs(seed)
    mod = np.ones(cp.shape[0])
    for a, kx, ky, kz in co:
        mod = mod + a * np.sin(kx * cp[:, 0] + ky * cp[:, 1] + kz * cp[:, 2])
    return np.cos(3.0 * th) * np.sin(2.0 * ph) * mod


def rhs_noisy_sph(band: Band, l: int = 10, m: int = 5, seed: int = 2, ijk=None) -> np.ndarray:
    """f = Y_l^m(cp(x)) + 1e-3 N(0,1)  (config 3)."""
    ijk = band.active if ijk is None else ijk
    return real_sph(l, m, cp_of(band, ijk)) + 1e-3 * seeded_inputs.normal(seed, ijk)
