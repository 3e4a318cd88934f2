"""Real spherical harmonics Y_l^m on the unit sphere — oracle.

Used for the manufactured solutions of BASELINE.json configs 0, 1, 3
("f = (c + l(l+1)) Y_l^m(cp(x))"), relying on Delta_S Y_l^m = -l(l+1) Y_l^m.

Reading R9: orthonormal real harmonics without the
Condon-Shortley phase,
  Y_l^0  = K_l^0 P_l(cos th)
  Y_l^m  = sqrt2 K_l^m P_l^m(cos th) cos(m ph)      m > 0
  Y_l^-m = sqrt2 K_l^m P_l^m(cos th) sin(m ph)      m > 0
  K_l^m  = sqrt((2l+1)/(4 pi) (l-m)!/(l+m)!),  th = polar angle, ph = azimuth,
with P_l^m(x) = (1-x^2)^{m/2} d^m/dx^m P_l(x) (scipy's lpmv times (-1)^m).
"""
from __future__ import annotations

import math

import numpy as np
from scipy.special import lpmv


def real_sph(l: int, m: int, xyz: np.ndarray) -> np.ndarray:
    """Y_l^m at the directions of the (n,3) points xyz (need not be unit length)."""
    xyz = np.asarray(xyz, dtype=np.float64)
    r = np.linalg.norm(xyz, axis=1)
    ct = np.clip(xyz[:, 2] / r, -1.0, 1.0)
    ph = np.arctan2(xyz[:, 1], xyz[:, 0])
    am = abs(m)
    K = math.sqrt((2 * l + 1) / (4 * math.pi) * math.factorial(l - am) / math.factorial(l + am))
    P = lpmv(am, l, ct) * (-1.0) ** am
    if m == 0:
        return K * P
    if m > 0:
        return math.sqrt(2.0) * K * P * np.cos(am * ph)
    return math.sqrt(2.0) * K * P * np.sin(am * ph)
