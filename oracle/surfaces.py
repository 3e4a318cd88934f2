"""Closest point functions cp_S (Eq. (3)) — oracle.

cp_S(x) = argmin_{y in S} ||x - y||_2.  Each surface returns (cp, dist) for an
(n, 3) float64 array of points, dist = ||x - cp(x)||.

Floating-point order is spelled out (sums left to right, products before
division) because the band membership test `dist <= lambda` and the stencil
base `floor(cp/h)` are integer decisions taken from these numbers; DESIGN.md
reading R3 fixes the same order for the CUDA path.
"""
from __future__ import annotations

import numpy as np


class Sphere:
    """Sphere of radius R centred at the origin; cp(x) = R x/|x|."""

    kind = "sphere"

    def __init__(self, R: float = 1.0):
        self.R = float(R)

    def cp(self, x: np.ndarray):
        x = np.asarray(x, dtype=np.float64)
        r = np.sqrt(x[:, 0] * x[:, 0] + x[:, 1] * x[:, 1] + x[:, 2] * x[:, 2])
        with np.errstate(divide="ignore", invalid="ignore"):
            cp = (self.R * x) / r[:, None]
        dist = np.abs(r - self.R)
        bad = r == 0.0  # centre: cp undefined (medial axis)
        cp[bad] = np.nan
        dist[bad] = np.inf
        return cp, dist

    def bbox(self, pad: float):
        """Axis-aligned box containing every point within `pad` of the surface."""
        e = self.R + pad
        return np.array([-e, -e, -e]), np.array([e, e, e])


class Torus:
    """Torus about the z axis: major radius R, minor radius r (BASELINE configs 2, 4).

    With rho = |(x, y)|, the nearest point of the core circle is
    q = (R x/rho, R y/rho, 0); cp = q + r (x - q)/|x - q|, dist = | |x-q| - r |.
    """

    kind = "torus"

    def __init__(self, R: float = 1.0, r: float = 0.4):
        self.R = float(R)
        self.r = float(r)

    def cp(self, x: np.ndarray):
        x = np.asarray(x, dtype=np.float64)
        rho = np.sqrt(x[:, 0] * x[:, 0] + x[:, 1] * x[:, 1])
        with np.errstate(divide="ignore", invalid="ignore"):
            qx = (self.R * x[:, 0]) / rho
            qy = (self.R * x[:, 1]) / rho
            dx = x[:, 0] - qx
            dy = x[:, 1] - qy
            dz = x[:, 2]
            dn = np.sqrt(dx * dx + dy * dy + dz * dz)
            cp = np.empty_like(x)
            cp[:, 0] = qx + (self.r * dx) / dn
            cp[:, 1] = qy + (self.r * dy) / dn
            cp[:, 2] = (self.r * dz) / dn
        dist = np.abs(dn - self.r)
        bad = (rho == 0.0) | (dn == 0.0)  # axis / core circle: cp undefined
        cp[bad] = np.nan
        dist[bad] = np.inf
        return cp, dist

    def bbox(self, pad: float):
        e = self.R + self.r + pad
        ez = self.r + pad
        return np.array([-e, -e, -ez]), np.array([e, e, ez])


class Plane:
    """Plane z = z0 (test surface only: reduces CPM to the 2-D 5-point Laplacian)."""

    kind = "plane"

    def __init__(self, z0: float = 0.0):
        self.z0 = float(z0)

    def cp(self, x: np.ndarray):
        x = np.asarray(x, dtype=np.float64)
        cp = x.copy()
        cp[:, 2] = self.z0
        return cp, np.abs(x[:, 2] - self.z0)

    def bbox(self, pad: float):
        big = 1e300
        return np.array([-big, -big, self.z0 - pad]), np.array([big, big, self.z0 + pad])


def make_surface(kind: str, **kw):
    if kind == "sphere":
        return Sphere(kw.get("R", 1.0))
    if kind == "torus":
        return Torus(kw.get("R", 1.0), kw.get("r", 0.4))
    if kind == "plane":
        return Plane(kw.get("z0", 0.0))
    raise ValueError(f"unknown surface {kind!r}")
