"""Schnakenberg reaction-diffusion on a surface by IMEX Euler — oracle (BASELINE config 4).

TEST INFRASTRUCTURE (see oracle/__init__.py): plain CPU fp64, shares no code with
the CUDA path.

BASELINE.json configs[4]:
    u_t = mu1 Delta_S u + gamma (a - u + u^2 v)
    v_t = mu2 Delta_S v + gamma (b - u^2 v)
"IMEX Euler dt=1e-3 ... (two shifted solves (1/(dt mu_i) - Delta_S) u = rhs per step)".
The paper's time-dependent examples treat "the diffusion terms implicitly" and
advance "the nonlinear coupling terms ... explicitly"; the
first-order member of that IMEX family is, with Delta_S^h of Eq. 4:

    (u1 - u0)/dt = mu1 Delta_S^h u1 + gamma (a - u0 + u0^2 v0)
    (v1 - v0)/dt = mu2 Delta_S^h v1 + gamma (b - u0^2 v0)

i.e. (c_i I - Delta_S^h) w1 = c_i (w0 + dt R_w(u0, v0)),  c_i = 1/(dt mu_i):
the shifted Poisson problem of Eq. 2 with shift c_i (reading R14 in DESIGN.md).
Both reaction terms use the OLD state (u0, v0).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse.linalg as spla

from .band import Band
from .operator import laplace_beltrami_matrix


@dataclass(frozen=True)
class SchnakenbergParams:
    a: float = 0.1
    b: float = 0.9
    gamma: float = 10.0
    mu1: float = 1e-3
    mu2: float = 1e-2      # mu2 / mu1 = 10 (BASELINE)
    dt: float = 1e-3


def reaction(u: np.ndarray, v: np.ndarray, p: SchnakenbergParams):
    """(R_u, R_v) = gamma (a - u + u^2 v, b - u^2 v)  (BASELINE configs[4])."""
    u2v = u * u * v
    return p.gamma * (p.a - u + u2v), p.gamma * (p.b - u2v)


def imex_rhs(u: np.ndarray, v: np.ndarray, p: SchnakenbergParams):
    """Right-hand sides c_i (w0 + dt R_w) of the two shifted solves."""
    ru, rv = reaction(u, v, p)
    c1, c2 = 1.0 / (p.dt * p.mu1), 1.0 / (p.dt * p.mu2)
    return c1 * (u + p.dt * ru), c2 * (v + p.dt * rv)


def imex_step(band: Band, u: np.ndarray, v: np.ndarray, p: SchnakenbergParams, L=None):
    """One IMEX Euler step by direct sparse solves of (c_i - Delta_S^h) w1 = rhs_i.

    L: Delta_S^h (optional, assembled once by the caller).  Returns (u1, v1)."""
    if L is None:
        L = laplace_beltrami_matrix(band)
    fu, fv = imex_rhs(u, v, p)
    c1, c2 = 1.0 / (p.dt * p.mu1), 1.0 / (p.dt * p.mu2)
    I = np.ones(band.nA)
    import scipy.sparse as sp

    A1 = (sp.diags(c1 * I) - L).tocsc()
    A2 = (sp.diags(c2 * I) - L).tocsc()
    return spla.spsolve(A1, fu), spla.spsolve(A2, fv)


def initial_state(band: Band, p: SchnakenbergParams, seed: int = 3, ijk=None):
    """u = a + b, v = b / (a + b)^2 plus 1e-2 U[-1,1] noise per lattice node (seed 3,
    streams 0 / 1 for u / v; reading R14)."""
    import seeded_inputs

    ijk = band.active if ijk is None else ijk
    us = p.a + p.b
    vs = p.b / (p.a + p.b) ** 2
    return (us + 1e-2 * seeded_inputs.uniform_pm1(seed, ijk, stream=0),
            vs + 1e-2 * seeded_inputs.uniform_pm1(seed, ijk, stream=1))


__all__ = ["SchnakenbergParams", "reaction", "imex_rhs", "imex_step", "initial_state"]
