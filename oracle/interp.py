"""Extension operator E by tensor-product barycentric Lagrange interpolation — oracle.

PAPER.md:76  "the function value f(cp_S(x_i)) is therefore found by
interpolating f over the points in Sigma_A near cp_S(x_i). We use tensor
product barycentric Lagrange interpolation [Tref:bary] of degree p, and thus
Sigma_A contains the union of all (p+1)^d cubes of grid points needed to
perform this extension. The interpolation weights are independent of the data
being interpolated, and E can be written as a matrix where each row holds the
interpolation weights for a given node in the computational domain
(consisting of Sigma_A and Sigma_G)."

Reading R2: for p = 3 the (p+1)^3 cube of a node x is the 4x4x4
block of lattice nodes with per-axis indices floor(s)-1 .. floor(s)+2,
s = cp(x)/h, i.e. the cube centred on the lattice cell that contains cp(x).
The 1-D weights are the barycentric formula of the second kind (Berrut and
Trefethen 2004, the paper's [Tref:bary]) on the equispaced nodes
tau = (-1, 0, 1, 2) with barycentric weights beta_j = 1/prod_{k!=j}(tau_j - tau_k)
= (-1/6, 1/2, -1/2, 1/6), evaluated at t = s - floor(s) in [0, 1).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .band import Band, lattice_points, _lookup, node_key

TAU = np.array([-1.0, 0.0, 1.0, 2.0])


def barycentric_betas(tau: np.ndarray) -> np.ndarray:
    """beta_j = 1 / prod_{k != j} (tau_j - tau_k)  (barycentric weights, [Tref:bary])."""
    n = len(tau)
    beta = np.empty(n)
    for j in range(n):
        prod = 1.0
        for k in range(n):
            if k != j:
                prod *= tau[j] - tau[k]
        beta[j] = 1.0 / prod
    return beta


BETA = barycentric_betas(TAU)


def lagrange_weights_1d(t: np.ndarray, tau: np.ndarray = TAU, beta: np.ndarray = BETA) -> np.ndarray:
    """Weights l_j(t) of degree-3 interpolation on nodes tau (second barycentric form).

    l_j(t) = (beta_j / (t - tau_j)) / sum_k (beta_k / (t - tau_k)); where t
    coincides with a node the weight vector is that node's unit vector.
    Returns shape (n, 4).
    """
    t = np.asarray(t, dtype=np.float64)
    diff = t[:, None] - tau[None, :]
    exact = diff == 0.0
    with np.errstate(divide="ignore", invalid="ignore"):
        q = beta[None, :] / diff
        w = q / np.sum(q, axis=1, keepdims=True)
    hit = np.any(exact, axis=1)
    w[hit] = exact[hit].astype(np.float64)
    return w


def stencil_of(cp: np.ndarray, h: float):
    """Per node: base lattice index (floor(cp/h) - 1) and offset t = cp/h - floor(cp/h)."""
    s = cp / h
    fl = np.floor(s)
    t = s - fl
    base = fl.astype(np.int64) - 1
    return base, t


OFFS = np.array([[a, b, c] for c in range(4) for b in range(4) for a in range(4)], dtype=np.int64)
# OFFS[q] = (a, b, c) with q = a + 4 b + 16 c


def extension_rows(band: Band, nodes_ijk: np.ndarray):
    """Column indices (into Sigma_A) and weights of E for the given nodes.

    Returns (cols (n, 64) int64, vals (n, 64) float64); raises if a stencil
    node is missing from Sigma_A ("StencilEscape") or cp is undefined.
    """
    x = lattice_points(nodes_ijk, band.h)
    cp, _ = band.surface.cp(x)
    if not np.all(np.isfinite(cp)):
        raise ValueError("closest point undefined at a band node (band too wide for the surface)")
    base, t = stencil_of(cp, band.h)
    wx = lagrange_weights_1d(t[:, 0])
    wy = lagrange_weights_1d(t[:, 1])
    wz = lagrange_weights_1d(t[:, 2])
    vals = wx[:, OFFS[:, 0]] * wy[:, OFFS[:, 1]] * wz[:, OFFS[:, 2]]
    sten = (base[:, None, :] + OFFS[None, :, :]).reshape(-1, 3)
    cols = _lookup(band.akeys, node_key(sten)).reshape(-1, 64)
    if np.any(cols < 0):
        raise ValueError("StencilEscape: interpolation stencil leaves Sigma_A")
    return cols, vals


def extension_matrix(band: Band) -> sp.csr_matrix:
    """E as an explicit sparse matrix: rows Sigma_A ++ Sigma_G, columns Sigma_A."""
    cols, vals = extension_rows(band, band.all)
    n = band.all.shape[0]
    rows = np.repeat(np.arange(n), 64)
    return sp.csr_matrix((vals.ravel(), (rows, cols.ravel())), shape=(n, band.nA))
