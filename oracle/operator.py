"""Discrete operators of the CPM — oracle.

PAPER.md:78  "The ambient Laplacian, Delta, over the embedding space is
discretized by standard second-order centered finite differences, denoted
Delta^h."
PAPER.md:80-85, Eq. (4):
    Delta_S^h = -(2d/h^2) I + (Delta^h + (2d/h^2) I) E
"where the removal of the diagonal elements from Delta^h avoids redundant
self-interpolation."
PAPER.md:31-34, Eq. (2):  (c - Delta_S) u = f,  c > 0.

With d = 3 the shifted operator is A = c I - Delta_S^h, which is BASELINE's
y = c u - [Delta_h E u - (6/h^2)(u - E u)].
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .band import NEIGHBORS6, Band
from .interp import OFFS, extension_matrix, extension_rows, lagrange_weights_1d, stencil_of


def laplacian_matrix(band: Band) -> sp.csr_matrix:
    """Delta^h: rows Sigma_A, columns Sigma_A ++ Sigma_G; 7-point, (1/h^2)(sum nbrs - 6 centre)."""
    nA = band.nA
    h2 = band.h * band.h
    rows = [np.arange(nA)]
    cols = [np.arange(nA)]
    vals = [np.full(nA, -6.0 / h2)]
    for off in NEIGHBORS6:
        idx = band.index_all(band.active + off[None, :])
        if np.any(idx < 0):
            raise ValueError("a neighbour of an active node is missing from Sigma_A u Sigma_G")
        rows.append(np.arange(nA))
        cols.append(idx)
        vals.append(np.full(nA, 1.0 / h2))
    return sp.csr_matrix(
        (np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
        shape=(nA, nA + band.nG),
    )


def laplace_beltrami_matrix(band: Band, E: sp.csr_matrix | None = None) -> sp.csr_matrix:
    """Delta_S^h = -(6/h^2) I + (Delta^h + (6/h^2) I) E   (Eq. 4, d = 3).

    The "I" inside the bracket is the |Sigma_A| x |Sigma_A u Sigma_G| selector of
    the active rows, so that Delta^h + (6/h^2) I drops exactly the diagonal of
    Delta^h.
    """
    if E is None:
        E = extension_matrix(band)
    nA = band.nA
    d2 = 6.0 / (band.h * band.h)
    Dh = laplacian_matrix(band)
    P = sp.csr_matrix((np.ones(nA), (np.arange(nA), np.arange(nA))), shape=(nA, nA + band.nG))
    return (-d2 * sp.identity(nA, format="csr") + (Dh + d2 * P) @ E).tocsr()


def shifted_operator(band: Band, c: float, E: sp.csr_matrix | None = None) -> sp.csr_matrix:
    """A = c I - Delta_S^h  (Eq. 2 discretised with Eq. 4)."""
    return (c * sp.identity(band.nA, format="csr") - laplace_beltrami_matrix(band, E)).tocsr()


def apply_rows(band: Band, c: float, u_of_ijk, rows_ijk: np.ndarray) -> np.ndarray:
    """(A u)_i for selected active nodes, one by one from the definition (Eq. 2, 4).

    u_of_ijk(ijk (n,3)) -> values of u at those lattice nodes (all in Sigma_A).
    Used for sampled parity at sizes where assembling E is too slow:
    (Delta_S^h u)_i = -(6/h^2) u_i + (1/h^2)(sum_nbr (Eu)_j - 6 (Eu)_i) + (6/h^2)(Eu)_i.
    """
    h2 = band.h * band.h
    d2 = 6.0 / h2
    rows_ijk = np.asarray(rows_ijk, dtype=np.int64)
    n = rows_ijk.shape[0]

    def Eu_at(ijk):
        x = ijk.astype(np.float64) * band.h
        cp, _ = band.surface.cp(x)
        base, t = stencil_of(cp, band.h)
        wx = lagrange_weights_1d(t[:, 0])
        wy = lagrange_weights_1d(t[:, 1])
        wz = lagrange_weights_1d(t[:, 2])
        w = wx[:, OFFS[:, 0]] * wy[:, OFFS[:, 1]] * wz[:, OFFS[:, 2]]
        sten = (base[:, None, :] + OFFS[None, :, :]).reshape(-1, 3)
        uv = u_of_ijk(sten).reshape(-1, 64)
        return np.sum(w * uv, axis=1)

    u_i = u_of_ijk(rows_ijk)
    Eu_i = Eu_at(rows_ijk)
    nb = np.zeros(n)
    for off in NEIGHBORS6:
        nb = nb + Eu_at(rows_ijk + off[None, :])
    lap = -d2 * u_i + (nb - 6.0 * Eu_i) / h2 + d2 * Eu_i
    return c * u_i - lap


__all__ = [
    "laplacian_matrix",
    "laplace_beltrami_matrix",
    "shifted_operator",
    "apply_rows",
    "extension_matrix",
    "extension_rows",
]
