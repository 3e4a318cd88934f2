"""One-level restricted additive Schwarz (RAS) preconditioner — oracle.

PAPER.md:91  "Consider splitting the global domain S into N_S disjoint
subdomains S~_j. Each disjoint subdomain is then grown to form an overlapping
set of subdomains S_j."
PAPER.md:99-102  "After the local solutions u_j are found on each overlapping
subdomain, a new global solution may be formed with respect to the disjoint
subdomains as u^(n+1) = sum_j u_j|_{S~_j}."
PAPER.md:105  T_jk = identity (Dirichlet transmission; the RAS default,
PAPER.md:252 "Dirichlet transmission conditions are the default option").

As a preconditioner (residual-correction form, zero Dirichlet data):
    z = M r = sum_j R~_j^T  A_j^{-1}  R_j r,     A_j = R_j A R_j^T,
R_j restricts to the overlapping S_j, R~_j^T prolongs from the disjoint S~_j.
Reading R6: A_j^{-1} is applied inexactly by exactly k_inner GMRES steps from
zero (north_star item 4, "inexact on-GPU local solves using a fixed inner
iteration count"); the preconditioner is then nonlinear, so the outer solver
is FGMRES (krylov.gmres with M).
Reading R7: overlap N_O is counted in lattice 6-neighbour layers inside
Sigma_A ("overlap 4h" = 4 layers).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .band import NEIGHBORS6, Band
from .krylov import arnoldi_fixed
from .order import band_order, slab_bounds


def disjoint_subdomains(band: Band, nsub: int) -> list[np.ndarray]:
    """S~_j: Morton slabs of the band order (reading R8), as sorted Sigma_A indices."""
    perm = band_order(band.active)
    b = slab_bounds(band.nA, nsub)
    return [np.sort(perm[b[s]: b[s + 1]]) for s in range(nsub)]


def grow_overlap(band: Band, disjoint: np.ndarray, layers: int) -> np.ndarray:
    """S_j: add `layers` rings of active 6-neighbours to S~_j (reading R7)."""
    inside = np.zeros(band.nA, dtype=bool)
    inside[disjoint] = True
    nbr = np.stack([band.index_active(band.active + off[None, :]) for off in NEIGHBORS6], axis=1)
    for _ in range(layers):
        grow = inside.copy()
        for c in range(6):
            ok = nbr[:, c] >= 0
            grow[ok] |= inside[nbr[ok, c]]
        inside = grow
    return np.nonzero(inside)[0]


class RAS:
    """z = sum_j R~_j^T solve_j(R_j r).  local='gmres' (k_inner steps) or 'exact'."""

    def __init__(self, band: Band, A: sp.csr_matrix, nsub: int, overlap: int,
                 k_inner: int = 10, local: str = "gmres"):
        self.nA = band.nA
        self.k = int(k_inner)
        self.local = local
        self.disjoint = disjoint_subdomains(band, nsub)
        self.over = [grow_overlap(band, d, overlap) for d in self.disjoint]
        self.Aj = [A[o][:, o].tocsr() for o in self.over]   # R_j A R_j^T
        # position of each disjoint node inside its overlapping subdomain
        self.keep = [np.searchsorted(o, d) for o, d in zip(self.over, self.disjoint)]
        self.lu = [spla.splu(Aj.tocsc()) for Aj in self.Aj] if local == "exact" else None

    def __call__(self, r: np.ndarray) -> np.ndarray:
        z = np.zeros(self.nA)
        for j, (o, d) in enumerate(zip(self.over, self.disjoint)):
            rj = r[o]
            if self.local == "exact":
                zj = self.lu[j].solve(rj)
            else:
                Aj = self.Aj[j]
                zj = arnoldi_fixed(lambda v, Aj=Aj: Aj @ v, rj, self.k)
            z[d] = zj[self.keep[j]]
        return z
