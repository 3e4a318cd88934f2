"""Computational band: active nodes Sigma_A and ghost nodes Sigma_G — oracle.

PAPER.md:62  "A structured grid with spacing h is placed over the embedding
space, and points near the surface are collected into the set of active
nodes Sigma_A. The points neighboring the members of Sigma_A are gathered
into the set of ghost nodes Sigma_G."
PAPER.md:78  "Along the edges of the tube of active nodes in Sigma_A there
will be incomplete finite difference stencils. The ghost nodes in Sigma_G
complete these stencils."

Reading R1: Sigma_A is the lambda-tube of BASELINE.json's
north_star, {x = h*(i,j,k) in [-L, L]^3 : |x - cp(x)| <= lambda},
lambda = sqrt(17)*h (the Ruuth-Merriman bandwidth for d=3, p=3).  Sigma_G is
every lattice node outside Sigma_A with a 6-neighbour in Sigma_A.

Lattice coordinates are integers (i, j, k); the point is x = i*h (one rounded
product per coordinate), the grid is |i|, |j|, |k| <= M = round(L/h).
"""
from __future__ import annotations

import math

import numpy as np

OFF = 1 << 20  # key offset, |i| < 2**20


def lam_of(h: float) -> float:
    """Band radius lambda = sqrt(17) h (north_star; reading R1)."""
    return math.sqrt(17.0) * h


def node_key(ijk: np.ndarray) -> np.ndarray:
    """Injective int64 key of lattice triples (lookup helper, no method arithmetic)."""
    ijk = np.asarray(ijk, dtype=np.int64)
    return ((ijk[:, 0] + OFF) << 42) | ((ijk[:, 1] + OFF) << 21) | (ijk[:, 2] + OFF)


def lattice_points(ijk: np.ndarray, h: float) -> np.ndarray:
    return np.asarray(ijk, dtype=np.int64).astype(np.float64) * h


NEIGHBORS6 = np.array(
    [[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]], dtype=np.int64
)


class Band:
    """Sigma_A (active, the unknowns) and Sigma_G (ghosts), sorted by node_key."""

    def __init__(self, surface, h: float, L: float = 2.0):
        self.surface = surface
        self.h = float(h)
        self.L = float(L)
        self.M = int(round(L / h))
        self.lam = lam_of(self.h)
        self.active = _active_nodes(surface, self.h, self.M, self.lam)
        self.akeys = node_key(self.active)
        self.ghost = _ghost_nodes(self.active, self.akeys)
        self.gkeys = node_key(self.ghost)
        # all nodes that carry a row of E: Sigma_A then Sigma_G
        self.all = np.concatenate([self.active, self.ghost], axis=0)
        self.allkeys = np.concatenate([self.akeys, self.gkeys])

    @property
    def nA(self) -> int:
        return self.active.shape[0]

    @property
    def nG(self) -> int:
        return self.ghost.shape[0]

    def index_active(self, ijk: np.ndarray) -> np.ndarray:
        """Row index in Sigma_A of each triple, -1 if absent."""
        return _lookup(self.akeys, node_key(ijk))

    def index_all(self, ijk: np.ndarray) -> np.ndarray:
        """Index in Sigma_A ++ Sigma_G, -1 if absent."""
        ia = _lookup(self.akeys, node_key(ijk))
        ig = _lookup(self.gkeys, node_key(ijk))
        return np.where(ia >= 0, ia, np.where(ig >= 0, ig + self.nA, -1))


def _lookup(sorted_keys: np.ndarray, q: np.ndarray) -> np.ndarray:
    if len(sorted_keys) == 0:
        return np.full(q.shape, -1, dtype=np.int64)
    pos = np.minimum(np.searchsorted(sorted_keys, q), len(sorted_keys) - 1)
    return np.where(sorted_keys[pos] == q, pos, -1).astype(np.int64)


def _active_nodes(surface, h: float, M: int, lam: float) -> np.ndarray:
    """Sigma_A by direct test of every lattice node in the surface's padded box."""
    lo, hi = surface.bbox(lam + h)
    ilo = [max(-M, int(math.floor(lo[c] / h)) - 1) for c in range(3)]
    ihi = [min(M, int(math.ceil(hi[c] / h)) + 1) for c in range(3)]
    ii, jj = np.meshgrid(
        np.arange(ilo[0], ihi[0] + 1, dtype=np.int64),
        np.arange(ilo[1], ihi[1] + 1, dtype=np.int64),
        indexing="ij",
    )
    ii = ii.ravel()
    jj = jj.ravel()
    out = []
    for k in range(ilo[2], ihi[2] + 1):
        ijk = np.stack([ii, jj, np.full_like(ii, k)], axis=1)
        x = lattice_points(ijk, h)
        _, dist = surface.cp(x)
        out.append(ijk[dist <= lam])
    act = np.concatenate(out, axis=0) if out else np.zeros((0, 3), np.int64)
    order = np.argsort(node_key(act), kind="stable")
    return act[order]


def _ghost_nodes(active: np.ndarray, akeys: np.ndarray) -> np.ndarray:
    cand = (active[:, None, :] + NEIGHBORS6[None, :, :]).reshape(-1, 3)
    ck = np.unique(node_key(cand))
    ghost_keys = ck[~np.isin(ck, akeys)]
    i = (ghost_keys >> 42) - OFF
    j = ((ghost_keys >> 21) & ((1 << 21) - 1)) - OFF
    k = (ghost_keys & ((1 << 21) - 1)) - OFF
    return np.stack([i, j, k], axis=1).astype(np.int64)


def brute_force_band(dist_fn, h: float, L: float = 2.0):
    """Pure-Python triple loop over the whole grid (pin for tiny grids only).

    dist_fn(x, y, z) -> distance to the surface, supplied by the test in an
    independent closed form (not the oracle's cp code).
    """
    M = int(round(L / h))
    lam = math.sqrt(17.0) * h
    act = set()
    for i in range(-M, M + 1):
        for j in range(-M, M + 1):
            for k in range(-M, M + 1):
                if dist_fn(i * h, j * h, k * h) <= lam:
                    act.add((i, j, k))
    ghost = set()
    for (i, j, k) in act:
        for di, dj, dk in NEIGHBORS6.tolist():
            q = (i + di, j + dj, k + dk)
            if q not in act:
                ghost.add(q)
    return act, ghost
