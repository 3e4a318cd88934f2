"""Band ordering and Morton-slab partitions — oracle.

Not in the paper (PAPER.md:250 delegates partitioning to ParMETIS "though any
partitioner included in the Petsc installation can be used").  Reading R8
 fixes the partition the CUDA path and this oracle both implement:

  brick(i)  = floor(i / 8)           local(i) = i - 8 * brick(i)  in 0..7
  morton    = bit-interleave of (brick_x + 2^16, brick_y + 2^16, brick_z + 2^16),
              bit b of x -> 3b, of y -> 3b+1, of z -> 3b+2 (17 bits each)
  key       = morton * 512 + local_z * 64 + local_y * 8 + local_x
  band order = active nodes sorted by key (ascending)
  slab s of S = band-order positions [floor(s nA / S), floor((s+1) nA / S))

The same slabs are the disjoint subdomains of RAS (BASELINE config 2: "8
Morton-slab subdomains") and the per-GPU partitions (north_star item 5).
"""
from __future__ import annotations

import numpy as np


def _interleave(v: int) -> int:
    out = 0
    for b in range(17):
        out |= ((v >> b) & 1) << (3 * b)
    return out


def band_order_key(ijk: np.ndarray) -> np.ndarray:
    """Key of reading R8 for each lattice triple (pure-Python bit loop per node)."""
    ijk = np.asarray(ijk, dtype=np.int64)
    keys = np.empty(ijk.shape[0], dtype=np.int64)
    for n in range(ijk.shape[0]):
        i, j, k = (int(v) for v in ijk[n])
        bx, by, bz = i // 8, j // 8, k // 8
        lx, ly, lz = i - 8 * bx, j - 8 * by, k - 8 * bz
        m = _interleave(bx + (1 << 16)) | (_interleave(by + (1 << 16)) << 1) | (_interleave(bz + (1 << 16)) << 2)
        keys[n] = m * 512 + lz * 64 + ly * 8 + lx
    return keys


def band_order(ijk: np.ndarray) -> np.ndarray:
    """Permutation sorting the given nodes into band order."""
    return np.argsort(band_order_key(ijk), kind="stable")


def slab_bounds(n: int, S: int) -> list[int]:
    return [(s * n) // S for s in range(S + 1)]
