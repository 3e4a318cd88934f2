"""Group sizes of eval nodes (Sigma_A u Sigma_G) by stencil base cell (analysis for
DESIGN.md §Open items; CPU, uses only oracle/ geometry — a tool, not a product path).

Prints, for the unit sphere at spacing h: nodes per distinct base over the whole band
(what a tiling by the BASE's brick would see) and per (node brick, base) pair (what the
current tiling by the NODE's brick sees), and the share of nodes in groups of >= 2 / >= 4.
"""
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from oracle.band import Band, lattice_points  # noqa: E402
from oracle.interp import stencil_of  # noqa: E402
from oracle.surfaces import Sphere  # noqa: E402


def stats(keys, label):
    _, cnt = np.unique(keys, return_counts=True, axis=0)
    n = cnt.sum()
    print(f"{label}: {len(cnt)} groups, mean {n / len(cnt):.2f} nodes; nodes in groups >=2: "
          f"{cnt[cnt >= 2].sum() / n:.3f}, >=4: {cnt[cnt >= 4].sum() / n:.3f}, >=6: {cnt[cnt >= 6].sum() / n:.3f}; "
          f"gathers per node with per-group reuse {64 * len(cnt) / n:.1f} (64 without)")


def main():
    h = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0 / 50
    b = Band(Sphere(1.0), h)
    nodes = np.concatenate([b.active, b.ghost])
    cp = b.surface.cp(lattice_points(nodes, h))[0]
    base = stencil_of(cp, h)[0]
    base = np.asarray(base, dtype=np.int64)
    print(f"sphere h={h:g}: {len(nodes)} eval nodes")
    stats(base, "by base (base-brick tiling)")
    nb = nodes >> 3
    stats(np.concatenate([nb, base], axis=1), "by (node brick, base) (current tiling)")
    bb = base >> 3
    _, tc = np.unique(bb, return_counts=True, axis=0)
    _, nc = np.unique(nb, return_counts=True, axis=0)
    print(f"tiles: {len(nc)} node bricks (mean {nc.mean():.0f} eval nodes), {len(tc)} base bricks (mean {tc.mean():.0f})")


if __name__ == "__main__":
    main()


def quad_efficiency(h):
    """Slots of a quad-item order (items of <= 4 equal-base nodes inside a node brick)."""
    b = Band(Sphere(1.0), h)
    nodes = np.concatenate([b.active, b.ghost])
    cp = b.surface.cp(lattice_points(nodes, h))[0]
    base = np.asarray(stencil_of(cp, h)[0], dtype=np.int64)
    _, cnt = np.unique(np.concatenate([nodes >> 3, base], axis=1), return_counts=True, axis=0)
    n = cnt.sum()
    items = ((cnt + 3) // 4).sum()
    hist = np.bincount(cnt)
    print("group-size histogram (share of nodes):", {g: round(float(g * hist[g] / n), 3) for g in range(1, len(hist)) if hist[g]})
    print(f"quad items {items}, slots {4 * items}, slot efficiency {n / (4 * items):.3f}, "
          f"value loads per node {64 * items / n:.1f}")


if __name__ == "__main__" and len(sys.argv) > 2:
    quad_efficiency(float(sys.argv[1]))
