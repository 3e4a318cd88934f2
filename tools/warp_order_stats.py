"""Shared-memory wavefronts of the extend's stencil gathers, predicted from the
band's node order (cpm_band_eval_order) with the measured B200 rule (DESIGN.md
§Kernels): an 8-byte warp load costs max(ceil(D / 16), largest number of distinct
addresses in one 8-byte bank) wavefronts, D = distinct addresses of the warp.

usage: python tools/warp_order_stats.py [h] [n_sample_tiles]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2110_06322_b200 as cpm

NT = 128  # threads per extend CTA (apply.cu kNtThreads)


def tile_warps(e0, e1, npnd, sx, sxy, eoff):
    """Per warp of the tile: (round k, slot bases [32] or -1, is-single flags).
    npnd = np | nd << 16 (apply.cu slot_node: pairs, nd duplicated singles, singles)."""
    ne = e1 - e0
    np_, nd = npnd & 0xFFFF, npnd >> 16
    np2 = 2 * np_
    nslot = ne + nd
    s = np.arange(nslot)
    node = np.where(s < np2, s, np.where(s < np2 + 2 * nd, np2 + (s - np2) // 2, s - nd))
    base = (eoff[e0 + node] & 0xFFFF).astype(np.int64)
    single = s >= np2
    out = []
    for w0 in range(0, nslot, 32):
        b = np.full(32, -1, dtype=np.int64)
        m = min(32, nslot - w0)
        b[:m] = base[w0:w0 + m]
        out.append(((w0 // NT), b, single[w0:w0 + m].mean()))
    return out


def warp_cost(b, sx, sxy):
    """Predicted wavefronts and ideal (ceil(D/16)) summed over the 64 gathers."""
    act = b[b >= 0]
    offs = np.array([c * sxy + bb * sx + i for c in range(4) for bb in range(4) for i in range(4)])
    addr = act[None, :] + offs[:, None]  # 64 x lanes
    wf = ideal = 0
    for row in addr:
        u = np.unique(row)
        d = len(u)
        bank = np.bincount(u % 16, minlength=16).max()
        wf += max((d + 15) // 16, bank)
        ideal += (d + 15) // 16
    return wf, ideal


def redeal(e0, e1, np_, eoff):
    """Alternative dealing (simulation, REDEAL=1): items (pairs, then singles)
    assigned to warps of 16 items greedily by residue, most constrained residue
    first; returns the slot bases in the kernel's slot order.  Predicts 16.5M
    instead of 17.0M wavefronts at h = 1/200; built in k_warp_order it left the
    extend time unchanged (134.7 vs 134.3 us), so the build keeps its dealing."""
    ne = e1 - e0
    base = (eoff[e0:e1] & 0xFFFF).astype(np.int64)
    pairs = [int(base[2 * p]) for p in range(np_)]
    singles = [int(b) for b in base[2 * np_:]]
    P, S = len(pairs), len(singles)
    I = P + S
    W = (I + 15) // 16
    cap_p = [min(16, max(0, P - 16 * w)) for w in range(W)]          # pair positions per warp
    cap_s = [(min(16, I - 16 * w)) - cap_p[w] for w in range(W)]      # single positions
    warps = [dict() for _ in range(W)]  # residue -> set of bases
    content_p = [[] for _ in range(W)]
    content_s = [[] for _ in range(W)]

    def place(items, cap, content):
        from collections import Counter
        cnt = Counter(b % 16 for b in items)
        order = sorted(items, key=lambda b: (-cnt[b % 16], b % 16, b))
        for b in order:
            r = b % 16
            best, bkey = -1, None
            for w in range(W):
                if cap[w] == 0:
                    continue
                d = warps[w].get(r, set())
                cost = 0 if (not d or b in d) else len(d)
                key = (cost, 0 if b in d else 1, -cap[w])
                if bkey is None or key < bkey:
                    best, bkey = w, key
            warps[best].setdefault(r, set()).add(b)
            cap[best] -= 1
            content[best].append(b)

    place(pairs, cap_p, content_p)
    place(singles, cap_s, content_s)
    slots = []
    for w in range(W):
        for b in content_p[w]:
            slots += [b, b]
    for w in range(W):
        for b in content_s[w]:
            slots += [b, b]
    return np.array(slots, dtype=np.int64)


def main():
    h = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0 / 200
    ns = int(sys.argv[2]) if len(sys.argv) > 2 else 1500
    band = cpm.cpm_build_band("sphere", h)
    tiles, eoff = cpm.cpm_band_eval_order(band)
    rng = np.random.default_rng(0)
    pick = rng.choice(len(tiles), size=min(ns, len(tiles)), replace=False)
    by_round = {}
    for t in pick:
        e0, e1, np_, sx, sxy, _ = (int(v) for v in tiles[t])
        if os.environ.get("REDEAL"):
            sl = redeal(e0, e1, np_ & 0xFFFF, eoff)
            ws = [(w0 // NT, np.pad(sl[w0:w0 + 32], (0, max(0, 32 - len(sl[w0:w0 + 32]))),
                                    constant_values=-1), 0.0) for w0 in range(0, len(sl), 32)]
        else:
            ws = tile_warps(e0, e1, np_, sx, sxy, eoff)
        for k, b, fs in ws:
            wf, ideal = warp_cost(b, sx, sxy)
            r = by_round.setdefault(min(k, 3), [0, 0, 0, 0.0])
            r[0] += 64
            r[1] += wf
            r[2] += ideal
            r[3] += fs * 64
    scale = len(tiles) / len(pick)
    tot = [0, 0, 0]
    for k in sorted(by_round):
        n, wf, ideal, fs = by_round[k]
        tot = [tot[0] + n, tot[1] + wf, tot[2] + ideal]
        print(f"round {k}{'+' if k == 3 else ''}: inst {n * scale / 1e6:6.2f}M  wf/inst {wf / n:.3f}  "
              f"ideal/inst {ideal / n:.3f}  single-slot fraction {fs / n:.2f}")
    print(f"total: inst {tot[0] * scale / 1e6:.2f}M wf {tot[1] * scale / 1e6:.2f}M ideal {tot[2] * scale / 1e6:.2f}M")


if __name__ == "__main__":
    main()
