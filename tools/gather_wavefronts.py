"""Predicted shared-memory wavefronts of the extend's stencil gathers from a band's
node order, with the measured half-warp rule (profiles/r02_micro_lds_halves.txt):
a warp LDS.64 costs 1 wavefront when its distinct addresses are <= 16 in distinct
bank pairs (residue = offset mod 16), else the sum over its two half-warps of the
largest number of distinct addresses sharing a residue.  Also the lower bound of the
singles region, max(ceil(S / 16), largest residue class) per tile, and what a
dealing into short (never-conflicting) half-warp groups would reach.

usage: python tools/gather_wavefronts.py ORDER.npz   (tiles, eoff of cpm_band_eval_order)
"""
import sys

import numpy as np


def warp_cost(b):
    act = b >= 0
    if not act.any():
        return 0
    addrs = np.unique(b[act])
    if len(addrs) <= 16 and len(np.unique(addrs & 15)) == len(addrs):
        return 1
    tot = 0
    for h in (b[:16], b[16:]):
        a = np.unique(h[h >= 0])
        if len(a):
            tot += np.bincount(a & 15).max()
    return tot


def main():
    d = np.load(sys.argv[1])
    tiles, eoff = d["tiles"].astype(np.int64), d["eoff"].astype(np.int64)
    cats = {}
    lb = 0
    for e0, e1, npnd, sx, sxy, cells in tiles:
        ne = e1 - e0
        np_, nd = npnd & 0xFFFF, npnd >> 16
        np2 = 2 * np_
        nslot = ne + nd
        s = np.arange(nslot)
        node = np.where(s < np2, s, np.where(s < np2 + 2 * nd, np2 + (s - np2) // 2, s - nd))
        base = eoff[e0 + node] & 0xFFFF
        for w0 in range(0, nslot, 32):
            b = np.full(32, -1)
            m = min(32, nslot - w0)
            b[:m] = base[w0:w0 + m]
            kind = "pair" if w0 + 32 <= np2 else ("single" if w0 >= np2 + 2 * nd else "mixed")
            c = cats.setdefault(kind, [0, 0])
            c[0] += warp_cost(b)
            c[1] += 1
        res = (base[np2 + 2 * nd:] & 15) if nslot > np2 + 2 * nd else np.zeros(0, dtype=np.int64)
        if len(res):
            cnt = np.bincount(res, minlength=16)
            lb += max((len(res) + 15) // 16, cnt.max())
    tot = sum(v[0] for v in cats.values())
    print(f"predicted gather wavefronts per apply: {64 * tot / 1e6:.2f} M")
    for k, (c, n) in cats.items():
        print(f"  {k:6s} warps {n:7d}  {64 * c / 1e6:.2f} M")
    print(f"singles region lower bound {64 * lb / 1e6:.2f} M (short-group dealing reaches it)")


if __name__ == "__main__":
    main()
