"""Per-SASS-opcode totals of an ncu report's source page (--import-source on):
instructions, thread instructions, shared wavefronts (actual / ideal), L1 global tag
requests, warp stall samples.

usage: python tools/ncu_sass_ops.py REP
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    ix = {n: i for i, n in enumerate(h)}
    cols = ["Instructions Executed", "Thread Instructions Executed", "L1 Wavefronts Shared",
            "L1 Wavefronts Shared Ideal", "L1 Tag Requests Global", "Warp Stall Sampling (All Samples)"]
    agg = defaultdict(lambda: [0.0] * len(cols))
    for r in rows[1:]:
        if len(r) != len(h):
            continue
        op = r[ix["Source"]].strip().split()
        if not op:
            continue
        k = op[0] if not op[0].startswith("@") else op[1]
        for j, c in enumerate(cols):
            try:
                agg[k][j] += float(r[ix[c]] or 0)
            except (ValueError, KeyError):
                pass
    tot = [sum(v[j] for v in agg.values()) for j in range(len(cols))]
    print(f"{'opcode':24s} {'inst':>12s} {'thr/inst':>8s} {'shWF':>12s} {'shWFideal':>12s} {'tags':>10s} {'stall%':>7s}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:30]:
        print(f"{k:24s} {v[0]:12.0f} {v[1] / max(v[0], 1):8.1f} {v[2]:12.0f} {v[3]:12.0f} {v[4]:10.0f} "
              f"{100 * v[5] / max(tot[5], 1):7.1f}")
    print(f"{'TOTAL':24s} {tot[0]:12.0f} {tot[1] / max(tot[0], 1):8.1f} {tot[2]:12.0f} {tot[3]:12.0f} {tot[4]:10.0f}")


if __name__ == "__main__":
    main()
