"""Group an ncu report's LDS.64 SASS lines by execution count (one group per
inlined code path) and print wavefronts per instruction, actual and ideal.

usage: python tools/ncu_lds_paths.py REP
"""
import csv
import subprocess
import sys
from collections import defaultdict

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1] if rows[0][0] == "Kernel Name" else rows[0]
ix = {n: i for i, n in enumerate(h)}
g = defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0, None])
for r in rows[2:]:
    if len(r) != len(h) or "LDS.64" not in r[ix["Source"]]:
        continue
    ins = float(r[ix["Instructions Executed"]] or 0)
    if ins == 0:
        continue
    v = g[int(ins)]
    v[0] += 1
    v[1] += ins
    v[2] += float(r[ix["L1 Wavefronts Shared"]] or 0)
    v[3] += float(r[ix["L1 Wavefronts Shared Ideal"]] or 0)
    v[4] += float(r[ix["Thread Instructions Executed"]] or 0)
    v[5] = v[5] or r[ix["Address"]]
for k, v in sorted(g.items(), key=lambda kv: -kv[1][1]):
    print(f"path@{v[5][-5:]} lines {v[0]:3d} inst {v[1]:10.0f} wf/inst {v[2] / v[1]:5.2f} "
          f"ideal {v[3] / v[1]:5.2f} threads {v[4] / v[1]:5.1f}")
