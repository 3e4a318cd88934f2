"""Per-source-line stall summary of an ncu report (`ncu -i REP --page source --csv`).

usage: python tools/ncu_source.py REP [top_n]
Prints the stall-reason totals and the source lines with the most warp samples.
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    lines = out.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    idx = {n: i for i, n in enumerate(h)}
    stall_cols = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
    tot = {n: 0.0 for n in stall_cols}
    body = []
    for r in rows[1:]:
        if len(r) != len(h):
            continue
        try:
            s = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        for n in stall_cols:
            try:
                tot[n] += float(r[idx[n]] or 0)
            except ValueError:
                pass
        body.append((s, r))
    all_s = sum(s for s, _ in body) or 1.0
    print("stall totals (% of samples):")
    for n, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
        print(f"  {n:28s} {100 * v / all_s:6.1f}")
    print(f"top {top} lines:")
    for s, r in sorted(body, key=lambda x: -x[0])[:top]:
        reasons = sorted(((float(r[idx[n]] or 0), n) for n in stall_cols), reverse=True)[:3]
        rs = ", ".join(f"{n[6:]}={100 * v / all_s:.1f}" for v, n in reasons if v > 0)
        print(f"{100 * s / all_s:5.1f}%  {r[idx['Source']][:90]:90s} | {rs}")


if __name__ == "__main__":
    main()
