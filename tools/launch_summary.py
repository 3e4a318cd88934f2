"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel."""
import csv
import sys
from collections import defaultdict


def summarise(path, title=""):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[i]
    ki, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[i + 1:]:
        if len(r) <= mi:
            continue
        name = r[ki].split("(")[0].split("<")[0].strip()
        if "::" in name:
            name = name.split("::")[-1]
        if name == "" or name.startswith("cpm"):
            name = r[ki].split("(")[0].split("::")[-1]
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        tot[name] += float(r[mi].replace(",", "")) * scale
        cnt[name] += 1
    T = sum(tot.values())
    out = [f"# {title}", "kernel,launches,total_us,mean_us,share"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"{k},{cnt[k]},{v:.1f},{v / cnt[k]:.2f},{v / T:.3f}")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    s = summarise(sys.argv[1], sys.argv[3] if len(sys.argv) > 3 else "")
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(s)
    print(s)
