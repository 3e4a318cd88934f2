"""Per-rank compute share of the partitioned path, measured on ONE GPU.

For N = 2, 4, 8 Morton slabs of a band, every rank's LOCAL operator apply
(`cpm_part_apply_local`: its sub-band's extend + laplace, the halo supplied by plain
indexing — what the exchange would deliver) and LOCAL RAS apply
(`cpm_part_ras_apply_local`: its n_sub/N subdomains' inner solves) are timed alone,
one rank after the other, and compared with the unpartitioned call's time / N.
max_r(local) is the compute time of an N-GPU step without its communication; the
ratio (full / N) / max_r(local) is the load-balance / redundancy efficiency of the
partition (boundary tiles are evaluated by both neighbours, RAS overlap layers by
both subdomain owners).  The exchange and allreduce times are NOT in it (no
multi-GPU node in this pool) — DESIGN.md §Multi-GPU.

  python tools/part_share.py [config]     config = 1 (sphere h=1/200) | 2 (torus h=1/400, default)
                                          | 3 (sphere h=1/800, c=0.1, k_inner 64, overlap 16)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2110_06322_b200 as cpm
import seeded_inputs
from paper_2110_06322_b200 import cpm as C


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    k_inner = int(os.environ.get("CPM_KINNER", 64 if cfg == 3 else 16))
    overlap = 16 if cfg == 3 else 4
    if cfg == 3:
        band, c, name = cpm.cpm_build_band("sphere", 1.0 / 800), 0.1, "config 3 (sphere h=1/800)"
    elif cfg == 1:
        band, c, name = cpm.cpm_build_band("sphere", 1.0 / 200), 10.0, "config 1 (sphere h=1/200)"
    else:
        band, c, name = cpm.cpm_build_band("torus", 1.0 / 400, R=1.0, r=0.4), 1.0, "config 2 (torus h=1/400)"
    n = band.n
    ga = cpm.cpm_band_active_coords(band).astype(np.int64)
    u = torch.from_numpy(seeded_inputs.uniform_pm1(0, ga)).cuda()
    del ga
    y = torch.empty_like(u)
    out = {"band": name, "n_active": n, "k_inner": k_inner, "overlap": overlap, "ranks": {}}
    out["apply_full_us"] = timed(lambda: cpm.cpm_apply(band, c, u, y), 50)
    ras = cpm.cpm_ras_setup(band, 8, overlap, k_inner, c)
    z = torch.empty_like(u)
    out["ras_full_us"] = timed(lambda: cpm.cpm_ras_apply(ras, u, z), 5)
    ras.close()
    del ras
    print(json.dumps({k: out[k] for k in ("band", "n_active", "apply_full_us", "ras_full_us")}), flush=True)
    for R in (2, 4, 8):
        rows = []
        for r in range(R):
            p = C.cpm_part_create(band, r, R)
            hn = torch.from_numpy(C.cpm_part_halo_nodes(p)).cuda()
            u_own = u[p.lo:p.hi].contiguous()
            u_halo = u[hn].contiguous()
            y_own = torch.empty(p.n_owned, dtype=torch.float64, device="cuda")
            t_apply = timed(lambda: C.cpm_part_apply_local(p, c, u_own, u_halo, y_own), 50)
            pr = C.cpm_part_ras_setup(p, 8, overlap, k_inner, c)
            rh = torch.from_numpy(C.cpm_ras_halo_nodes(pr)).cuda()
            r_halo = u[rh].contiguous()
            t_ras = timed(lambda: C.cpm_part_ras_apply_local(pr, u_own, r_halo, y_own), 5)
            rows.append({"rank": r, "owned": p.n_owned, "halo": p.n_halo, "tiles": p.n_tiles,
                         "interior_tiles": p.n_interior_tiles, "ras_halo": int(rh.numel()),
                         "apply_local_us": t_apply, "ras_local_us": t_ras})
            pr.close()
            p.close()
            del pr, p, hn, rh, u_own, u_halo, r_halo, y_own
            torch.cuda.empty_cache()
        ma = max(x["apply_local_us"] for x in rows)
        mr = max(x["ras_local_us"] for x in rows)
        out["ranks"][R] = {
            "per_rank": rows,
            "apply_local_max_us": ma, "apply_share_efficiency": out["apply_full_us"] / R / ma,
            "ras_local_max_us": mr, "ras_share_efficiency": out["ras_full_us"] / R / mr,
            "halo_max": max(x["halo"] for x in rows), "ras_halo_max": max(x["ras_halo"] for x in rows),
        }
        print(json.dumps({"N": R, **{k: v for k, v in out["ranks"][R].items() if k != "per_rank"}}), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
