"""Full-size BASELINE configs on the GPU: band build, RAS set-up, RAS-FGMRES(50) solve
(configs 2, 3), Schnakenberg IMEX steps (config 4); one JSON line per run.

usage: python tools/run_configs.py [2] [3] [4] [--k 16] [--h H] [--nsub 8]
       torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/run_configs.py 2 --dist
         (config 2 / 3 partitioned over N GPUs: NCCL halo + distributed RAS + FGMRES)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2110_06322_b200 as cpm
import seeded_inputs


def run(cfg: int, k_inner: int = 8, restart: int = 50, maxit: int = 20000, h=None, nsub: int = 8,
        overlap: int = 4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if cfg == 2:
        band = cpm.cpm_build_band("torus", h or 1.0 / 400, R=1.0, r=0.4)
        c = 1.0
    else:
        band = cpm.cpm_build_band("sphere", h or 1.0 / 800)
        c = 0.1
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    n = band.n
    f = torch.empty(n, dtype=torch.float64, device="cuda")
    if cfg == 2:
        cpm.cpm_eval_torus_rhs(band, seeded_inputs.smooth_modulation_coeffs(1), f)
    else:
        cpm.cpm_eval_sph(band, 10, 5, 1.0, f)
        ga = cpm.cpm_band_active_coords(band).astype(np.int64)
        f += torch.from_numpy(1e-3 * seeded_inputs.normal(2, ga)).cuda()
    t0 = time.perf_counter()
    ras = cpm.cpm_ras_setup(band, nsub, overlap, k_inner, c) if k_inner > 0 else None
    torch.cuda.synchronize()
    t_ras = time.perf_counter() - t0
    u = torch.zeros_like(f)
    cpm.cpm_profile_reset()
    cpm.cpm_profile_enable(True)
    st = cpm.cpm_solve(band, c, f, u, rtol=1e-10, restart=restart, maxit=maxit, ras=ras)
    cpm.cpm_profile_enable(False)
    prof = {k: round(cpm.cpm_profile_read(k)[0], 1) for k in
            ["extend", "laplace", "mdot", "cgs_update", "cgs_final", "axpy", "other"]}
    return {"config": cfg, "h": band.info.h, "nsub": nsub if k_inner > 0 else 0, "overlap": overlap, "n_active": n, "n_ghost": band.info.n_ghost, "tiles": band.info.n_tiles,
            "build_s": round(t_build, 3), "ras_setup_s": round(t_ras, 3), "k_inner": k_inner,
            "solve_s": round(st.seconds, 3), "iterations": st.iterations, "converged": bool(st.converged),
            "resid_true_rel": st.resid_true / st.bnorm, "ms_per_iteration": round(1e3 * st.seconds / max(st.iterations, 1), 3),
            "kernel_ms": prof, "device_bytes": band.info.bytes_device}


def run_rd(h=1.0 / 400, steps=200):
    """Config 4: Schnakenberg IMEX Euler on the torus, dt = 1e-3, `steps` steps."""
    band = cpm.cpm_build_band("torus", h, R=1.0, r=0.4)
    ga = cpm.cpm_band_active_coords(band).astype(np.int64)
    a, b = 0.1, 0.9
    u = torch.from_numpy(a + b + 1e-2 * seeded_inputs.uniform_pm1(3, ga, stream=0)).cuda()
    v = torch.from_numpy(b / (a + b) ** 2 + 1e-2 * seeded_inputs.uniform_pm1(3, ga, stream=1)).cuda()
    its = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        s1, s2 = cpm.cpm_rd_step(band, u, v)
        its.append((s1.iterations, s2.iterations))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    it = np.array(its)
    return {"config": 4, "h": h, "n_active": band.n, "steps": steps, "seconds": round(dt, 3),
            "ms_per_step": round(1e3 * dt / steps, 3), "gmres_its_u_mean": float(it[:, 0].mean()),
            "gmres_its_v_mean": float(it[:, 1].mean()), "u_range": [float(u.min()), float(u.max())],
            "v_range": [float(v.min()), float(v.max())]}


def run_dist(cfg: int, k_inner: int = 16, restart: int = 50, maxit: int = 20000, h=None, nsub: int = 8):
    """Config 2 / 3 partitioned over the ranks of a torchrun job (one GPU each): Morton
    slabs, NCCL halo exchange, distributed RAS (nsub a multiple of the rank count),
    distributed FGMRES; prints the max-over-ranks solve time on rank 0."""
    import torch.distributed as dist

    from paper_2110_06322_b200.distributed import DistributedCPM

    dist.init_process_group("nccl")
    rank, nr = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    if cfg == 2:
        band = cpm.cpm_build_band("torus", h or 1.0 / 400, R=1.0, r=0.4)
        c = 1.0
    else:
        band = cpm.cpm_build_band("sphere", h or 1.0 / 800)
        c = 0.1
    f = torch.empty(band.n, dtype=torch.float64, device="cuda")
    if cfg == 2:
        cpm.cpm_eval_torus_rhs(band, seeded_inputs.smooth_modulation_coeffs(1), f)
    else:
        cpm.cpm_eval_sph(band, 10, 5, 1.0, f)
        ga = cpm.cpm_band_active_coords(band).astype(np.int64)
        f += torch.from_numpy(1e-3 * seeded_inputs.normal(2, ga)).cuda()
    D = DistributedCPM(band)
    ras = D.setup_ras(nsub, 4, k_inner, c)
    fo = f[D.lo:D.hi].contiguous()
    uo = torch.zeros_like(fo)
    dist.barrier()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    st = D.solve(c, fo, uo, rtol=1e-10, restart=restart, maxit=maxit, ras=ras)
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / 1e3], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"config": cfg, "ranks": nr, "n_active": band.n, "nsub": nsub, "k_inner": k_inner,
                          "solve_s_max_over_ranks": float(t.item()), "iterations": st.iterations,
                          "converged": bool(st.converged), "resid_true_rel": st.resid_true / st.bnorm}),
              flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", type=int, default=[2, 3])
    ap.add_argument("--h", type=float, default=None, help="override the lattice spacing")
    ap.add_argument("--k", type=int, nargs="*", default=[8], help="inner GMRES steps (0: no RAS)")
    ap.add_argument("--nsub", type=int, default=8)
    ap.add_argument("--overlap", type=int, nargs="*", default=[4], help="RAS overlap (lattice layers)")
    ap.add_argument("--maxit", type=int, default=20000)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--dist", action="store_true",
                    help="partitioned solve under torchrun (one rank per GPU, NCCL)")
    a = ap.parse_args()
    if a.dist:
        for c in a.configs:
            run_dist(c, k_inner=a.k[0], h=a.h, nsub=a.nsub, maxit=a.maxit)
        sys.exit(0)
    if 4 in a.configs:
        print(json.dumps(run_rd(h=a.h or 1.0 / 400, steps=a.steps)), flush=True)
    for c in [c for c in a.configs if c != 4]:
        for k in a.k:
            for ov in a.overlap:
                print(json.dumps(run(c, k_inner=k, h=a.h, nsub=a.nsub, maxit=a.maxit, overlap=ov)),
                      flush=True)
