#!/usr/bin/env python
"""bench.py — CPM hot path on B200 (BASELINE.json metric, config 1).

A step is one pass of the hot path over config 1 (BASELINE.json configs[1]):
unit sphere, h = 1/200 (~4.1M band nodes), fp64:
  * 100 operator applies y = (c - Delta_S^h) u on u ~ U[-1,1] (seed 0), c = 10
  * the manufactured solve (c - Delta_S^h) u = (c + 42) Y_6^3(cp), GMRES(50), rtol 1e-10
`value` = band-node applies per second over the timed applies (CUDA events on the
launching stream, max over ranks); `solve` reports the GMRES solve time.  The
band is built once, outside the timed region (its build time is reported).
Outside the timed steps, rank 0 also reports `config4_rd` (config-4 IMEX steps)
and `config2_solve` (one config-2 RAS-FGMRES solve, ~40 s; --c2-kinner 0 skips it);
with --c2-dist under torchrun (N | 8) every rank joins a partitioned config-2
solve (`config2_solve_distributed`, max-over-ranks time).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1 (torchrun): every rank runs the config on its own GPU ("replicas";
DESIGN.md §Multi-GPU), value = total applies / max-over-ranks time.
--impl reference: the CPU oracle (oracle/, the tier's reference arm) on the host
cores, same config and metric, on a bounded sample of rows per step.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(surface="sphere", R=1.0, h=1.0 / 200, c=10.0, applies=100, l=6, m=3, restart=50,
           rtol=1e-10)
WORKLOAD = ("BASELINE configs[1]: unit sphere h=1/200, fp64, 100 applies on U[-1,1] seed 0 "
            "+ Y_6^3 solve c=10 GMRES(50) rtol 1e-10, 1 GPU")
METRIC = "CPM apply band-nodes/s"
UNIT = "band-nodes/s"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.t is not None:
            self.t.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for nm, v in zip(names, r[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


KERNELS = ["extend", "laplace", "mdot", "cgs_update", "cgs_final", "axpy", "other"]


def _traffic():
    """ncu DRAM bytes (read + write) per apply, from the committed capture summary."""
    p = os.path.join(ROOT, "profiles", "r01_traffic.json")
    try:
        d = json.load(open(p))
        return float(d["apply_dram_bytes"])
    except Exception:
        return None


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_oracle_rate(n_rows: int, seed: int = 0):
    """Oracle (oracle.operator.apply_rows, as it stands) on n_rows sampled band rows of config 1.
    Returns (rows/s, seconds, threads)."""
    from oracle.band import lam_of
    from oracle.operator import apply_rows
    from oracle.surfaces import Sphere
    import seeded_inputs

    h = CFG["h"]

    class _B:
        pass

    _B.h = h
    _B.surface = Sphere(CFG["R"])
    # sample lattice nodes inside the lambda-tube by the oracle's own test
    rng = np.random.default_rng(seed)
    rows = []
    got = 0
    lam = lam_of(h)
    while got < n_rows:
        d = rng.normal(size=(2 * n_rows, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        r = CFG["R"] + rng.uniform(-lam, lam, size=(2 * n_rows, 1))
        ijk = np.round(d * r / h).astype(np.int64)
        _, dist = _B.surface.cp(ijk.astype(np.float64) * h)
        ijk = ijk[dist <= lam]
        rows.append(ijk)
        got += len(ijk)
    ijk = np.concatenate(rows)[:n_rows]
    t0 = time.perf_counter()
    for s in range(0, n_rows, 8192):
        apply_rows(_B, CFG["c"], lambda q: seeded_inputs.uniform_pm1(0, q), ijk[s:s + 8192])
    dt = time.perf_counter() - t0
    return n_rows / dt, dt, 1


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    rows = args.ref_rows
    for _ in range(args.warmup):
        cpu_oracle_rate(max(rows // 8, 1024))
    rates, secs = [], []
    for k in range(args.steps):
        r, dt, thr = cpu_oracle_rate(rows, seed=k)
        rates.append(r)
        secs.append(dt)
    value = float(np.mean(rates))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(secs)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded U[-1,1] per lattice node)",
        "config": {"workload": WORKLOAD, "sample": f"{rows} oracle rows per step"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{rows} sampled active rows of config 1 per step, "
                                   "oracle.operator.apply_rows (numpy, 1 thread)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_mine(args):
    import torch

    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2110_06322_b200._build import build

    if rank == 0:
        build()
    if ws > 1:
        torch.distributed.barrier()
    import paper_2110_06322_b200 as cpm
    import seeded_inputs

    stream = torch.cuda.current_stream(dev)
    t0 = time.perf_counter()
    band = cpm.cpm_build_band(CFG["surface"], CFG["h"], R=CFG["R"])
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    nA, nG = band.info.n_active, band.info.n_ghost
    nE = nA + nG
    coords = cpm.cpm_band_active_coords(band).astype(np.int64)
    u_host = torch.from_numpy(seeded_inputs.uniform_pm1(0, coords)).pin_memory()
    u = u_host.to(dev, non_blocking=False)
    y = torch.empty_like(u)
    f = torch.empty_like(u)
    cpm.cpm_eval_sph(band, CFG["l"], CFG["m"], CFG["c"] + CFG["l"] * (CFG["l"] + 1), f)
    x = torch.zeros_like(u)
    c = CFG["c"]

    prof = {"apply": {}, "solve": {}}

    def take_profile(phase):
        for k in KERNELS:
            ms, n = cpm.cpm_profile_read(k)
            a, b = prof[phase].get(k, (0.0, 0))
            prof[phase][k] = (a + ms, b + n)
        cpm.cpm_profile_reset()

    def step(record, profile=False):
        evs = []
        if profile:
            cpm.cpm_profile_reset()
            cpm.cpm_profile_enable(True)
        for _ in range(CFG["applies"]):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            cpm.cpm_apply(band, c, u, y)
            b.record(stream)
            evs.append((a, b))
        if profile:
            take_profile("apply")
        x.zero_()
        sa = torch.cuda.Event(enable_timing=True)
        sb = torch.cuda.Event(enable_timing=True)
        sa.record(stream)
        st = cpm.cpm_solve(band, c, f, x, rtol=CFG["rtol"], restart=CFG["restart"])
        sb.record(stream)
        if profile:
            take_profile("solve")
            cpm.cpm_profile_enable(False)
        if record is not None:
            record.append((evs, (sa, sb), st))

    for _ in range(args.warmup):
        step(None)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    launches0 = cpm.cpm_kernel_launches()
    rec = []
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ga = torch.cuda.Event(enable_timing=True)
    gb = torch.cuda.Event(enable_timing=True)
    ga.record(stream)
    for _ in range(args.steps):
        step(rec)
    gb.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    launches = cpm.cpm_kernel_launches() - launches0
    clk = clocks.stop()
    # one more (untimed) step with per-kernel CUDA events: the kernel breakdown and
    # the per-launch times of the roofline (the timed steps run without them)
    step(None, profile=True)
    torch.cuda.synchronize()
    total_ms = ga.elapsed_time(gb)
    apply_ms = sum(a.elapsed_time(b) for evs, _, _ in rec for a, b in evs)
    solve_ms = [sa.elapsed_time(sb) for _, (sa, sb), _ in rec]
    stats = [st for _, _, st in rec]
    ext_ms, ext_n = prof["apply"]["extend"]
    lap_ms, lap_n = prof["apply"]["laplace"]

    # config 4 (Schnakenberg IMEX Euler on the torus, h = 1/400), a bounded number of steps
    rd = None
    if args.rd_steps > 0 and rank == 0:
        try:
            tb = cpm.cpm_build_band("torus", 1.0 / 400, R=1.0, r=0.4)
            tg = cpm.cpm_band_active_coords(tb).astype(np.int64)
            ru = torch.from_numpy(1.0 + 1e-2 * seeded_inputs.uniform_pm1(3, tg, stream=0)).to(dev)
            rv = torch.from_numpy(0.9 / 1.0 + 1e-2 * seeded_inputs.uniform_pm1(3, tg, stream=1)).to(dev)
            cpm.cpm_rd_step(tb, ru, rv)                     # warm-up (workspace allocation)
            its = []
            ra = torch.cuda.Event(enable_timing=True)
            rb = torch.cuda.Event(enable_timing=True)
            ra.record(stream)
            for _ in range(args.rd_steps):
                s1, s2 = cpm.cpm_rd_step(tb, ru, rv)
                its.append(s1.iterations + s2.iterations)
            rb.record(stream)
            torch.cuda.synchronize()
            rd = {"workload": "BASELINE configs[4]: Schnakenberg on torus R=1 r=0.4, h=1/400, IMEX Euler "
                              "dt=1e-3 (two GMRES(50) shifted solves per step), 1 GPU",
                  "n_active": tb.n, "steps_timed": args.rd_steps,
                  "ms_per_step": ra.elapsed_time(rb) / args.rd_steps,
                  "gmres_its_per_step": float(np.mean(its))}
            del tb, ru, rv
        except Exception as e:  # report, never fail the main metric
            rd = {"error": str(e)[:200]}

    # config 2 (torus h = 1/400, RAS-FGMRES(50), 8 subdomains, overlap 4h): one solve, 1 GPU
    c2 = None
    if args.c2_kinner > 0 and rank == 0:
        try:
            cb = cpm.cpm_build_band("torus", 1.0 / 400, R=1.0, r=0.4)
            cf = torch.empty(cb.n, dtype=torch.float64, device=dev)
            cpm.cpm_eval_torus_rhs(cb, seeded_inputs.smooth_modulation_coeffs(1), cf)
            cras = cpm.cpm_ras_setup(cb, 8, 4, args.c2_kinner, 1.0)
            cu = torch.zeros_like(cf)
            ca = torch.cuda.Event(enable_timing=True)
            cbv = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            ca.record(stream)
            cst = cpm.cpm_solve(cb, 1.0, cf, cu, rtol=1e-10, restart=50, ras=cras)
            cbv.record(stream)
            torch.cuda.synchronize()
            c2 = {"workload": "BASELINE configs[2]: torus R=1 r=0.4, h=1/400, c=1, f=cos(3theta)sin(2phi)"
                              "(1 + seed-1 smooth modulation); RAS-FGMRES(50), 8 Morton-slab subdomains, "
                              f"overlap 4h, {args.c2_kinner} inner GMRES steps, rtol 1e-10, 1 GPU",
                  "n_active": cb.n, "solve_s": ca.elapsed_time(cbv) / 1e3, "iterations": cst.iterations,
                  "converged": bool(cst.converged), "resid_true_rel": cst.resid_true / cst.bnorm}
            del cras, cb, cf, cu
        except Exception as e:  # report, never fail the main metric
            c2 = {"error": str(e)[:200]}

    # N > 1: the same config-2 solve partitioned over the ranks (Morton slabs, NCCL
    # halo exchange + allreduce, distributed RAS with n_sub = 8 a multiple of N)
    c2d = None
    if args.c2_dist and args.c2_kinner > 0 and 8 % ws == 0 and "RANK" in os.environ:
        try:
            from paper_2110_06322_b200.distributed import DistributedCPM

            if not torch.distributed.is_initialized():  # torchrun with one rank
                torch.distributed.init_process_group("nccl")

            cb = cpm.cpm_build_band("torus", 1.0 / 400, R=1.0, r=0.4)
            cf = torch.empty(cb.n, dtype=torch.float64, device=dev)
            cpm.cpm_eval_torus_rhs(cb, seeded_inputs.smooth_modulation_coeffs(1), cf)
            D = DistributedCPM(cb)
            dras = D.setup_ras(8, 4, args.c2_kinner, 1.0)
            fo = cf[D.lo:D.hi].contiguous()
            uo = torch.zeros_like(fo)
            torch.distributed.barrier()
            torch.cuda.synchronize()
            ea = torch.cuda.Event(enable_timing=True)
            eb = torch.cuda.Event(enable_timing=True)
            ea.record(stream)
            dst = D.solve(1.0, fo, uo, rtol=1e-10, restart=50, ras=dras)
            eb.record(stream)
            torch.cuda.synchronize()
            tt = torch.tensor([ea.elapsed_time(eb) / 1e3], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            c2d = {"workload": "BASELINE configs[2] partitioned over the ranks (Morton slabs, NCCL), "
                               f"RAS-FGMRES(50), 8 subdomains, overlap 4h, {args.c2_kinner} inner steps",
                   "ranks": ws, "solve_s_max_over_ranks": float(tt.item()), "iterations": dst.iterations,
                   "converged": bool(dst.converged), "resid_true_rel": dst.resid_true / dst.bnorm}
            del dras, D, cb, cf, fo, uo
        except Exception as e:  # report, never fail the main metric
            c2d = {"error": str(e)[:200]}

    # e2e: same metric through the C ABI with HOST buffers (pinned), copies inside the timed region
    y_host = torch.empty(nA, dtype=torch.float64).pin_memory()
    u_np, y_np = u_host.numpy(), y_host.numpy()
    e2e_steps = max(1, min(args.steps, 2))
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    t_e = time.perf_counter()
    for _ in range(e2e_steps):
        for _ in range(CFG["applies"]):
            cpm.cpm_apply(band, c, u_np, y_np)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t_e

    # reductions over ranks (max time)
    vals = torch.tensor([apply_ms, total_ms, e2e_s, float(np.median(solve_ms))], dtype=torch.float64, device=dev)
    if ws > 1:
        torch.distributed.all_reduce(vals, op=torch.distributed.ReduceOp.MAX)
    apply_ms, total_ms, e2e_s, solve_med_ms = [float(v) for v in vals.cpu()]
    n_applies = CFG["applies"] * args.steps
    value = ws * nA * n_applies / (apply_ms / 1e3)
    e2e_value = ws * nA * CFG["applies"] * e2e_steps / e2e_s

    peak, peak_src = _peaks()
    alg_bytes = 16 * nA + 28 * nE          # u + y + (t_xyz + eoff) per eval node
    # per apply (2 launches) over the timed region, CUDA events on the launching stream
    mean_apply_s = apply_ms / 1e3 / (CFG["applies"] * args.steps)
    achieved = alg_bytes / mean_apply_s / 1e9
    traffic = _traffic()
    # Krylov passes of the solve (delayed CGS2): per Arnoldi step j one reduction
    # pass (reads V_0..V_j and z: (j + 2) * 8 n bytes) and one update pass (reads the
    # same, writes q_j and u_{j+1}: (j + 4) * 8 n bytes); steps j = 0 .. per cycle
    st_last = stats[-1]
    kry_bytes = 0
    left, m = st_last.iterations, CFG["restart"]
    while left > 0:
        steps = min(left, m)
        for j in range(steps + 1):          # + the final reduction of the cycle
            kry_bytes += 8 * nA * ((j + 2) + ((j + 4) if j < steps else 0))
        left -= steps
    kry_ms = sum(prof["solve"][k][0] for k in ("mdot", "cgs_update", "cgs_final"))
    kry_gbs = kry_bytes / (kry_ms / 1e3) / 1e9 if kry_ms > 0 else None
    if rank == 0:
        cpu_rate, cpu_s, cores = (None, None, None)
        if not args.no_cpu and ws == 1:
            cpu_rate, cpu_s, cores = cpu_oracle_rate(args.cpu_rows)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded U[-1,1] per lattice node; manufactured Y_6^3 rhs)",
            "config": {"workload": WORKLOAD, "n_active": nA, "n_ghost": nG, "n_tiles": band.info.n_tiles,
                       "applies_per_step": CFG["applies"], "parallelism": f"replicas x{ws}",
                       "l2": f"inputs larger than L2: apply working set "
                             f"{(alg_bytes + band.info.n_tiles * 4096) / 1e6:.0f} MB vs 126 MB L2"},
            "solve": {"seconds_median": solve_med_ms / 1e3, "iterations": stats[-1].iterations,
                      "converged": stats[-1].converged, "resid_true_rel": stats[-1].resid_true / stats[-1].bnorm},
            "build_band_s": build_s,
            "roofline": {"kernel": "apply = k_extend_nt + k_laplace (one apply, the metric's unit)",
                         "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "alg_bytes_per_apply": alg_bytes,
                         "apply_ms": mean_apply_s * 1e3,
                         "extend_ms": ext_ms / max(ext_n, 1), "laplace_ms": lap_ms / max(lap_n, 1),
                         "note": "extend is bound by its per-tile load chain overlapped with FP64 and "
                                 "shared-memory gathers (DESIGN.md §Kernels, ablations); "
                                 "traffic = ncu DRAM bytes per apply (profiles/r01_traffic.json)"},
            "roofline_solve": {"kernel": "Krylov passes of the solve (k_dcgs_dots + k_dcgs_update), "
                                         "the largest share of a step",
                               "bound": "hbm", "achieved": kry_gbs, "peak": peak, "unit": "GB/s",
                               "frac": (kry_gbs / peak) if kry_gbs else None,
                               "alg_bytes_per_solve": kry_bytes, "ms_per_solve": kry_ms},
            "kernels_ms_per_step": {ph: {k: v[0] for k, v in d.items() if v[1]}
                                    for ph, d in prof.items()},
            "cpu_baseline": ({"value": cpu_rate, "unit": UNIT, "cores": cores, "kind": "oracle",
                              "sample": f"{args.cpu_rows} sampled active rows of config 1, "
                                        f"oracle.operator.apply_rows, {cpu_s:.1f} s"}
                             if cpu_rate else None),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * nA * CFG["applies"],
                    "d2h_bytes_per_step": 8 * nA * CFG["applies"]},
            "config4_rd": rd,
            "config2_solve": c2,
            "config2_solve_distributed": c2d,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--cpu-rows", type=int, default=1 << 18)
    ap.add_argument("--ref-rows", type=int, default=1 << 16)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--rd-steps", type=int, default=20, help="config-4 IMEX steps timed (0: skip)")
    ap.add_argument("--c2-kinner", type=int, default=16,
                    help="inner GMRES steps of the config-2 RAS solve (0: skip that solve)")
    ap.add_argument("--c2-dist", action="store_true",
                    help="under torchrun (N | 8): also time the config-2 solve partitioned over "
                         "the ranks (NCCL); opt-in, run here with one rank only")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_mine(args)


if __name__ == "__main__":
    sys.exit(main())
