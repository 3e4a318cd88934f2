#!/usr/bin/env python
"""bench.py — CPM hot path on B200 (BASELINE.json metric, config 1).

A step is one pass of the hot path over config 1 (BASELINE.json configs[1]):
unit sphere, h = 1/200 (~4.1M band nodes), fp64:
  * 100 operator applies y = (c - Delta_S^h) u on u ~ U[-1,1] (seed 0), c = 10
  * the manufactured solve (c - Delta_S^h) u = (c + 42) Y_6^3(cp), GMRES(50), rtol 1e-10
`value` = band-node applies per second over the timed applies (CUDA events on the
launching stream, max over ranks); `solve` reports the GMRES solve time.  The
band is built once, outside the timed region (its build time is reported).
Outside the timed steps rank 0 also reports `config4_rd` (config-4 IMEX steps)
and `config2_solve` (one config-2 RAS-FGMRES solve, ~40 s; --c2-kinner 0 skips it);
--c3 adds the config-3 solve (sphere h = 1/800, c = 0.1, RAS k_inner 64, overlap
16; ~40 min on one GPU).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1: STRONG scaling of the partitioned path: without
torchrun, bench.py re-launches itself under `torch.distributed.run` with N ranks;
every rank owns a Morton slab of the SAME config-1 band, `value` = global band
nodes x applies / max-over-ranks time of cpm_part_apply (NCCL halo exchange inside
the timed region), `solve` = the partitioned GMRES(50) solve (NCCL allreduces),
and (N | 8) the partitioned config-2 RAS-FGMRES solve and config-4 IMEX steps.
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
    p = os.path.join(ROOT, "profiles", "r02_traffic_v3.json")
    try:
        d = json.load(open(p))
        return float(d["apply_dram_bytes"])
    except Exception:
        return None


def _l1tex_events():
    """l1tex data-stage events (shared wavefronts + global tag requests) of one config-1
    extend launch, from the committed ncu capture (profiles/r02_ncu_v3.txt)."""
    p = os.path.join(ROOT, "profiles", "r02_l1tex_events.json")
    try:
        d = json.load(open(p))
        return float(d["shared_wavefronts"]) + float(d["global_tag_requests"])
    except Exception:
        return None


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _oracle_rows(n_rows: int, seed: int):
    """n_rows lattice nodes of config 1's lambda-tube, sampled by the oracle's own test."""
    from oracle.band import lam_of
    from oracle.surfaces import Sphere

    h = CFG["h"]
    sph = Sphere(CFG["R"])
    rng = np.random.default_rng(seed)
    rows = []
    got = 0
    lam = lam_of(h)
    while got < n_rows:
        d = rng.normal(size=(2 * n_rows, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        r = CFG["R"] + rng.uniform(-lam, lam, size=(2 * n_rows, 1))
        ijk = np.round(d * r / h).astype(np.int64)
        _, dist = sph.cp(ijk.astype(np.float64) * h)
        ijk = ijk[dist <= lam]
        rows.append(ijk)
        got += len(ijk)
    return np.concatenate(rows)[:n_rows]


def _oracle_chunk(ijk):
    """oracle.operator.apply_rows on one chunk of rows (a pool worker, one thread)."""
    from oracle.operator import apply_rows
    from oracle.surfaces import Sphere
    import seeded_inputs

    class _B:
        pass

    _B.h = CFG["h"]
    _B.surface = Sphere(CFG["R"])
    apply_rows(_B, CFG["c"], lambda q: seeded_inputs.uniform_pm1(0, q), ijk)
    return len(ijk)


def _pool_init():
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"


def cpu_oracle_rate(n_rows: int, seed: int = 0, cores: int | None = None):
    """Oracle (oracle.operator.apply_rows, as it stands) on n_rows sampled band rows of
    config 1, spread over `cores` worker processes (default: every host core), one
    numpy thread each.  Returns (rows/s, seconds, cores)."""
    import multiprocessing as mproc

    cores = cores or os.cpu_count() or 1
    ijk = _oracle_rows(n_rows, seed)
    chunks = [ijk[s:s + 4096] for s in range(0, n_rows, 4096)]
    ctx = mproc.get_context("fork")
    with ctx.Pool(cores, initializer=_pool_init) as pool:
        pool.map(_oracle_chunk, chunks[:cores])           # warm the workers (imports)
        t0 = time.perf_counter()
        done = sum(pool.map(_oracle_chunk, chunks, chunksize=1))
        dt = time.perf_counter() - t0
    return done / dt, dt, cores


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    rows = args.ref_rows
    for _ in range(args.warmup):
        cpu_oracle_rate(max(rows // 8, 1024))
    rates, secs = [], []
    thr = 1
    for k in range(args.steps):
        r, dt, thr = cpu_oracle_rate(rows, seed=k)
        rates.append(r)
        secs.append(dt)
    value = float(np.mean(rates))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(secs)),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded U[-1,1] per lattice node)",
        "config": {"workload": WORKLOAD, "sample": f"{rows} oracle rows per step"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": thr, "kind": "oracle",
                         "sample": f"{rows} sampled active rows of config 1 per step, "
                                   f"oracle.operator.apply_rows (numpy, {thr} worker processes x 1 thread)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_mine(args):
    import torch

    ws, rank, local = 1, 0, int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2110_06322_b200._build import build

    build()
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
    torch.cuda.synchronize()
    ga = torch.cuda.Event(enable_timing=True)
    gb = torch.cuda.Event(enable_timing=True)
    ga.record(stream)
    for _ in range(args.steps):
        step(rec)
    gb.record(stream)
    torch.cuda.synchronize()
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

    # config 3 (sphere h = 1/800, 66M unknowns, c = 0.1): RAS-FGMRES(50), 8 subdomains,
    # k_inner 64, overlap 16 (the setting that converges), --c3 only
    c3 = None
    if args.c3:
        try:
            b3 = cpm.cpm_build_band("sphere", 1.0 / 800)
            g3 = cpm.cpm_band_active_coords(b3).astype(np.int64)
            f3 = torch.empty(b3.n, dtype=torch.float64, device=dev)
            cpm.cpm_eval_sph(b3, 10, 5, 1.0, f3)
            f3 += torch.from_numpy(1e-3 * seeded_inputs.normal(2, g3)).to(dev)
            del g3
            r3 = cpm.cpm_ras_setup(b3, 8, 16, 64, 0.1)
            u3 = torch.zeros_like(f3)
            a3 = torch.cuda.Event(enable_timing=True)
            e3 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a3.record(stream)
            s3 = cpm.cpm_solve(b3, 0.1, f3, u3, rtol=1e-10, restart=50, ras=r3)
            e3.record(stream)
            torch.cuda.synchronize()
            c3 = {"workload": "BASELINE configs[3]: unit sphere h=1/800, c=0.1, f=Y_10^5 + 1e-3 N(0,1) seed 2; "
                              "RAS-FGMRES(50), 8 Morton-slab subdomains, overlap 16, 64 inner GMRES steps, "
                              "rtol 1e-10, 1 GPU",
                  "n_active": b3.n, "solve_s": a3.elapsed_time(e3) / 1e3, "iterations": s3.iterations,
                  "converged": bool(s3.converged), "resid_true_rel": s3.resid_true / s3.bnorm}
            del r3, b3, f3, u3
        except Exception as e:  # report, never fail the main metric
            c3 = {"error": str(e)[:200]}

    # e2e: same metric through the C ABI with HOST buffers (pinned), copies inside the
    # timed region: cpm_apply_async pipelines consecutive applies (the copy of the next
    # u overlaps this apply and the copy-out of y), cpm_apply_sync before the clock stops
    y_host = torch.empty(nA, dtype=torch.float64).pin_memory()
    u_np, y_np = u_host.numpy(), y_host.numpy()
    e2e_steps = max(1, min(args.steps, 2))
    cpm.cpm_apply_async(band, c, u_np, y_np)          # staging allocation, outside the clock
    cpm.cpm_apply_sync(band)
    torch.cuda.synchronize()
    t_e = time.perf_counter()
    for _ in range(e2e_steps):
        for _ in range(CFG["applies"]):
            cpm.cpm_apply_async(band, c, u_np, y_np)
    cpm.cpm_apply_sync(band)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t_e
    e2e_sync_s = None
    if args.steps > 0:  # the synchronous host-pointer cpm_apply, for comparison (not the e2e value)
        t_e = time.perf_counter()
        for _ in range(CFG["applies"]):
            cpm.cpm_apply(band, c, u_np, y_np)
        torch.cuda.synchronize()
        e2e_sync_s = time.perf_counter() - t_e

    # the e2e roof: the same bytes per apply (u in, y out) copied with nothing else,
    # H2D and D2H concurrently on two streams (the host link's rate for this traffic)
    link_value = None
    try:
        d_in = torch.empty(nA, dtype=torch.float64, device=dev)
        d_out = torch.empty(nA, dtype=torch.float64, device=dev)
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        reps = 20
        for _ in range(2):
            torch.cuda.synchronize()
            t_l = time.perf_counter()
            for _ in range(reps):
                with torch.cuda.stream(s_in):
                    d_in.copy_(u_host, non_blocking=True)
                with torch.cuda.stream(s_out):
                    y_host.copy_(d_out, non_blocking=True)
            torch.cuda.synchronize()
            link_value = nA * reps / (time.perf_counter() - t_l)
        del d_in, d_out
    except Exception:
        link_value = None

    solve_med_ms = float(np.median(solve_ms))
    n_applies = CFG["applies"] * args.steps
    value = nA * n_applies / (apply_ms / 1e3)
    e2e_value = nA * CFG["applies"] * e2e_steps / e2e_s

    peak, peak_src = _peaks()
    alg_bytes = 16 * nA + 28 * nE          # u + y + (t_xyz + eoff) per eval node
    # per apply (2 launches) over the timed region, CUDA events on the launching stream
    mean_apply_s = apply_ms / 1e3 / (CFG["applies"] * args.steps)
    achieved = alg_bytes / mean_apply_s / 1e9
    traffic = _traffic()
    # what limits the extend (not HBM): its l1tex data stage, one shared wavefront or one
    # global tag request per clock per SM; events from the ncu capture, the clock and the
    # time measured in this run
    l1ev = _l1tex_events()
    ext_s = ext_ms / max(ext_n, 1) / 1e3
    sm_hz = (clk.get("sm_mhz") or 0.0) * 1e6
    limiter = None
    if l1ev and ext_s > 0 and sm_hz > 0:
        per_clk = l1ev / (ext_s * 148 * sm_hz)
        limiter = {"kernel": "k_extend_nt", "bound": "l1tex data stage (shared-memory wavefronts + global tag "
                   "requests)", "events_per_launch": l1ev, "achieved": per_clk, "peak": 1.0,
                   "unit": "events/clk/SM", "frac": per_clk, "sm_mhz": clk.get("sm_mhz"),
                   "source": "profiles/r02_l1tex_events.json (ncu), time and clock of this run"}
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
        if not args.no_cpu:
            cpu_rate, cpu_s, cores = cpu_oracle_rate(args.cpu_rows)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded U[-1,1] per lattice node; manufactured Y_6^3 rhs)",
            "config": {"workload": WORKLOAD, "n_active": nA, "n_ghost": nG, "n_tiles": band.info.n_tiles,
                       "applies_per_step": CFG["applies"], "parallelism": "single GPU (N = 1 of the strong-scaling series)",
                       "l2": f"inputs larger than L2: apply working set "
                             f"{(alg_bytes + band.info.n_tiles * 4096) / 1e6:.0f} MB vs 126 MB L2"},
            "solve": {"seconds_median": solve_med_ms / 1e3, "iterations": stats[-1].iterations,
                      "converged": stats[-1].converged, "resid_true_rel": stats[-1].resid_true / stats[-1].bnorm},
            "build_band_s": build_s,
            "roofline": {"kernel": "apply = k_extend_nt + k_laplace_tma (one apply, the metric's unit)",
                         "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "frac_of_nominal_8tbs": achieved / 8000.0,   # north_star's denominator
                         "limiter": limiter,
                         "alg_bytes_per_apply": alg_bytes,
                         "apply_ms": mean_apply_s * 1e3,
                         "extend_ms": ext_ms / max(ext_n, 1), "laplace_ms": lap_ms / max(lap_n, 1),
                         "note": "the extend is bound by its l1tex data path (64 shared-memory gathers per node "
                                 "slot, the cp.async box fill, scattered E u stores: DESIGN.md §Kernels, "
                                 "profiles/r02_ncu_v3.txt); traffic = ncu DRAM bytes per apply "
                                 "(profiles/r02_traffic_v3.json)"},
            "roofline_solve": {"kernel": "Krylov passes of the solve (k_dcgs_dots + k_dcgs_update), "
                                         "the largest share of a step",
                               "bound": "hbm", "achieved": kry_gbs, "peak": peak, "unit": "GB/s",
                               "frac": (kry_gbs / peak) if kry_gbs else None,
                               "alg_bytes_per_solve": kry_bytes, "ms_per_solve": kry_ms},
            "kernels_ms_per_step": {ph: {k: v[0] for k, v in d.items() if v[1]}
                                    for ph, d in prof.items()},
            "cpu_baseline": ({"value": cpu_rate, "unit": UNIT, "cores": cores, "kind": "oracle",
                              "sample": f"{args.cpu_rows} sampled active rows of config 1, "
                                        f"oracle.operator.apply_rows on {cores} worker processes "
                                        f"(1 thread each), {cpu_s:.1f} s"}
                             if cpu_rate else None),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * nA * CFG["applies"],
                    "d2h_bytes_per_step": 8 * nA * CFG["applies"],
                    "api": "cpm_apply_async on pinned host buffers (+ cpm_apply_sync), 100 applies per step",
                    "sync_cpm_apply_value": (nA * CFG["applies"] / e2e_sync_s) if e2e_sync_s else None,
                    "link_bound_value": link_value,
                    "link_frac": (e2e_value / link_value) if link_value else None,
                    "link_note": "link_bound_value: the same 8 B in + 8 B out per active node copied alone "
                                 "(pinned, H2D and D2H concurrent on two streams), the host link's roof "
                                 "for e2e"},
            "config4_rd": rd,
            "config2_solve": c2,
            "config3_solve": c3,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    return 0


def run_partitioned(args):
    """N > 1 ranks (torchrun): strong scaling of the partitioned path on the same
    global config-1 band."""
    import torch
    import torch.distributed as dist

    # CPM_TRANSPORT=host: the host-staged transport over gloo, so that N ranks can share
    # one GPU (checks this code path on a one-GPU box; the timing is then not a scaling
    # number).  Default: NCCL, one GPU per rank.
    host = os.environ.get("CPM_TRANSPORT", "nccl") == "host"
    ws, rank, local = _dist()
    if not host:
        os.environ.setdefault("NCCL_DEBUG", "INFO")      # the driver reads the communicator size
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    local = local % max(torch.cuda.device_count(), 1) if host else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if host:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    rdev = torch.device("cpu") if host else dev          # device of the bench's own reductions
    transport = "host" if host else "nccl"
    from paper_2110_06322_b200._build import build

    if rank == 0:
        build()
    dist.barrier()
    import paper_2110_06322_b200 as cpm
    import seeded_inputs
    from paper_2110_06322_b200.distributed import DistributedCPM

    stream = torch.cuda.current_stream(dev)

    def max_over_ranks(vals):
        t = torch.tensor(vals, dtype=torch.float64, device=rdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(v) for v in t.cpu()]

    def sum_over_ranks(vals):
        t = torch.tensor(vals, dtype=torch.float64, device=rdev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return [float(v) for v in t.cpu()]

    t0 = time.perf_counter()
    band = cpm.cpm_build_band(CFG["surface"], CFG["h"], R=CFG["R"])
    D = DistributedCPM(band, transport=transport)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    nA, nG = band.info.n_active, band.info.n_ghost
    lo, hi = D.lo, D.hi
    coords = cpm.cpm_band_active_coords(band).astype(np.int64)
    u_host = torch.from_numpy(seeded_inputs.uniform_pm1(0, coords[lo:hi])).pin_memory()
    u = u_host.to(dev)
    y = torch.empty_like(u)
    fg = torch.empty(nA, dtype=torch.float64, device=dev)
    cpm.cpm_eval_sph(band, CFG["l"], CFG["m"], CFG["c"] + CFG["l"] * (CFG["l"] + 1), fg)
    f = fg[lo:hi].contiguous()
    del fg
    x = torch.zeros_like(u)
    c = CFG["c"]
    pinfo = D.part

    def step(record, profile=False):
        evs = []
        if profile:
            cpm.cpm_profile_reset()
            cpm.cpm_profile_enable(True)
        for _ in range(CFG["applies"]):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            D.apply(c, u, y)
            b.record(stream)
            evs.append((a, b))
        prof = None
        if profile:
            prof = {k: cpm.cpm_profile_read(k) for k in KERNELS}
            cpm.cpm_profile_reset()
        x.zero_()
        sa = torch.cuda.Event(enable_timing=True)
        sb = torch.cuda.Event(enable_timing=True)
        sa.record(stream)
        st = D.solve(c, f, x, rtol=CFG["rtol"], restart=CFG["restart"])
        sb.record(stream)
        if profile:
            cpm.cpm_profile_enable(False)
        if record is not None:
            record.append((evs, (sa, sb), st))
        return prof

    for _ in range(args.warmup):
        step(None)
    torch.cuda.synchronize()
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
    launches0 = cpm.cpm_kernel_launches()
    rec = []
    dist.barrier()
    torch.cuda.synchronize()
    ga = torch.cuda.Event(enable_timing=True)
    gb = torch.cuda.Event(enable_timing=True)
    ga.record(stream)
    for _ in range(args.steps):
        step(rec)
    gb.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    launches = cpm.cpm_kernel_launches() - launches0
    clk = clocks.stop() if clocks else None
    prof = step(None, profile=True)
    torch.cuda.synchronize()
    total_ms = ga.elapsed_time(gb)
    apply_ms = sum(a.elapsed_time(b) for evs, _, _ in rec for a, b in evs)
    solve_ms = float(np.median([sa.elapsed_time(sb) for _, (sa, sb), _ in rec]))
    st = rec[-1][2]

    # e2e through the public API with host buffers: each rank copies its owned slice
    # of u in (pinned), applies (halo exchange inside), copies its slice of y out
    y_host = torch.empty(hi - lo, dtype=torch.float64).pin_memory()
    e2e_steps = max(1, min(args.steps, 2))
    dist.barrier()
    torch.cuda.synchronize()
    ea = torch.cuda.Event(enable_timing=True)
    eb = torch.cuda.Event(enable_timing=True)
    ea.record(stream)
    for _ in range(e2e_steps):
        for _ in range(CFG["applies"]):
            u.copy_(u_host, non_blocking=True)
            D.apply(c, u, y)
            y_host.copy_(y, non_blocking=True)
    eb.record(stream)
    torch.cuda.synchronize()
    e2e_ms = ea.elapsed_time(eb)

    # config 2 (torus h = 1/400) partitioned RAS-FGMRES(50), 8 subdomains (N | 8), and
    # config 4 (Schnakenberg IMEX on the same torus band) partitioned steps
    c2 = rd = None
    if 8 % ws == 0 and (args.c2_kinner > 0 or args.rd_steps > 0):
        try:
            tb = cpm.cpm_build_band("torus", 1.0 / 400, R=1.0, r=0.4)
            DT = DistributedCPM(tb, transport=transport)
            tlo, thi = DT.lo, DT.hi
            if args.c2_kinner > 0:
                cf = torch.empty(tb.n, dtype=torch.float64, device=dev)
                cpm.cpm_eval_torus_rhs(tb, seeded_inputs.smooth_modulation_coeffs(1), cf)
                fo = cf[tlo:thi].contiguous()
                del cf
                ras = DT.setup_ras(8, 4, args.c2_kinner, 1.0)
                uo = torch.zeros_like(fo)
                dist.barrier()
                torch.cuda.synchronize()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                cst = DT.solve(1.0, fo, uo, rtol=1e-10, restart=50, ras=ras)
                b.record(stream)
                torch.cuda.synchronize()
                (sec,) = max_over_ranks([a.elapsed_time(b) / 1e3])
                rr = sum_over_ranks([cst.resid_true ** 2])
                c2 = {"workload": f"BASELINE configs[2] partitioned over the ranks (Morton slabs, {transport} halo "
                                  "exchange + allreduce, distributed RAS: 8 subdomains, overlap 4h, "
                                  f"{args.c2_kinner} inner GMRES steps), RAS-FGMRES(50), rtol 1e-10",
                      "ranks": ws, "n_active": tb.n, "solve_s": sec, "iterations": cst.iterations,
                      "converged": bool(cst.converged), "resid_true_rel": cst.resid_true / cst.bnorm}
                del ras, fo, uo
            if args.rd_steps > 0:
                tg = cpm.cpm_band_active_coords(tb).astype(np.int64)[tlo:thi]
                ru = torch.from_numpy(1.0 + 1e-2 * seeded_inputs.uniform_pm1(3, tg, stream=0)).to(dev)
                rv = torch.from_numpy(0.9 / 1.0 + 1e-2 * seeded_inputs.uniform_pm1(3, tg, stream=1)).to(dev)
                DT.rd_step(ru, rv)                         # warm-up (workspace allocation)
                its = []
                dist.barrier()
                torch.cuda.synchronize()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                for _ in range(args.rd_steps):
                    s1, s2 = DT.rd_step(ru, rv)
                    its.append(s1.iterations + s2.iterations)
                b.record(stream)
                torch.cuda.synchronize()
                (ms,) = max_over_ranks([a.elapsed_time(b) / args.rd_steps])
                rd = {"workload": "BASELINE configs[4]: Schnakenberg on torus R=1 r=0.4, h=1/400, IMEX Euler "
                                  f"dt=1e-3, partitioned over {ws} ranks (cpm_part_rd_step)",
                      "n_active": tb.n, "steps_timed": args.rd_steps, "ms_per_step": ms,
                      "gmres_its_per_step": float(np.mean(its))}
            del DT, tb
        except Exception as e:  # report, never fail the main metric
            c2 = c2 or {"error": str(e)[:200]}

    apply_ms, total_ms, solve_ms, e2e_ms = max_over_ranks([apply_ms, total_ms, solve_ms, e2e_ms])
    ext_ms, lap_ms, n_ext = max_over_ranks([prof["extend"][0], prof["laplace"][0], prof["extend"][1]])
    (launches_all,) = sum_over_ranks([float(launches)])
    nT_local = D.part.n_tiles
    n_applies = CFG["applies"] * args.steps
    value = nA * n_applies / (apply_ms / 1e3)
    e2e_value = nA * CFG["applies"] * e2e_steps / (e2e_ms / 1e3)
    peak, peak_src = _peaks()
    alg_bytes = 16 * nA + 28 * (nA + nG)       # whole band per apply (row (d))
    mean_apply_s = apply_ms / 1e3 / n_applies
    achieved_per_gpu = alg_bytes / ws / mean_apply_s / 1e9
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded U[-1,1] per lattice node; manufactured Y_6^3 rhs)",
            "config": {"workload": WORKLOAD.replace(", 1 GPU", f", partitioned over {ws} GPUs"),
                       "n_active": nA, "n_ghost": nG, "applies_per_step": CFG["applies"],
                       "parallelism": f"Morton-slab partition x{ws} "
                                      + ("(host-staged gloo transport, ranks sharing a GPU: NOT a scaling number)"
                                         if host else "(NCCL halo send/recv + allreduce)"),
                       "rank0_owned": hi - lo, "rank0_halo": pinfo.n_halo, "rank0_tiles": nT_local,
                       "rank0_interior_tiles": pinfo.n_interior_tiles,
                       "l2": "inputs larger than L2 at N <= 4; the timed applies include the halo exchange"},
            "solve": {"seconds_median": solve_ms / 1e3, "iterations": st.iterations, "converged": st.converged,
                      "resid_true_rel": st.resid_true / st.bnorm,
                      "kind": f"partitioned GMRES(50) ({'host-transport' if host else 'NCCL'} allreduce)"},
            "setup_s": setup_s,
            "roofline": {"kernel": "apply = halo exchange + k_extend_nt + k_laplace_tma on each rank's sub-band",
                         "bound": "hbm", "achieved": achieved_per_gpu, "peak": peak, "unit": "GB/s",
                         "frac": achieved_per_gpu / peak, "traffic": None, "peak_source": peak_src,
                         "alg_bytes_per_apply_per_gpu": alg_bytes / ws, "apply_ms": mean_apply_s * 1e3,
                         "extend_ms_max_rank": ext_ms / max(n_ext, 1), "laplace_ms_max_rank": lap_ms / max(n_ext, 1)},
            "cpu_baseline": None,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * nA * CFG["applies"],
                    "d2h_bytes_per_step": 8 * nA * CFG["applies"]},
            "config2_solve": c2, "config4_rd": rd,
            "gpu_launches": int(launches_all),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def _self_launch(args) -> int:
    """--gpus N > 1 without torchrun: re-run this script under torch.distributed.run."""
    import socket

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--cpu-rows", type=int, default=1 << 20)
    ap.add_argument("--ref-rows", type=int, default=1 << 16)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--rd-steps", type=int, default=20, help="config-4 IMEX steps timed (0: skip)")
    ap.add_argument("--c2-kinner", type=int, default=16,
                    help="inner GMRES steps of the config-2 RAS solve (0: skip that solve)")
    ap.add_argument("--c3", action="store_true",
                    help="also run the config-3 solve (sphere h=1/800, c=0.1, RAS-FGMRES(50), k_inner 64, "
                         "overlap 16; ~40 min on one GPU)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return _self_launch(args)
    if ws > 1 or (os.environ.get("CPM_BENCH_PARTITIONED") == "1" and "WORLD_SIZE" in os.environ):
        return run_partitioned(args)  # (the env switch runs this path with one rank, as a check)
    return run_mine(args)


if __name__ == "__main__":
    sys.exit(main())
