"""Quick apply timing on config 1 (for iterating on kernels).

CPM_ORDERS="1 0" times the apply for each extend node order (CPM_ITEMS = 1: items,
k_extend_it; 0: pairs, k_extend_nt; band rebuilt per order) and prints the max
difference against the first (0 = bit-identical).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2110_06322_b200 as cpm
import seeded_inputs

h = float(os.environ.get("CPM_H", 1.0 / 200))
ks = [int(k) for k in os.environ.get("CPM_ORDERS", "1").split()]
ref = None
for K in ks:
    os.environ["CPM_ITEMS"] = str(K)
    band = cpm.cpm_build_band("sphere", h)
    coords = cpm.cpm_band_active_coords(band).astype(np.int64)
    u = torch.from_numpy(seeded_inputs.uniform_pm1(0, coords)).cuda()
    y = torch.empty_like(u)
    for _ in range(5):
        cpm.cpm_apply(band, 10.0, u, y)
    torch.cuda.synchronize()
    if ref is None:
        ref = y.clone()
    err = float((y - ref).abs().max() / ref.abs().max())
    cpm.cpm_profile_reset()
    cpm.cpm_profile_enable(True)
    N = 50
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(N):
        cpm.cpm_apply(band, 10.0, u, y)
    b.record()
    torch.cuda.synchronize()
    cpm.cpm_profile_enable(False)
    ms = a.elapsed_time(b) / N
    e, _ = cpm.cpm_profile_read("extend")
    l, _ = cpm.cpm_profile_read("laplace")
    nA, nG = band.info.n_active, band.info.n_ghost
    alg = 16 * nA + 28 * (nA + nG)
    print(f"{'FUSED ' if os.environ.get('CPM_FUSED') == '1' else ''}items={K} nA={nA} tiles={band.info.n_tiles} runs={band.info.n_runs} maxbox={band.info.max_box} "
          f"apply {ms*1e3:.1f} us (extend {e/N*1e3:.1f} us, laplace {l/N*1e3:.1f} us) -> "
          f"{alg/ms/1e6:.0f} GB/s alg, {nA/ms/1e6:.2f} Gnodes/s, diff vs first {err:.1e}", flush=True)
    del band
if os.environ.get("CPM_SOLVE"):
    band = cpm.cpm_build_band("sphere", h)
    f = torch.empty_like(u)
    cpm.cpm_eval_sph(band, 6, 3, 52.0, f)
    x = torch.zeros_like(u)
    cpm.cpm_profile_reset()
    cpm.cpm_profile_enable(True)
    st = cpm.cpm_solve(band, 10.0, f, x, rtol=1e-10, restart=50, maxit=200)
    cpm.cpm_profile_enable(False)
    out = {k: cpm.cpm_profile_read(k) for k in ["extend", "laplace", "mdot", "cgs_update", "cgs_final", "axpy", "other"]}
    print("solve 200 its:", f"{st.seconds:.3f}s", {k: f"{v[0]:.1f}ms/{v[1]}" for k, v in out.items()})
    for _ in range(2):
        x.zero_()
        st = cpm.cpm_solve(band, 10.0, f, x, rtol=1e-10, restart=50, maxit=200)
        print("solve 200 its, profiling off:", f"{st.seconds:.3f}s")
    x.zero_()
    st = cpm.cpm_solve(band, 10.0, f, x, rtol=1e-10, restart=50)
    print("full solve, profiling off:", f"{st.seconds:.3f}s", st.iterations, "its")
