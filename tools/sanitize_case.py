"""Small walk over every C-ABI entry point, for compute-sanitizer (tools/sanitize.sh):
band build (sphere, torus), apply (device, host, async), GMRES, RAS apply and
RAS-FGMRES, the IMEX step, the partitioned apply / RAS / solve of every rank of a
2-rank split (halo by indexing, as tests/test_gpu_partition.py).  Sizes are the
smallest that still span several tiles, ragged tails and both pair / single
warps; nothing is compared with the oracle here — the parity suite does that."""
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2110_06322_b200 as cpm  # noqa: E402
import seeded_inputs  # noqa: E402
from paper_2110_06322_b200 import cpm as C  # noqa: E402
from paper_2110_06322_b200.distributed import owners, request_counts, slab_bounds  # noqa: E402


def main():
    torch.cuda.set_device(0)
    for kind, h, kw in (("sphere", 0.125, {}), ("torus", 0.06, {"R": 1.0, "r": 0.4})):
        band = cpm.cpm_build_band(kind, h, **kw)
        n = band.n
        ga = cpm.cpm_band_active_coords(band).astype(np.int64)
        u_h = seeded_inputs.uniform_pm1(0, ga)
        u = torch.from_numpy(u_h).cuda()
        y = torch.empty_like(u)
        cpm.cpm_apply(band, 1.0, u, y)
        yh = np.empty(n)
        cpm.cpm_apply(band, 1.0, u_h, yh)                        # host pointers
        up = torch.from_numpy(u_h).pin_memory()
        yp = torch.empty(n, dtype=torch.float64).pin_memory()
        for _ in range(3):
            cpm.cpm_apply_async(band, 1.0, up, yp)
        cpm.cpm_apply_sync(band)
        torch.cuda.synchronize()
        assert np.array_equal(yh, y.cpu().numpy()) and np.array_equal(yp.numpy(), yh)

        f = torch.empty_like(u)
        if kind == "sphere":
            cpm.cpm_eval_sph(band, 3, 2, 13.0, f)
        else:
            f.copy_(y)
        x = torch.zeros_like(f)
        st = cpm.cpm_solve(band, 1.0, f, x, rtol=1e-8, restart=10)
        assert st.converged, st
        print(kind, "n", n, "gmres its", st.iterations, flush=True)

        ras = cpm.cpm_ras_setup(band, 4, 2, 6, 1.0)
        z = torch.empty_like(f)
        cpm.cpm_ras_apply(ras, f, z)
        x.zero_()
        st = cpm.cpm_solve(band, 1.0, f, x, rtol=1e-8, restart=20, ras=ras)
        assert st.converged, st
        print(kind, "ras-fgmres its", st.iterations, flush=True)

        v = torch.from_numpy(seeded_inputs.uniform_pm1(1, ga)).cuda()
        w = u.clone()
        cpm.cpm_rd_step(band, w, v, dt=1e-3, rtol=1e-8, restart=10)

        R = 2
        bounds = slab_bounds(n, R)
        parts = [C.cpm_part_create(band, r, R) for r in range(R)]
        halos = [C.cpm_part_halo_nodes(p) for p in parts]
        y_cat = torch.empty_like(u)
        for r, p in enumerate(parts):
            request_counts(halos[r], bounds)
            u_own = u[p.lo:p.hi].contiguous()
            u_halo = u[torch.from_numpy(halos[r]).cuda()].contiguous()
            y_own = torch.empty(p.n_owned, dtype=torch.float64, device="cuda")
            C.cpm_part_apply_local(p, 1.0, u_own, u_halo, y_own)
            y_cat[p.lo:p.hi] = y_own
            send = [halos[q][owners(halos[q], bounds) == r] for q in range(R)]
            C.cpm_part_set_send(p, np.concatenate(send), np.array([len(s) for s in send]))
            pr = C.cpm_part_ras_setup(p, 4, 2, 6, 1.0)
            rh = C.cpm_ras_halo_nodes(pr)
            z_own = torch.empty(p.n_owned, dtype=torch.float64, device="cuda")
            C.cpm_part_ras_apply_local(pr, f[p.lo:p.hi].contiguous(),
                                       f[torch.from_numpy(rh).cuda()].contiguous(), z_own)
        torch.cuda.synchronize()
        assert torch.equal(y_cat, y)
        p1 = C.cpm_part_create(band, 0, 1)
        x1 = torch.zeros_like(f)
        st = C.cpm_part_solve(p1, None, 1.0, f, x1, rtol=1e-8, restart=10)
        assert st.converged, st
        w1, v1 = u.clone(), v.clone()
        C.cpm_part_rd_step(p1, None, w1, v1, dt=1e-3, rtol=1e-8, restart=10)
        torch.cuda.synchronize()
        print(kind, "partition ok", flush=True)
    print("sanitize_case ok")


if __name__ == "__main__":
    main()
