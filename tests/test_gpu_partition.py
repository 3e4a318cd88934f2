"""Multi-GPU partition (north_star item 5) validated on ONE GPU: the R ranks'
local operators are built and applied in one process, the halo exchange is done
by plain indexing (what NCCL moves), and the concatenated owned outputs must be
bit-identical to the single-band apply.  No kernel waits on another rank."""
import numpy as np
import pytest

import seeded_inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cpm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2110_06322_b200._build import build

    build()
    import paper_2110_06322_b200 as p

    return p


@pytest.mark.parametrize("kind,h,R", [("sphere", 0.1, 2), ("sphere", 0.1, 8), ("torus", 0.05, 4),
                                      ("sphere", 1.0 / 64, 8)])
def test_partitioned_apply_bit_exact(cpm, kind, h, R):
    from paper_2110_06322_b200 import cpm as C
    from paper_2110_06322_b200.distributed import owners, request_counts, slab_bounds

    band = cpm.cpm_build_band(kind, h) if kind == "sphere" else cpm.cpm_build_band(kind, h, R=1.0, r=0.4)
    n = band.n
    ga = cpm.cpm_band_active_coords(band).astype(np.int64)
    u = torch.from_numpy(seeded_inputs.uniform_pm1(0, ga)).cuda()
    y = torch.empty_like(u)
    cpm.cpm_apply(band, 3.0, u, y)
    bounds = slab_bounds(n, R)
    parts = [C.cpm_part_create(band, r, R) for r in range(R)]
    halos = [C.cpm_part_halo_nodes(p) for p in parts]
    y_cat = torch.empty_like(u)
    for r, p in enumerate(parts):
        assert (p.lo, p.hi) == (bounds[r], bounds[r + 1])
        h_ = halos[r]
        assert np.all(np.diff(h_) > 0)
        assert not np.any((h_ >= p.lo) & (h_ < p.hi))
        counts = request_counts(h_, bounds)
        assert counts[r] == 0
        u_own = u[p.lo:p.hi].contiguous()
        u_halo = u[torch.from_numpy(h_).cuda()].contiguous()
        y_own = torch.empty(p.n_owned, dtype=torch.float64, device="cuda")
        C.cpm_part_apply_local(p, 3.0, u_own, u_halo, y_own)
        y_cat[p.lo:p.hi] = y_own
    torch.cuda.synchronize()
    assert torch.equal(y_cat, y)
    # sub-band tiles: [0, n_interior_tiles) read no halo node (extended while the halo
    # exchange is in flight), every rank of R >= 2 has boundary tiles
    for p in parts:
        assert 0 <= p.n_interior_tiles < p.n_tiles

    # send plan = inverse of the receive plans (what exchange_requests computes)
    for r, p in enumerate(parts):
        send = [halos[q][owners(halos[q], bounds) == r] for q in range(R)]
        C.cpm_part_set_send(p, np.concatenate(send), np.array([len(s) for s in send]))
        assert p.n_send == sum(len(s) for s in send)
    with pytest.raises(cpm.CpmError):
        C.cpm_part_set_send(parts[0], np.array([bounds[1]]), np.array([0, 1] + [0] * (R - 2)))


def test_single_rank_partition_solve_matches_cpm_solve(cpm):
    """nranks = 1: cpm_part_solve runs without a communicator and equals cpm_solve."""
    from paper_2110_06322_b200 import cpm as C

    band = cpm.cpm_build_band("sphere", 0.1)
    p = C.cpm_part_create(band, 0, 1)
    assert p.n_halo == 0 and p.n_owned == band.n
    f = torch.empty(band.n, dtype=torch.float64, device="cuda")
    cpm.cpm_eval_sph(band, 3, 2, 13.0, f)
    u1 = torch.zeros_like(f)
    u2 = torch.zeros_like(f)
    s1 = cpm.cpm_solve(band, 1.0, f, u1, rtol=1e-10, restart=30)
    s2 = C.cpm_part_solve(p, None, 1.0, f, u2, rtol=1e-10, restart=30)
    assert s1.iterations == s2.iterations
    assert torch.equal(u1, u2)


@pytest.mark.parametrize("kind,h,R,S", [("torus", 0.05, 2, 8), ("sphere", 0.1, 4, 8), ("sphere", 0.1, 8, 8)])
def test_partitioned_ras_matches_global_ras(cpm, kind, h, R, S):
    """Distributed RAS on one GPU: every rank's share (its S/R subdomains, overlap
    values from the other slabs given by indexing = what the RAS-halo exchange moves)
    concatenates to the single-GPU RAS apply, up to the rounding of the inner
    GMRES reductions (different segment batching)."""
    from paper_2110_06322_b200 import cpm as C
    from paper_2110_06322_b200.distributed import owners, slab_bounds

    band = cpm.cpm_build_band(kind, h) if kind == "sphere" else cpm.cpm_build_band(kind, h, R=1.0, r=0.4)
    n, c, k = band.n, 1.0, 8
    ga = cpm.cpm_band_active_coords(band).astype(np.int64)
    r = torch.from_numpy(seeded_inputs.uniform_pm1(7, ga)).cuda()
    z = torch.empty_like(r)
    cpm.cpm_ras_apply(cpm.cpm_ras_setup(band, S, 4, k, c), r, z)
    bounds = slab_bounds(n, R)
    z_cat = torch.empty_like(r)
    rs = []
    for q in range(R):
        p = C.cpm_part_create(band, q, R)
        ras = C.cpm_part_ras_setup(p, S, 4, k, c)
        inf = C.cpm_ras_get_info(ras)
        assert (inf["n_sub_local"], inf["sub0"], inf["n_owned"]) == (S // R, q * (S // R), p.n_owned)
        halo = C.cpm_ras_halo_nodes(ras)
        assert np.all(np.diff(halo) > 0) and not np.any((halo >= p.lo) & (halo < p.hi))
        zq = torch.empty(p.n_owned, dtype=torch.float64, device="cuda")
        C.cpm_part_ras_apply_local(ras, r[p.lo:p.hi].contiguous(), r[torch.from_numpy(halo).cuda()].contiguous(), zq)
        z_cat[p.lo:p.hi] = zq
        rs.append((p, ras, halo))
    torch.cuda.synchronize()
    err = float((z_cat - z).abs().max() / z.abs().max())
    assert err <= 1e-12, err
    # send plans = inverse of the receive plans
    for q, (p, ras, _) in enumerate(rs):
        send = [rs[t][2][owners(rs[t][2], bounds) == q] for t in range(R)]
        C.cpm_ras_set_send(ras, np.concatenate(send), np.array([len(s) for s in send]))
        assert C.cpm_ras_get_info(ras)["n_send"] == sum(len(s) for s in send)
    with pytest.raises(cpm.CpmError, match="multiple"):
        C.cpm_part_ras_setup(rs[0][0], S + 1, 4, k, c)
    with pytest.raises(cpm.CpmError, match="partitioned"):
        cpm.cpm_ras_apply(rs[0][1], r, z)


def test_single_rank_partition_ras_solve_matches_cpm_solve(cpm):
    """nranks = 1: the partitioned RAS-FGMRES equals cpm_solve with cpm_ras_setup."""
    from paper_2110_06322_b200 import cpm as C

    band = cpm.cpm_build_band("torus", 0.05, R=1.0, r=0.4)
    p = C.cpm_part_create(band, 0, 1)
    f = torch.empty(band.n, dtype=torch.float64, device="cuda")
    cpm.cpm_eval_torus_rhs(band, seeded_inputs.smooth_modulation_coeffs(1), f)
    u1 = torch.zeros_like(f)
    u2 = torch.zeros_like(f)
    s1 = cpm.cpm_solve(band, 1.0, f, u1, rtol=1e-10, restart=50, ras=cpm.cpm_ras_setup(band, 8, 4, 8, 1.0))
    ras = C.cpm_part_ras_setup(p, 8, 4, 8, 1.0)
    assert C.cpm_ras_get_info(ras)["n_halo"] == 0
    s2 = C.cpm_part_solve(p, None, 1.0, f, u2, rtol=1e-10, restart=50, ras=ras)
    assert s1.converged and s2.converged and s1.iterations == s2.iterations
    assert float((u1 - u2).abs().max() / u1.abs().max()) <= 1e-12
