"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerances (north_star): one apply agrees to relative max-norm 1e-12; converged
solutions agree to 1e-8 relative at rtol 1e-10 with iteration counts +-1.
Integer work (band membership, ordering) is compared bit-exactly.
"""
import math

import numpy as np
import pytest

import seeded_inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.band import Band as OBand, node_key  # noqa: E402
from oracle.krylov import gmres as ogmres  # noqa: E402
from oracle.operator import apply_rows, shifted_operator  # noqa: E402
from oracle.order import band_order_key  # noqa: E402
from oracle.problems import exact_sph, rhs_sph, rhs_torus  # noqa: E402
from oracle.surfaces import Sphere, Torus  # noqa: E402

APPLY_TOL = 1e-12
SOLVE_TOL = 1e-8


@pytest.fixture(scope="module")
def cpm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2110_06322_b200._build import build

    build()
    import paper_2110_06322_b200 as p

    return p


def _perm_to_oracle(gpu_ijk: np.ndarray, ob: OBand) -> np.ndarray:
    """index into the oracle's Sigma_A for each GPU node (asserts all present)."""
    idx = ob.index_active(gpu_ijk.astype(np.int64))
    assert np.all(idx >= 0)
    return idx


def _gpu_band(cpm, kind, h, **kw):
    return cpm.cpm_build_band(kind, h, **kw)


CASES = [("sphere", 0.1, {}), ("sphere", 0.13, {}), ("torus", 0.05, {"R": 1.0, "r": 0.4}),
         ("sphere", 0.06, {"R": 0.7}),
         ("sphere", 0.19, {}),  # coarsest spacing with lambda + h < reach: sparse, ragged tiles
         ("sphere", 0.1, {"L": 1.2}),  # band clipped by the box [-L, L]^3 (stencils still inside)
         ("sphere", 0.09, {"R": 1.3}),  # radius and spacing off the lattice
         ("torus", 0.045, {"R": 1.2, "r": 0.5})]


def _oracle_surface(kind, kw):
    return Sphere(kw.get("R", 1.0)) if kind == "sphere" else Torus(kw.get("R", 1.0), kw.get("r", 0.4))


@pytest.mark.parametrize("kind,h,kw", CASES)
def test_band_bit_exact(cpm, kind, h, kw):
    gb = _gpu_band(cpm, kind, h, **kw)
    ob = OBand(_oracle_surface(kind, kw), h, L=kw.get("L", 2.0))
    ga = cpm.cpm_band_active_coords(gb).astype(np.int64)
    gg = cpm.cpm_band_ghost_coords(gb).astype(np.int64)
    assert gb.info.n_active == ob.nA and gb.info.n_ghost == ob.nG
    assert np.array_equal(np.sort(node_key(ga)), ob.akeys)
    assert np.array_equal(np.sort(node_key(gg)), ob.gkeys)
    # band order (reading R8): strictly increasing Morton-brick key
    keys = band_order_key(ga)
    assert np.all(np.diff(keys) > 0)


def _band_with_env(cpm, env, kind, h, **kw):
    """A band built with build-time switches (read by cpm_build_band from the environment)."""
    import os
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return _gpu_band(cpm, kind, h, **kw)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


def _item_order_band(cpm, kind, h, **kw):
    """A band in the item order (CPM_ITEMS=1: the k_extend_it experiment)."""
    return _band_with_env(cpm, {"CPM_ITEMS": "1"}, kind, h, **kw)


@pytest.mark.parametrize("kind,h,kw", [CASES[0], CASES[2], CASES[4], CASES[7]])
def test_item_order_invariants(cpm, kind, h, kw):
    """The item order (build.cu k_item_order): the
    rounds of a tile cover its eval nodes once, in order; an item's two nodes share
    a stencil base; in a chunk round (lanes in use even, every lane pair one base)
    a warp reads at most 16 distinct bases, in a lone round at most 32; every
    stencil stays inside its tile's box."""
    gb = _item_order_band(cpm, kind, h, **kw)
    tiles, eoff = cpm.cpm_band_eval_order(gb)
    rounds = cpm.cpm_band_item_rounds(gb)
    assert int((tiles[:, 1] - tiles[:, 0]).sum()) == gb.info.n_active + gb.info.n_ghost
    for t, (e0, e1, word, sx, sxy, cells) in enumerate(tiles.astype(np.int64)):
        assert word >> 30 == 1
        nr = word & 0xFFFF
        ne = e1 - e0
        assert e0 % 4 == 0 and 1 <= nr <= 32 and np.all(rounds[t, nr:] == 0)
        eo = eoff[e0:e1].astype(np.int64)
        base, cell = eo & 0xFFFF, eo >> 16
        assert np.all(cell < 512) and len(np.unique(cell)) == ne
        assert np.all(base + 3 * sxy + 3 * sx + 3 < cells)
        nxt = 0
        for w in rounds[t, :nr].astype(np.uint64):
            w = int(w)
            flags, first, nv = w & 0xFFFFFFFF, (w >> 32) & 0xFFFF, (w >> 48) & 0x3F
            assert first == nxt and 1 <= nv <= 32 and flags >> nv == 0
            starts = [first + l + bin(flags & ((1 << l) - 1)).count("1") for l in range(nv)]
            two = [(flags >> l) & 1 for l in range(nv)]
            for st, tw in zip(starts, two):
                if tw:
                    assert base[st] == base[st + 1]
            lane_base = [base[st] for st in starts]
            pair_round = nv % 2 == 0 and all(lane_base[2 * k] == lane_base[2 * k + 1] for k in range(nv // 2))
            assert len(set(lane_base)) <= (16 if pair_round else 32)
            nxt = starts[-1] + 1 + two[-1]
        assert nxt == ne


@pytest.mark.parametrize("kind,h,kw", CASES)
def test_eval_order_invariants(cpm, kind, h, kw):
    """The extend's node order (build.cu k_warp_order): every
    eval node once per tile, pairs share a stencil base, each warp of the pair
    region (32 slots, the nd unpaired nodes completing its last warp on 2 slots)
    reads at most 16 distinct bases, every stencil stays inside its tile's box."""
    gb = _gpu_band(cpm, kind, h, **kw)
    tiles, eoff = cpm.cpm_band_eval_order(gb)
    with pytest.raises(cpm.CpmError):
        cpm.cpm_band_item_rounds(gb)
    assert int((tiles[:, 1] - tiles[:, 0]).sum()) == gb.info.n_active + gb.info.n_ghost
    for e0, e1, npnd, sx, sxy, cells in tiles.astype(np.int64):
        npair, nd = npnd & 0xFFFF, npnd >> 16
        ne = e1 - e0
        assert e0 % 4 == 0 and 0 <= 2 * npair + nd <= ne and 0 <= nd < 16
        eo = eoff[e0:e1].astype(np.int64)
        base, cell = eo & 0xFFFF, eo >> 16
        assert np.all(cell < 512) and len(np.unique(cell)) == ne
        assert np.all(base + 3 * sxy + 3 * sx + 3 < cells)
        assert np.array_equal(base[0:2 * npair:2], base[1:2 * npair:2])
        np2 = 2 * npair
        s = np.arange(ne + nd)
        node = np.where(s < np2, s, np.where(s < np2 + 2 * nd, np2 + (s - np2) // 2, s - nd))
        assert np.array_equal(np.unique(node), np.arange(ne))
        for w0 in range(0, np2 + 2 * nd, 32):           # pair-region warps
            assert len(np.unique(base[node[w0:w0 + 32]])) <= 16
        # the unpaired region starts on a warp boundary (or the tile's last warp)
        assert (np2 + 2 * nd) % 32 == 0 or np2 + nd == ne


@pytest.mark.parametrize("kind,h,kw", [CASES[0], CASES[2], CASES[4], CASES[7]])
def test_item_order_apply_bit_identical_to_pair_order(cpm, kind, h, kw):
    """k_extend_it (the item-order experiment) evaluates each node with
    k_extend_nt's operations in the same order: the two node orders give
    bit-identical applies."""
    gi = _item_order_band(cpm, kind, h, **kw)
    gp = _gpu_band(cpm, kind, h, **kw)
    ga = cpm.cpm_band_active_coords(gi).astype(np.int64)
    assert np.array_equal(ga, cpm.cpm_band_active_coords(gp))
    u = torch.from_numpy(seeded_inputs.uniform_pm1(0, ga)).cuda()
    yi, yp = torch.empty_like(u), torch.empty_like(u)
    cpm.cpm_apply(gi, 1.0, u, yi)
    cpm.cpm_apply(gp, 1.0, u, yp)
    torch.cuda.synchronize()
    assert torch.equal(yi, yp)


@pytest.mark.parametrize("kind,h,kw", [CASES[2], CASES[4]])
def test_run_order_does_not_change_the_apply(cpm, kind, h, kw):
    """The fill runs in source order (default) or box-row order (CPM_RUNSORT=0)
    stage the same box: bit-identical applies."""
    g0 = _gpu_band(cpm, kind, h, **kw)
    g1 = _band_with_env(cpm, {"CPM_RUNSORT": "0"}, kind, h, **kw)
    ga = cpm.cpm_band_active_coords(g0).astype(np.int64)
    u = torch.from_numpy(seeded_inputs.uniform_pm1(0, ga)).cuda()
    y0, y1 = torch.empty_like(u), torch.empty_like(u)
    cpm.cpm_apply(g0, 1.0, u, y0)
    cpm.cpm_apply(g1, 1.0, u, y1)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)


@pytest.mark.parametrize("kind,h,kw", CASES)
@pytest.mark.parametrize("c", [1.0, 10.0])
def test_apply_parity(cpm, kind, h, kw, c):
    gb = _gpu_band(cpm, kind, h, **kw)
    ob = OBand(_oracle_surface(kind, kw), h, L=kw.get("L", 2.0))
    ga = cpm.cpm_band_active_coords(gb).astype(np.int64)
    perm = _perm_to_oracle(ga, ob)
    u_h = seeded_inputs.uniform_pm1(0, ga)
    u = torch.from_numpy(u_h).cuda()
    y = torch.empty_like(u)
    cpm.cpm_apply(gb, c, u, y)
    torch.cuda.synchronize()
    A = shifted_operator(ob, c)
    u_o = np.empty(ob.nA)
    u_o[perm] = u_h
    y_o = (A @ u_o)[perm]
    err = np.abs(y.cpu().numpy() - y_o).max() / np.abs(y_o).max()
    assert err <= APPLY_TOL, err


@pytest.mark.parametrize("kind,h,kw", [CASES[0], CASES[2], CASES[4]])
def test_outputs_written_only_in_range(cpm, kind, h, kw):
    """Sentinels around the caller's vectors: apply, solve and RAS apply write
    exactly their n outputs (every one of them) and nothing before or after."""
    gb = _gpu_band(cpm, kind, h, **kw)
    n, pad = gb.n, 4096
    ga = cpm.cpm_band_active_coords(gb).astype(np.int64)
    u = torch.from_numpy(seeded_inputs.uniform_pm1(0, ga)).cuda()
    sentinel = 12345.0

    def guarded():
        buf = torch.full((n + 2 * pad,), sentinel, dtype=torch.float64, device="cuda")
        return buf, buf[pad:pad + n]

    def intact(buf):
        torch.cuda.synchronize()
        return bool((buf[:pad] == sentinel).all()) and bool((buf[pad + n:] == sentinel).all())

    yb, y = guarded()
    cpm.cpm_apply(gb, 1.0, u, y)
    assert intact(yb) and not bool((y == sentinel).any())
    # inputs inside NaN padding: a read outside [0, n) would show up in the result
    ub = torch.full((n + 2 * pad,), float("nan"), dtype=torch.float64, device="cuda")
    ub[pad:pad + n] = u
    y2 = torch.empty_like(u)
    cpm.cpm_apply(gb, 1.0, ub[pad:pad + n], y2)
    torch.cuda.synchronize()
    assert torch.equal(y2, y)
    xb, x = guarded()
    x.zero_()
    st = cpm.cpm_solve(gb, 1.0, u, x, rtol=1e-6, restart=20, maxit=60)
    assert intact(xb) and st.iterations > 0
    ras = cpm.cpm_ras_setup(gb, 4, 2, 4, 1.0)
    zb, z = guarded()
    cpm.cpm_ras_apply(ras, u, z)
    assert intact(zb) and not bool((z == sentinel).any())


def test_apply_host_pointers_match_device(cpm):
    gb = _gpu_band(cpm, "sphere", 0.1)
    ga = cpm.cpm_band_active_coords(gb).astype(np.int64)
    u_h = seeded_inputs.uniform_pm1(3, ga)
    y_h = np.empty_like(u_h)
    cpm.cpm_apply(gb, 2.0, u_h, y_h)                       # host in, host out
    u = torch.from_numpy(u_h).cuda()
    y = torch.empty_like(u)
    cpm.cpm_apply(gb, 2.0, u, y)
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), y_h)           # same kernels, same bits


def test_apply_edge_cases(cpm):
    gb = _gpu_band(cpm, "sphere", 0.1)
    n = gb.n
    z = torch.zeros(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(z)
    cpm.cpm_apply(gb, 3.0, z, y)
    assert torch.count_nonzero(y).item() == 0
    one = torch.ones(n, dtype=torch.float64, device="cuda")
    cpm.cpm_apply(gb, 3.0, one, y)                         # Delta_S 1 = 0 (E rows sum to 1)
    assert torch.max(torch.abs(y - 3.0)).item() <= 1e-12 * 6 / 0.01
    with pytest.raises(cpm.CpmError):
        cpm.cpm_apply(gb, 1.0, one, one)                   # aliasing rejected
    with pytest.raises(cpm.CpmError):
        cpm.cpm_apply(gb, 1.0, one[:-1], y)                # wrong length


def test_band_errors(cpm):
    with pytest.raises(cpm.CpmError, match="undefined|StencilEscape"):
        cpm.cpm_build_band("sphere", 0.25)                 # lambda + h > reach 1
    with pytest.raises(cpm.CpmError, match="empty|no active"):
        cpm.cpm_build_band("sphere", 0.1, L=0.3)           # box misses the surface
    with pytest.raises(cpm.CpmError, match="p = 3"):
        cpm.cpm_build_band("sphere", 0.1, p=2)
    # box clipping the band so that stencils leave Sigma_A: both sides refuse
    with pytest.raises(cpm.CpmError, match="StencilEscape"):
        cpm.cpm_build_band("sphere", 0.1, L=1.1)
    from oracle.interp import extension_matrix

    with pytest.raises(ValueError, match="StencilEscape"):
        extension_matrix(OBand(Sphere(1.0), 0.1, L=1.1))


def test_solve_parity_config0(cpm):
    """BASELINE config 0: unit sphere h=0.1, c=1, f=(c+12)Y_3^2, GMRES(30), rtol 1e-10."""
    h, c = 0.1, 1.0
    gb = _gpu_band(cpm, "sphere", h)
    ob = OBand(Sphere(1.0), h)
    ga = cpm.cpm_band_active_coords(gb).astype(np.int64)
    perm = _perm_to_oracle(ga, ob)
    f = torch.empty(gb.n, dtype=torch.float64, device="cuda")
    cpm.cpm_eval_sph(gb, 3, 2, c + 12.0, f)
    f_o = rhs_sph(ob, c, 3, 2)
    assert np.abs(f.cpu().numpy() - f_o[perm]).max() <= 1e-13 * np.abs(f_o).max()
    u = torch.zeros_like(f)
    st = cpm.cpm_solve(gb, c, f, u, rtol=1e-10, restart=30)
    A = shifted_operator(ob, c)
    x_o, so = ogmres(lambda v: A @ v, f_o, restart=30, rtol=1e-10)
    assert st.converged and so.converged
    assert abs(st.iterations - so.iterations) <= 1, (st.iterations, so.iterations)
    ug = u.cpu().numpy()
    err = np.abs(ug - x_o[perm]).max() / np.abs(x_o).max()
    assert err <= SOLVE_TOL, err
    assert st.resid_true <= 1.5e-10 * st.bnorm
    # and the discrete solution is O(h^2)-close to the manufactured solution
    assert np.abs(ug - exact_sph(ob, 3, 2)[perm]).max() < 0.03


@pytest.mark.parametrize("restart,its_tol", [(50, 1), (30, 1), (5, 0.10)])
def test_solve_parity_torus(cpm, restart, its_tol):
    """Torus R=1 r=0.4 (config 2 shape) at h=0.05.  Iteration counts must agree +-1 for
    the BASELINE restarts; for GMRES(5) (hundreds of restart cycles) the count is
    rounding-sensitive — the oracle itself gives 1889 on one host and 1811 on
    another — so only a 10 % band is asserted there (parity notes)."""
    h, c = 0.05, 1.0
    gb = _gpu_band(cpm, "torus", h, R=1.0, r=0.4)
    ob = OBand(Torus(1.0, 0.4), h)
    ga = cpm.cpm_band_active_coords(gb).astype(np.int64)
    perm = _perm_to_oracle(ga, ob)
    f_o = rhs_torus(ob, seed=1)
    f = torch.empty(gb.n, dtype=torch.float64, device="cuda")
    cpm.cpm_eval_torus_rhs(gb, seeded_inputs.smooth_modulation_coeffs(1), f)
    assert np.abs(f.cpu().numpy() - f_o[perm]).max() <= 1e-12
    u = torch.zeros_like(f)
    st = cpm.cpm_solve(gb, c, f, u, rtol=1e-10, restart=restart)
    A = shifted_operator(ob, c)
    x_o, so = ogmres(lambda v: A @ v, f_o, restart=restart, rtol=1e-10)
    assert st.converged and so.converged
    if isinstance(its_tol, int):
        assert abs(st.iterations - so.iterations) <= its_tol, (st.iterations, so.iterations)
    else:
        assert abs(st.iterations - so.iterations) <= its_tol * so.iterations, (st.iterations, so.iterations)
    err = np.abs(u.cpu().numpy() - x_o[perm]).max() / np.abs(x_o).max()
    assert err <= SOLVE_TOL, err


def test_solve_host_pointers_and_x0(cpm):
    gb = _gpu_band(cpm, "sphere", 0.1)
    f = np.empty(gb.n)
    cpm.cpm_eval_sph(gb, 3, 2, 13.0, f)
    u = np.zeros(gb.n)
    st = cpm.cpm_solve(gb, 1.0, f, u, rtol=1e-10, restart=30)
    assert st.converged
    st2 = cpm.cpm_solve(gb, 1.0, f, u.copy(), rtol=1e-10, restart=30)   # x0 = solution
    assert st2.iterations <= 3


def test_solve_parity_large_restart(cpm):
    """GMRES(64): the Krylov passes for k > 52 columns (128-element tiles)."""
    h, c = 0.1, 1.0
    gb = _gpu_band(cpm, "sphere", h)
    ob = OBand(Sphere(1.0), h)
    ga = cpm.cpm_band_active_coords(gb).astype(np.int64)
    perm = _perm_to_oracle(ga, ob)
    f = torch.empty(gb.n, dtype=torch.float64, device="cuda")
    cpm.cpm_eval_sph(gb, 3, 2, c + 12.0, f)
    u = torch.zeros_like(f)
    st = cpm.cpm_solve(gb, c, f, u, rtol=1e-10, restart=64)
    A = shifted_operator(ob, c)
    xo, so = ogmres(lambda v: A @ v, rhs_sph(ob, c, 3, 2), restart=64, rtol=1e-10)
    assert st.converged and so.converged
    assert abs(st.iterations - so.iterations) <= 1, (st.iterations, so.iterations)
    err = np.abs(u.cpu().numpy() - xo[perm]).max() / np.abs(xo).max()
    assert err <= SOLVE_TOL, err


def test_solve_degenerate_cases(cpm):
    """f = 0: u = 0 without an Arnoldi step; maxit reached: not converged, no error,
    the returned u still reduces the residual; restart = 1 (GMRES(1)) converges."""
    gb = _gpu_band(cpm, "sphere", 0.1)
    z = torch.zeros(gb.n, dtype=torch.float64, device="cuda")
    u = torch.zeros_like(z)
    st = cpm.cpm_solve(gb, 1.0, z, u, rtol=1e-10, restart=30)
    assert st.converged and st.iterations == 0 and torch.count_nonzero(u).item() == 0
    f = torch.empty_like(z)
    cpm.cpm_eval_sph(gb, 3, 2, 13.0, f)
    u.zero_()
    st = cpm.cpm_solve(gb, 1.0, f, u, rtol=1e-10, restart=30, maxit=5)
    assert not st.converged and st.iterations == 5 and st.resid_true < st.bnorm
    u.zero_()
    st = cpm.cpm_solve(gb, 10.0, f, u, rtol=1e-8, restart=1, maxit=20000)
    assert st.converged and st.resid_true <= 2e-8 * st.bnorm


# ------------------------------------------------------------------ full size (config 1)
@pytest.fixture(scope="module")
def big(cpm):
    gb = cpm.cpm_build_band("sphere", 1.0 / 200)
    return gb


def test_full_size_band_count(cpm, big):
    """config 1 band, h=1/200: node count against the oracle's own enumeration."""
    ob = OBand(Sphere(1.0), 1.0 / 200)
    assert big.info.n_active == ob.nA and big.info.n_ghost == ob.nG
    ga = cpm.cpm_band_active_coords(big).astype(np.int64)
    assert np.array_equal(np.sort(node_key(ga)), ob.akeys)


def test_full_size_apply_sampled(cpm, big):
    """config 1 apply (u ~ U[-1,1], seed 0) on 3000 sampled rows vs the oracle's row formula."""
    h = 1.0 / 200
    ga = cpm.cpm_band_active_coords(big).astype(np.int64)
    u = torch.from_numpy(seeded_inputs.uniform_pm1(0, ga)).cuda()
    y = torch.empty_like(u)
    cpm.cpm_apply(big, 10.0, u, y)
    torch.cuda.synchronize()
    rng = np.random.default_rng(11)
    sel = np.concatenate([rng.choice(big.n, 2990, replace=False), np.arange(5), big.n - 1 - np.arange(5)])

    class _B:
        pass

    _B.h = h
    _B.surface = Sphere(1.0)
    y_o = apply_rows(_B, 10.0, lambda q: seeded_inputs.uniform_pm1(0, q), ga[sel])
    yg = y.cpu().numpy()
    err = np.abs(yg[sel] - y_o).max() / np.abs(y_o).max()
    assert err <= APPLY_TOL, err
    # property at any size: constants are in the kernel of Delta_S^h
    one = torch.ones_like(u)
    cpm.cpm_apply(big, 10.0, one, y)
    assert torch.max(torch.abs(y - 10.0)).item() <= 1e-11 * 6 * 200 ** 2


def test_full_size_manufactured_solve(cpm, big):
    """config 1 solve: c=10, f=(c+42)Y_6^3, GMRES(50), rtol 1e-10: converges; residual
    recomputed by the oracle row formula on samples; O(h^2) error vs Y_6^3(cp)."""
    h, c = 1.0 / 200, 10.0
    f = torch.empty(big.n, dtype=torch.float64, device="cuda")
    cpm.cpm_eval_sph(big, 6, 3, c + 42.0, f)
    u = torch.zeros_like(f)
    st = cpm.cpm_solve(big, c, f, u, rtol=1e-10, restart=50)
    assert st.converged
    assert st.resid_true <= 2e-10 * st.bnorm
    ga = cpm.cpm_band_active_coords(big).astype(np.int64)
    ug = u.cpu().numpy()
    ob_s = Sphere(1.0)

    class _B:
        pass

    _B.h = h
    _B.surface = ob_s
    from oracle.sph import real_sph

    x = ga.astype(np.float64) * h
    cp, _ = ob_s.cp(x)
    exact = real_sph(6, 3, cp)
    assert np.abs(ug - exact).max() < 5e-3
    # oracle residual on sampled rows: u looked up by lattice coordinate
    keys = node_key(ga)
    order = np.argsort(keys)
    sk = keys[order]

    def u_of(q):
        pos = np.searchsorted(sk, node_key(q))
        assert np.all(sk[pos] == node_key(q))
        return ug[order[pos]]

    sel = np.random.default_rng(2).choice(big.n, 500, replace=False)
    fr = f.cpu().numpy()[sel] - apply_rows(_B, c, u_of, ga[sel])
    assert np.abs(fr).max() <= 1e-6 * np.abs(f.cpu().numpy()).max()


def test_apply_async_pinned_matches_apply(cpm):
    """cpm_apply_async on pinned host buffers (pipelined copies, two staging slots)
    gives the device apply's result for every call of a sequence."""
    gb = _gpu_band(cpm, "sphere", 0.1)
    ga = cpm.cpm_band_active_coords(gb).astype(np.int64)
    us = [torch.from_numpy(seeded_inputs.uniform_pm1(s, ga)).pin_memory() for s in range(5)]
    ys = [torch.empty(gb.n, dtype=torch.float64).pin_memory() for _ in range(5)]
    for u, y in zip(us, ys):
        cpm.cpm_apply_async(gb, 2.0, u.numpy(), y.numpy())
    cpm.cpm_apply_sync(gb)
    torch.cuda.synchronize()
    for u, y in zip(us, ys):
        yd = torch.empty(gb.n, dtype=torch.float64, device="cuda")
        cpm.cpm_apply(gb, 2.0, u.cuda(), yd)
        torch.cuda.synchronize()
        assert torch.equal(yd.cpu(), y)
    # pageable host memory falls back to the synchronous cpm_apply
    yp = np.empty(gb.n)
    cpm.cpm_apply_async(gb, 2.0, us[0].numpy().copy(), yp)
    assert np.array_equal(yp, ys[0].numpy())
