"""GPU parity for the solver settings the BASELINE configs use beyond the round-1
cases, and the solver's degenerate-input behaviour:

* RAS-FGMRES(50) at c = 0.1 on a config-3-shaped problem (unit sphere, f = Y_10^5 +
  1e-3 N(0,1) seed 2) with k_inner in {16, 64} and overlap in {4, 16} against
  oracle.ras.RAS + oracle.krylov.gmres (iterations +-1, solution 1e-8);
* cpm_ras_apply with k_inner = 64 (the 64-column segmented register class);
* GMRES(128), whose last step of a cycle reduces k = 129 columns (the second
  column per thread of the 128-thread reduction pass);
* the config-1 geometry (unit sphere, c = 10, f = (c + 42) Y_6^3) at h = 1/100,
  GMRES(50): iteration-count parity on a ~1M-node band;
* non-finite inputs: an error for a non-finite f, a breakdown (no endless restart
  loop) for a non-finite initial guess.
"""
import numpy as np
import pytest

import seeded_inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.band import Band as OBand  # noqa: E402
from oracle.krylov import gmres as ogmres  # noqa: E402
from oracle.operator import shifted_operator  # noqa: E402
from oracle.problems import rhs_noisy_sph, rhs_sph  # noqa: E402
from oracle.ras import RAS as ORAS  # noqa: E402
from oracle.surfaces import Sphere  # noqa: E402

SOLVE_TOL = 1e-8


@pytest.fixture(scope="module")
def cpm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2110_06322_b200._build import build

    build()
    import paper_2110_06322_b200 as p

    return p


def _sphere(cpm, h):
    gb, ob = cpm.cpm_build_band("sphere", h), OBand(Sphere(1.0), h)
    ga = cpm.cpm_band_active_coords(gb).astype(np.int64)
    perm = ob.index_active(ga)
    assert np.all(perm >= 0)
    return gb, ob, ga, perm


@pytest.fixture(scope="module")
def c3(cpm):
    """config-3-shaped problem at h = 0.08: c = 0.1, f = Y_10^5(cp) + 1e-3 N(0,1) seed 2."""
    c = 0.1
    gb, ob, ga, perm = _sphere(cpm, 0.08)
    A = shifted_operator(ob, c)
    f_o = rhs_noisy_sph(ob, 10, 5, seed=2)
    f = torch.empty(gb.n, dtype=torch.float64, device="cuda")
    cpm.cpm_eval_sph(gb, 10, 5, 1.0, f)
    f += torch.from_numpy(1e-3 * seeded_inputs.normal(2, ga)).cuda()
    assert np.abs(f.cpu().numpy() - f_o[perm]).max() <= 1e-13
    return gb, ob, perm, A, f, f_o, c


@pytest.mark.parametrize("k_inner,overlap", [(16, 4), (64, 16), (16, 16), (64, 4)])
def test_ras_fgmres_parity_c01(cpm, c3, k_inner, overlap):
    gb, ob, perm, A, f, f_o, c = c3
    ras = cpm.cpm_ras_setup(gb, 8, overlap, k_inner, c)
    u = torch.zeros_like(f)
    st = cpm.cpm_solve(gb, c, f, u, rtol=1e-10, restart=50, ras=ras)
    M_o = ORAS(ob, A, nsub=8, overlap=overlap, k_inner=k_inner, local="gmres")
    x_o, so = ogmres(lambda v: A @ v, f_o, restart=50, rtol=1e-10, M=M_o)
    assert st.converged and so.converged
    assert abs(st.iterations - so.iterations) <= 1, (st.iterations, so.iterations)
    err = np.abs(u.cpu().numpy() - x_o[perm]).max() / np.abs(x_o).max()
    assert err <= SOLVE_TOL, err


@pytest.mark.parametrize("nsub,overlap", [(8, 16), (3, 4)])
def test_ras_apply_parity_k64(cpm, c3, nsub, overlap):
    gb, ob, perm, A, f, f_o, c = c3
    ga = cpm.cpm_band_active_coords(gb).astype(np.int64)
    ras = cpm.cpm_ras_setup(gb, nsub, overlap, 64, c)
    r_h = seeded_inputs.uniform_pm1(5, ga)
    z = torch.empty(gb.n, dtype=torch.float64, device="cuda")
    cpm.cpm_ras_apply(ras, torch.from_numpy(r_h).cuda(), z)
    torch.cuda.synchronize()
    r_o = np.empty(ob.nA)
    r_o[perm] = r_h
    z_o = ORAS(ob, A, nsub=nsub, overlap=overlap, k_inner=64, local="gmres")(r_o)[perm]
    err = np.abs(z.cpu().numpy() - z_o).max() / np.abs(z_o).max()
    assert err <= 1e-10, err


def test_gmres128_parity(cpm):
    """GMRES(128) over several full cycles (random f: ~230 iterations), so every
    cycle's final reduction covers k = 129 columns."""
    h, c = 0.05, 1.0
    gb, ob, ga, perm = _sphere(cpm, h)
    f_h = seeded_inputs.uniform_pm1(4, ga)
    f_o = np.empty(ob.nA)
    f_o[perm] = f_h
    A = shifted_operator(ob, c)
    x_o, so = ogmres(lambda v: A @ v, f_o, restart=128, rtol=1e-10)
    assert so.converged and so.iterations > 129
    u = torch.zeros(gb.n, dtype=torch.float64, device="cuda")
    st = cpm.cpm_solve(gb, c, torch.from_numpy(f_h).cuda(), u, rtol=1e-10, restart=128)
    assert st.converged
    assert abs(st.iterations - so.iterations) <= 1, (st.iterations, so.iterations)
    err = np.abs(u.cpu().numpy() - x_o[perm]).max() / np.abs(x_o).max()
    assert err <= SOLVE_TOL, err


def test_solve_parity_config1_geometry_h100(cpm):
    """Config-1 problem (c = 10, f = (c + 42) Y_6^3) at h = 1/100 (~1M nodes), GMRES(50)."""
    h, c = 0.01, 10.0
    gb, ob, ga, perm = _sphere(cpm, h)
    f = torch.empty(gb.n, dtype=torch.float64, device="cuda")
    cpm.cpm_eval_sph(gb, 6, 3, c + 42.0, f)
    u = torch.zeros_like(f)
    st = cpm.cpm_solve(gb, c, f, u, rtol=1e-10, restart=50)
    A = shifted_operator(ob, c)
    x_o, so = ogmres(lambda v: A @ v, rhs_sph(ob, c, 6, 3), restart=50, rtol=1e-10)
    assert st.converged and so.converged
    assert abs(st.iterations - so.iterations) <= 1, (st.iterations, so.iterations)
    err = np.abs(u.cpu().numpy() - x_o[perm]).max() / np.abs(x_o).max()
    assert err <= SOLVE_TOL, err


def test_nonfinite_inputs(cpm):
    gb = cpm.cpm_build_band("sphere", 0.1)
    f = torch.empty(gb.n, dtype=torch.float64, device="cuda")
    cpm.cpm_eval_sph(gb, 3, 2, 13.0, f)
    bad = f.clone()
    bad[7] = float("nan")
    with pytest.raises(cpm.CpmError, match="not finite"):
        cpm.cpm_solve(gb, 1.0, bad, torch.zeros_like(f), rtol=1e-10, restart=30)
    for restart in (30, 50):
        u = torch.zeros_like(f)
        u[3] = float("nan")
        st = cpm.cpm_solve(gb, 1.0, f, u, rtol=1e-10, restart=restart, maxit=100000)
        assert not st.converged and st.breakdown and st.iterations == 0
    # FGMRES (RAS) path: the estimate turns non-finite -> stop, no endless restart loop
    ras = cpm.cpm_ras_setup(gb, 4, 2, 4, 1.0)
    u = torch.zeros_like(f)
    u[3] = float("inf")
    st = cpm.cpm_solve(gb, 1.0, f, u, rtol=1e-10, restart=30, maxit=100000, ras=ras)
    assert not st.converged and st.iterations < 100000
