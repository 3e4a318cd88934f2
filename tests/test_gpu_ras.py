"""GPU parity of the RAS preconditioner (batched inexact local GMRES) and of
FGMRES + RAS against the oracle (oracle/ras.py, oracle/krylov.py)."""
import numpy as np
import pytest

import seeded_inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.band import Band as OBand  # noqa: E402
from oracle.krylov import gmres as ogmres  # noqa: E402
from oracle.operator import shifted_operator  # noqa: E402
from oracle.problems import rhs_sph, rhs_torus  # noqa: E402
from oracle.ras import RAS as ORAS  # noqa: E402
from oracle.surfaces import Sphere, Torus  # noqa: E402


@pytest.fixture(scope="module")
def cpm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2110_06322_b200._build import build

    build()
    import paper_2110_06322_b200 as p

    return p


def _setup(cpm, kind, h, c):
    if kind == "sphere":
        gb, ob = cpm.cpm_build_band("sphere", h), OBand(Sphere(1.0), h)
    else:
        gb, ob = cpm.cpm_build_band("torus", h, R=1.0, r=0.4), OBand(Torus(1.0, 0.4), h)
    ga = cpm.cpm_band_active_coords(gb).astype(np.int64)
    perm = ob.index_active(ga)
    assert np.all(perm >= 0)
    return gb, ob, ga, perm, shifted_operator(ob, c)


@pytest.mark.parametrize("nsub,overlap,k", [(8, 4, 10), (3, 2, 5), (1, 0, 12), (16, 1, 3)])
def test_ras_apply_parity(cpm, nsub, overlap, k):
    c = 1.0
    gb, ob, ga, perm, A = _setup(cpm, "sphere", 0.1, c)
    M_o = ORAS(ob, A, nsub=nsub, overlap=overlap, k_inner=k, local="gmres")
    ras = cpm.cpm_ras_setup(gb, nsub, overlap, k, c)
    r_h = seeded_inputs.uniform_pm1(5, ga)
    r = torch.from_numpy(r_h).cuda()
    z = torch.empty_like(r)
    cpm.cpm_ras_apply(ras, r, z)
    torch.cuda.synchronize()
    r_o = np.empty(ob.nA)
    r_o[perm] = r_h
    z_o = M_o(r_o)[perm]
    err = np.abs(z.cpu().numpy() - z_o).max() / np.abs(z_o).max()
    assert err <= 1e-10, err


def test_ras_apply_host_pointers(cpm):
    gb, ob, ga, perm, A = _setup(cpm, "sphere", 0.1, 1.0)
    ras = cpm.cpm_ras_setup(gb, 4, 2, 4, 1.0)
    r_h = seeded_inputs.uniform_pm1(6, ga)
    z_h = np.empty_like(r_h)
    cpm.cpm_ras_apply(ras, r_h, z_h)
    z = torch.empty(gb.n, dtype=torch.float64, device="cuda")
    cpm.cpm_ras_apply(ras, torch.from_numpy(r_h).cuda(), z)
    torch.cuda.synchronize()
    assert np.array_equal(z.cpu().numpy(), z_h)


def test_ras_args(cpm):
    gb = cpm.cpm_build_band("sphere", 0.1)
    for bad in [(0, 1, 4), (8, -1, 4), (8, 2, 0), (8, 2, 65), (65, 2, 4)]:
        with pytest.raises(cpm.CpmError):
            cpm.cpm_ras_setup(gb, *bad, 1.0)


@pytest.mark.parametrize("kind,h,c,restart", [("sphere", 0.1, 1.0, 30), ("torus", 0.05, 1.0, 50)])
def test_fgmres_ras_parity(cpm, kind, h, c, restart):
    """RAS-preconditioned FGMRES (config 2 shape: 8 Morton slabs, overlap 4)."""
    gb, ob, ga, perm, A = _setup(cpm, kind, h, c)
    if kind == "sphere":
        f_o = rhs_sph(ob, c, 3, 2)
        f = torch.empty(gb.n, dtype=torch.float64, device="cuda")
        cpm.cpm_eval_sph(gb, 3, 2, c + 12.0, f)
    else:
        f_o = rhs_torus(ob, seed=1)
        f = torch.empty(gb.n, dtype=torch.float64, device="cuda")
        cpm.cpm_eval_torus_rhs(gb, seeded_inputs.smooth_modulation_coeffs(1), f)
    k = 8
    ras = cpm.cpm_ras_setup(gb, 8, 4, k, c)
    u = torch.zeros_like(f)
    st = cpm.cpm_solve(gb, c, f, u, rtol=1e-10, restart=restart, ras=ras)
    M_o = ORAS(ob, A, nsub=8, overlap=4, k_inner=k, local="gmres")
    x_o, so = ogmres(lambda v: A @ v, f_o, restart=restart, rtol=1e-10, M=M_o)
    assert st.converged and so.converged
    assert abs(st.iterations - so.iterations) <= 1, (st.iterations, so.iterations)
    err = np.abs(u.cpu().numpy() - x_o[perm]).max() / np.abs(x_o).max()
    assert err <= 1e-8, err
    # and it is the solution of the unpreconditioned problem
    x0, _ = ogmres(lambda v: A @ v, f_o, restart=restart, rtol=1e-10)
    assert np.abs(u.cpu().numpy() - x0[perm]).max() / np.abs(x0).max() <= 1e-8
