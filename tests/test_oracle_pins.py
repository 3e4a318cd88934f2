"""Pins of the CPU oracle to things other than itself (rule ③).

Every check here compares the oracle with the paper, mathematics or an
independent computation: textbook values, closed forms, invariants, special
cases reducing to a textbook stencil, brute force on tiny inputs, dense
direct solves, and the manufactured-solution convergence the north_star names.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest
import scipy.sparse.linalg as spla

import seeded_inputs
from oracle.band import Band, brute_force_band, lattice_points
from oracle.interp import OFFS, extension_matrix, extension_rows, lagrange_weights_1d, stencil_of
from oracle.krylov import arnoldi_fixed, gmres
from oracle.operator import apply_rows, laplace_beltrami_matrix, laplacian_matrix, shifted_operator
from oracle.order import band_order_key, slab_bounds
from oracle.problems import exact_sph, rhs_noisy_sph, rhs_sph, rhs_torus, torus_angles
from oracle.ras import RAS, disjoint_subdomains, grow_overlap
from oracle.sph import real_sph
from oracle.surfaces import Plane, Sphere, Torus

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            rows.append([float(Fraction(tok)) for tok in line.split()])
    return np.array(rows)


# ---------------------------------------------------------------- inputs
def test_seeded_inputs_counter_based():
    ijk = np.array([[0, 0, 0], [1, -2, 3], [-5, 7, 11]])
    a = seeded_inputs.uniform_pm1(0, ijk)
    b = seeded_inputs.uniform_pm1(0, ijk[::-1])[::-1]
    assert np.array_equal(a, b)                      # order independent
    assert np.all((a >= -1) & (a < 1))
    assert not np.array_equal(a, seeded_inputs.uniform_pm1(1, ijk))
    big = np.stack(np.meshgrid(*[np.arange(-20, 20)] * 3, indexing="ij"), -1).reshape(-1, 3)
    u = seeded_inputs.uniform_pm1(0, big)
    assert abs(u.mean()) < 0.01 and abs(u.var() - 1 / 3) < 0.01
    z = seeded_inputs.normal(2, big)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01


# ---------------------------------------------------------------- surfaces (Eq. 3)
def test_sphere_cp_closed_form():
    x = np.array([[2.0, 0, 0], [0.3, -0.4, 0.0], [0.1, 0.2, -1.7]])
    cp, d = Sphere(1.0).cp(x)
    assert np.allclose(cp[0], [1, 0, 0]) and d[0] == 1.0
    assert np.allclose(cp[1], [0.6, -0.8, 0]) and abs(d[1] - 0.5) < 1e-15
    assert np.allclose(np.linalg.norm(cp, axis=1), 1.0, atol=1e-15)
    assert np.allclose(np.linalg.norm(x - cp, axis=1), d, atol=1e-15)
    cp2, d2 = Sphere(1.0).cp(cp)                     # idempotence
    assert np.all(d2 < 1e-15)
    # radius R != 1 (cp = R x/|x|, PAPER.md:56-60 with the sphere's closed form)
    cp3, d3 = Sphere(2.5).cp(x)
    assert np.allclose(cp3[0], [2.5, 0, 0]) and d3[0] == 0.5
    assert np.allclose(cp3[1], [1.5, -2.0, 0]) and abs(d3[1] - 2.0) < 1e-15
    assert np.allclose(np.linalg.norm(x - cp3, axis=1), d3, atol=1e-15)


def _torus_pt(p):
    return np.array([(1 + 0.4 * np.cos(p[0])) * np.cos(p[1]),
                     (1 + 0.4 * np.cos(p[0])) * np.sin(p[1]), 0.4 * np.sin(p[0])])


def test_torus_cp_matches_brute_force_minimisation():
    from scipy.optimize import minimize

    rng = np.random.default_rng(5)
    T = Torus(1.0, 0.4)
    # random points within 0.3 of the torus
    th = rng.uniform(0, 2 * np.pi, 40)
    ph = rng.uniform(0, 2 * np.pi, 40)
    rr = 0.4 + rng.uniform(-0.3, 0.3, 40)
    x = np.stack([(1 + rr * np.cos(th)) * np.cos(ph), (1 + rr * np.cos(th)) * np.sin(ph), rr * np.sin(th)], 1)
    x += rng.normal(0, 0.02, x.shape)
    cp, d = T.cp(x)
    # brute force: dense parametric sampling + local refinement by golden search
    for n in range(x.shape[0]):
        a = np.linspace(0, 2 * np.pi, 721)
        A, B = np.meshgrid(a, a, indexing="ij")
        P = np.stack([(1 + 0.4 * np.cos(A)) * np.cos(B), (1 + 0.4 * np.cos(A)) * np.sin(B), 0.4 * np.sin(A)], -1)
        D = np.linalg.norm(P - x[n], axis=-1)
        q = np.unravel_index(np.argmin(D), D.shape)
        assert D[q] >= d[n] - 1e-12                 # nothing on the surface is closer
        res = minimize(lambda p: np.linalg.norm(_torus_pt(p) - x[n]), [a[q[0]], a[q[1]]],
                       method="Nelder-Mead", options={"xatol": 1e-12, "fatol": 1e-15})
        assert abs(res.fun - d[n]) < 1e-9            # refined optimum = oracle distance
        assert np.linalg.norm(_torus_pt(res.x) - cp[n]) < 1e-5
    # cp lies on the torus: (rho - R)^2 + z^2 = r^2
    rho = np.hypot(cp[:, 0], cp[:, 1])
    assert np.allclose((rho - 1) ** 2 + cp[:, 2] ** 2, 0.16, atol=1e-13)


# ---------------------------------------------------------------- band (§2.1)
@pytest.mark.parametrize(
    "surf,h,dist",
    [
        (Sphere(1.0), 0.2, lambda x, y, z: abs(math.sqrt(x * x + y * y + z * z) - 1.0)),
        (Torus(1.0, 0.4), 0.09, lambda x, y, z: abs(math.hypot(math.hypot(x, y) - 1.0, z) - 0.4)),
    ],
)
def test_band_matches_pure_python_triple_loop(surf, h, dist):
    b = Band(surf, h)
    act, ghost = brute_force_band(dist, h)
    assert set(map(tuple, b.active.tolist())) == act
    assert set(map(tuple, b.ghost.tolist())) == ghost
    assert b.nA == len(act) and b.nG == len(ghost)


def test_band_clipped_by_the_grid_box():
    """The grid is |i|, |j|, |k| <= M = round(L/h) (oracle/band.py header; cpm_build_band's L):
    with L = 1 the unit sphere's tube is cut by the box.  Counted here by a plain loop:
    active nodes are the lattice nodes of the box within lambda of the sphere, the box's
    faces included."""
    h, L = 0.2, 1.0
    b = Band(Sphere(1.0), h, L=L)
    M = 5
    lam = math.sqrt(17.0) * h
    want = {(i, j, k) for i in range(-M, M + 1) for j in range(-M, M + 1) for k in range(-M, M + 1)
            if abs(math.sqrt((i * h) ** 2 + (j * h) ** 2 + (k * h) ** 2) - 1.0) <= lam}
    got = set(map(tuple, b.active.tolist()))
    assert got == want
    assert any(max(abs(c) for c in n) == M for n in got)          # nodes on the box faces are kept
    assert len(got) < Band(Sphere(1.0), h).nA                       # and the box does clip the tube


def test_band_size_scales_as_h_minus_2():
    n1 = Band(Sphere(1.0), 0.1).nA
    n2 = Band(Sphere(1.0), 0.05).nA
    # codimension-1 tube of width 2 lambda: nA ~ 4 pi * 2 sqrt(17) / h^2
    assert 3.6 < n2 / n1 < 4.4
    assert abs(n2 - 4 * math.pi * 2 * math.sqrt(17) / 0.05 ** 2) / n2 < 0.05


# ---------------------------------------------------------------- interpolation / E (§2.1)
def test_lagrange_weights_golden():
    g = _golden("lagrange_p3.txt")
    w = lagrange_weights_1d(g[:, 0])
    assert np.allclose(w, g[:, 1:], atol=2e-16, rtol=0)


def test_lagrange_reproduces_cubics_1d():
    t = np.linspace(0, 1, 101, endpoint=False)
    w = lagrange_weights_1d(t)
    tau = np.array([-1.0, 0, 1, 2])
    for k in range(4):
        assert np.allclose(w @ tau ** k, t ** k, atol=1e-14)


@pytest.mark.parametrize("surf,h", [(Sphere(1.0), 0.1), (Torus(1.0, 0.4), 0.05)])
def test_E_rows_sum_to_one_and_reproduce_tricubics(surf, h):
    b = Band(surf, h)
    E = extension_matrix(b)
    assert np.abs(np.asarray(E.sum(axis=1)).ravel() - 1).max() < 1e-13
    xa = lattice_points(b.active, h)
    cp, _ = surf.cp(lattice_points(b.all, h))
    rng = np.random.default_rng(1)
    for _ in range(6):
        a, bb, c = rng.integers(0, 4, 3)
        q = lambda P: (P[:, 0] ** a) * (P[:, 1] ** bb) * (P[:, 2] ** c)
        assert np.abs(E @ q(xa) - q(cp)).max() < 1e-12


def test_E_on_lattice_plane_is_selection():
    P = Plane(0.0)
    b_nodes = np.array([[i, j, k] for i in range(-3, 4) for j in range(-3, 4) for k in range(-2, 3)])

    class _B:  # minimal band: every node is "active"
        h = 0.25
        surface = P
        akeys = None

    from oracle.band import node_key

    _B.akeys = np.sort(node_key(np.array([[i, j, k] for i in range(-8, 9) for j in range(-8, 9) for k in range(-4, 5)])))
    _B.all = b_nodes
    cols, vals = extension_rows(_B, b_nodes)
    assert np.all(np.isclose(vals, 0) | np.isclose(vals, 1))
    assert np.allclose(vals.sum(1), 1)


# ---------------------------------------------------------------- operators (Eq. 2, 4)
def test_delta_h_exact_on_quadratics():
    b = Band(Sphere(1.0), 0.1)
    D = laplacian_matrix(b)
    X = lattice_points(b.all, b.h)
    p = 3 * X[:, 0] ** 2 - X[:, 1] * X[:, 2] + 2 * X[:, 2] ** 2 + X[:, 0]
    assert np.allclose(D @ p, 10.0, atol=1e-9)


def test_semidiscrete_2d_golden_on_plane():
    """the flat case reduces to the 2-D -4/h^2, +1/h^2 stencil."""
    for h, centre, nb in _golden("semidiscrete_2d.txt"):
        P = Plane(0.0)

        class _B:
            pass

        _B.h = h
        _B.surface = P
        probes = np.array([[0, 0, 0], [1, -2, 0], [3, 1, 0]])
        # u = delta function at a probe and its neighbours -> read off stencil weights
        for pr in probes:
            def u_delta(ijk, tgt):
                return np.all(ijk == tgt[None, :], axis=1).astype(float)

            y_c = apply_rows(_B, 0.0, lambda q: u_delta(q, pr), pr[None, :])[0]
            y_n = apply_rows(_B, 0.0, lambda q: u_delta(q, pr + np.array([1, 0, 0])), pr[None, :])[0]
            y_z = apply_rows(_B, 0.0, lambda q: u_delta(q, pr + np.array([0, 0, 1])), pr[None, :])[0]
            # A = c I - Delta_S^h with c = 0  ->  -Delta_S^h
            assert abs(-y_c - centre) < 1e-9 * abs(centre)
            assert abs(-y_n - nb) < 1e-9 * abs(nb)
            assert abs(y_z) == 0.0                   # off-plane values are never read


def test_offlattice_plane_golden_rows():
    """Eq. 4 on a plane between lattice planes (z0 = h/2, h/4), where
    u != E u so the stabilisation term -(6/h^2)(I - E) is exercised; values derived by
    hand in tests/golden/offlattice_plane.txt.  Pins the sign and weight of that term
    (the row formula apply_rows; test_apply_rows_equals_assembled_matrix ties the
    assembled matrix to it)."""
    rows = _golden("offlattice_plane.txt")
    for h in (0.25, 0.1):
        for t, si, sj, sk, pi, pj, pk, val in rows:
            class _B:
                pass

            _B.h = h
            _B.surface = Plane(t * h)
            src = np.array([si, sj, sk], dtype=np.int64)
            probe = np.array([[pi, pj, pk]], dtype=np.int64)
            u_delta = lambda ijk: np.all(ijk == src[None, :], axis=1).astype(float)
            y = apply_rows(_B, 0.0, u_delta, probe)[0]      # (c I - Delta_S^h) u, c = 0
            assert abs(-y * h * h - val) <= 1e-12 * max(1.0, abs(val)), (t, si, sj, sk, pi, pj, pk)


def test_constants_in_kernel():
    b = Band(Sphere(1.0), 0.1)
    L = laplace_beltrami_matrix(b)
    assert np.abs(L @ np.ones(b.nA)).max() < 1e-9 * 6 / b.h ** 2


def test_apply_rows_equals_assembled_matrix():
    b = Band(Torus(1.0, 0.4), 0.05)
    A = shifted_operator(b, 2.5)
    u_of = lambda ijk: seeded_inputs.uniform_pm1(7, ijk)
    u = u_of(b.active)
    y = A @ u
    sel = np.random.default_rng(0).choice(b.nA, 300, replace=False)
    y1 = apply_rows(b, 2.5, u_of, b.active[sel])
    assert np.abs(y1 - y[sel]).max() <= 1e-12 * np.abs(y).max()


def test_eigenfunction_second_order():
    """Closed form on the unit sphere: the closest point extension of Y is constant on rays,
    so Delta(E Y)(x) = Delta_S Y / |x|^2 = -l(l+1) Y / |x|^2.  Eq. (4) must reproduce it
    at every band node up to O(h^2) (FD error O(h^2) + interpolation error O(h^4)/h^2)."""
    errs = []
    for h in (0.1, 0.05):
        b = Band(Sphere(1.0), h)
        L = laplace_beltrami_matrix(b)
        Y = exact_sph(b, 3, 2)
        r2 = np.sum(lattice_points(b.active, h) ** 2, axis=1)
        r = L @ Y + 12 * Y / r2
        errs.append(np.abs(r).max())
    assert errs[0] / errs[1] > 3.2


# ---------------------------------------------------------------- spherical harmonics
def test_real_sph_orthonormal():
    xg, wg = np.polynomial.legendre.leggauss(40)
    ph = np.linspace(0, 2 * np.pi, 80, endpoint=False)
    CT, PH = np.meshgrid(xg, ph, indexing="ij")
    W = np.repeat(wg[:, None], 80, 1) * (2 * np.pi / 80)
    st = np.sqrt(1 - CT ** 2)
    P = np.stack([st * np.cos(PH), st * np.sin(PH), CT], -1).reshape(-1, 3)
    lm = [(3, 2), (6, 3), (10, 5), (2, -1), (0, 0), (6, -3)]
    Ys = [real_sph(l, m, P) for l, m in lm]
    for a in range(len(lm)):
        for b_ in range(len(lm)):
            ip = np.sum(Ys[a] * Ys[b_] * W.ravel())
            assert abs(ip - (a == b_)) < 1e-12


@pytest.mark.parametrize("l,m", [(3, 2), (6, 3), (10, 5)])
def test_real_sph_is_harmonic_polynomial(l, m):
    """r^l Y_l^m(x/r) is harmonic: its 3-D Laplacian vanishes (=> Delta_S Y = -l(l+1) Y)."""
    rng = np.random.default_rng(l)
    x = rng.normal(size=(20, 3))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    f = lambda P: np.linalg.norm(P, axis=1) ** l * real_sph(l, m, P)
    d = 1e-3
    lap = -6 * f(x)
    for c in range(3):
        e = np.zeros(3)
        e[c] = d
        lap = lap + f(x + e) + f(x - e)
    lap /= d * d
    scale = l * l * np.abs(f(x)).max() + 1
    assert np.abs(lap).max() < 1e-4 * scale


# ---------------------------------------------------------------- manufactured solve (north_star pin)
def test_manufactured_solution_second_order():
    """u = Y_3^2(cp(x)), f = (c + 12) u converges at 2nd order (direct sparse solves)."""
    errs = []
    for h in (0.16, 0.08):
        b = Band(Sphere(1.0), h)
        A = shifted_operator(b, 1.0)
        u = spla.spsolve(A.tocsc(), rhs_sph(b, 1.0, 3, 2))
        errs.append(np.abs(u - exact_sph(b, 3, 2)).max())
    assert errs[1] < 0.01
    assert errs[0] / errs[1] > 3.2                  # observed order >= ~1.7 (pre-asymptotic ~3)


# ---------------------------------------------------------------- GMRES
def test_gmres_identity_one_iteration():
    b = np.arange(1.0, 11.0)
    x, st = gmres(lambda v: v, b, restart=5, rtol=1e-12)
    assert st.iterations == 1 and np.allclose(x, b)


def test_gmres_dense_random_vs_lu():
    rng = np.random.default_rng(3)
    A = rng.normal(size=(60, 60)) + 15 * np.eye(60)
    b = rng.normal(size=60)
    x, st = gmres(lambda v: A @ v, b, restart=7, rtol=1e-12)
    assert st.converged
    assert np.abs(x - np.linalg.solve(A, b)).max() < 1e-10
    assert st.resid_true <= 1.01e-12 * np.linalg.norm(b) + 1e-14


def test_gmres_cpm_tiny_band_vs_dense_direct():
    b = Band(Sphere(1.0), 0.16)
    A = shifted_operator(b, 1.0)
    f = rhs_sph(b, 1.0, 3, 2)
    x, st = gmres(lambda v: A @ v, f, restart=30, rtol=1e-10)
    xd = np.linalg.solve(A.toarray(), f)
    assert st.converged
    assert np.abs(x - xd).max() / np.abs(xd).max() < 1e-8


def test_arnoldi_fixed_full_dimension_is_exact():
    rng = np.random.default_rng(4)
    A = rng.normal(size=(12, 12)) + 6 * np.eye(12)
    r = rng.normal(size=12)
    z = arnoldi_fixed(lambda v: A @ v, r, 12)
    assert np.allclose(A @ z, r, atol=1e-10)


def test_arnoldi_fixed_minimises_residual_over_krylov_space():
    """k < n GMRES steps (reading R6): z_k = argmin_{z in K_k(A, b)} ||b - A z||_2.
    Checked against an independent least-squares fit on the explicit (column-normalised)
    Krylov basis [b, Ab, ..., A^{k-1} b] (the defining property of GMRES, Saad §6.5.1);
    a FOM (Galerkin) solve of the square Hessenberg system gives a larger residual."""
    rng = np.random.default_rng(11)
    n = 40
    A = rng.normal(size=(n, n)) + 4 * np.eye(n)
    b = rng.normal(size=n)
    for k in (1, 2, 3, 5, 8):
        z = arnoldi_fixed(lambda v: A @ v, b, k)
        K = np.empty((n, k))
        v = b.copy()
        for q in range(k):
            K[:, q] = v / np.linalg.norm(v)
            v = A @ K[:, q]
        coef, *_ = np.linalg.lstsq(A @ K, b, rcond=None)
        r_min = np.linalg.norm(b - A @ (K @ coef))
        r_z = np.linalg.norm(b - A @ z)
        assert abs(r_z - r_min) <= 1e-10 * np.linalg.norm(b), k
        # z lies in K_k(A, b)
        c2, *_ = np.linalg.lstsq(K, z, rcond=None)
        assert np.linalg.norm(K @ c2 - z) <= 1e-9 * np.linalg.norm(z)


# ---------------------------------------------------------------- RAS (§2.2)
def test_order_key_hand_values():
    k = band_order_key(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [8, 0, 0], [-1, 0, 0]]))
    base = (1 << 48) | (1 << 49) | (1 << 50)   # interleave(2^16) for x, y, z
    assert k[0] == base * 512
    assert k[1] == base * 512 + 1 and k[2] == base * 512 + 8 and k[3] == base * 512 + 64
    assert k[4] == (base | 1) * 512
    # brick -1 in x: 2^16 - 1 = 0xFFFF interleaved -> bits 0,3,...,45
    m = sum(1 << (3 * b) for b in range(16)) | (1 << 49) | (1 << 50)
    assert k[5] == m * 512 + 7
    # the axes of the brick Morton key (reading R8: x bits lowest, then y, then z): bit b
    # of the brick's x, y, z index sits at key bit 3b, 3b + 1, 3b + 2
    k2 = band_order_key(np.array([[0, 8, 0], [0, 0, 8], [0, 16, 0], [0, 0, 16], [16, 8, 24]]))
    assert k2[0] == (base | 2) * 512 and k2[1] == (base | 4) * 512
    assert k2[2] == (base | (1 << 4)) * 512 and k2[3] == (base | (1 << 5)) * 512
    # bricks (2, 1, 3): x bit 1 -> key bit 3; y bit 0 -> 1; z bits 0, 1 -> 2, 5
    assert k2[4] == (base | (1 << 3) | (1 << 1) | (1 << 2) | (1 << 5)) * 512


def test_partition_and_overlap_invariants():
    b = Band(Sphere(1.0), 0.1)
    dis = disjoint_subdomains(b, 8)
    allidx = np.sort(np.concatenate(dis))
    assert np.array_equal(allidx, np.arange(b.nA))
    assert max(len(d) for d in dis) - min(len(d) for d in dis) <= 1
    o2 = grow_overlap(b, dis[3], 2)
    o4 = grow_overlap(b, dis[3], 4)
    assert set(dis[3]).issubset(o2) and set(o2).issubset(o4)
    assert slab_bounds(10, 3) == [0, 3, 6, 10]


def test_overlap_equals_graph_distance_ball():
    """Reading R7 (-mesh_nover 4): S_j = the active nodes within
    lattice 6-neighbour graph distance N_O of S~_j, checked with an independent
    shortest-path computation (scipy.sparse.csgraph) on the active adjacency graph."""
    import scipy.sparse as sps
    from scipy.sparse.csgraph import shortest_path

    b = Band(Sphere(1.0), 0.2)
    key = {tuple(p): n for n, p in enumerate(b.active.tolist())}
    ri, ci = [], []
    for n, (i, j, k) in enumerate(b.active.tolist()):
        for d in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)):
            m = key.get((i + d[0], j + d[1], k + d[2]))
            if m is not None:
                ri.append(n)
                ci.append(m)
    G = sps.csr_matrix((np.ones(len(ri)), (ri, ci)), shape=(b.nA, b.nA))
    dis = disjoint_subdomains(b, 4)
    for s in (0, 2):
        D = shortest_path(G, unweighted=True, indices=dis[s]).min(axis=0)
        for layers in (0, 1, 2, 4):
            want = np.nonzero(D <= layers)[0]
            got = grow_overlap(b, dis[s], layers)
            assert np.array_equal(np.sort(got), want), (s, layers)


def test_ras_stationary_iteration_converges_to_solution():
    """Eq. 5-6 with Dirichlet transmission and exact local solves,
    iterated as a stationary method u^{n+1} = u^n + M (f - A u^n), converges to the
    single-domain solution A^{-1} f (restricted prolongation u^{n+1} = sum_j u_j|_{S~_j});
    an additive prolongation (sum over the overlapping S_j) over-corrects the overlap
    and does not."""
    b = Band(Sphere(1.0), 0.16)
    A = shifted_operator(b, 1.0)
    f = rhs_sph(b, 1.0, 3, 2)
    x = spla.spsolve(A.tocsc(), f)
    M = RAS(b, A, nsub=4, overlap=2, local="exact")
    u = np.zeros(b.nA)
    for _ in range(60):
        u = u + M(f - A @ u)
    assert np.abs(u - x).max() <= 1e-8 * np.abs(x).max()


def test_ras_single_subdomain_exact_is_inverse():
    b = Band(Sphere(1.0), 0.16)
    A = shifted_operator(b, 1.0)
    M = RAS(b, A, nsub=1, overlap=0, local="exact")
    f = rhs_sph(b, 1.0, 3, 2)
    x, st = gmres(lambda v: A @ v, f, restart=30, rtol=1e-10, M=M)
    assert st.iterations == 1


def test_ras_fgmres_converges_to_single_domain_solution():
    b = Band(Sphere(1.0), 0.1)
    A = shifted_operator(b, 1.0)
    f = rhs_sph(b, 1.0, 3, 2)
    x0, s0 = gmres(lambda v: A @ v, f, restart=30, rtol=1e-10)
    for local, k in (("exact", 0), ("gmres", 8)):
        M = RAS(b, A, nsub=8, overlap=4, k_inner=k, local=local)
        x1, s1 = gmres(lambda v: A @ v, f, restart=30, rtol=1e-10, M=M)
        assert s1.converged
        assert np.abs(x1 - x0).max() / np.abs(x0).max() < 1e-8


# ---------------------------------------------------------------- Schnakenberg IMEX (config 4)
from oracle.reaction import SchnakenbergParams, imex_step, initial_state, reaction  # noqa: E402


def test_schnakenberg_constant_state_is_scalar_euler():
    """Spatially constant data: Delta_S^h kills constants, so one IMEX step is the
    explicit Euler step of the kinetics ODE, u1 = u0 + dt gamma (a - u0 + u0^2 v0),
    v1 = v0 + dt gamma (b - u0^2 v0) (hand formula, not the oracle's)."""
    p = SchnakenbergParams()
    b = Band(Sphere(1.0), 0.15)
    u0, v0 = 0.7, 1.3
    u1, v1 = imex_step(b, np.full(b.nA, u0), np.full(b.nA, v0), p)
    eu = u0 + p.dt * p.gamma * (p.a - u0 + u0 * u0 * v0)
    ev = v0 + p.dt * p.gamma * (p.b - u0 * u0 * v0)
    assert np.abs(u1 - eu).max() <= 1e-10 and np.abs(v1 - ev).max() <= 1e-10


def test_schnakenberg_steady_state_is_fixed_point():
    """(a + b, b / (a + b)^2) zeroes both reaction terms: a step leaves it unchanged."""
    p = SchnakenbergParams()
    us, vs = p.a + p.b, p.b / (p.a + p.b) ** 2
    ru, rv = reaction(np.array([us]), np.array([vs]), p)
    assert abs(ru[0]) < 1e-14 and abs(rv[0]) < 1e-14
    b = Band(Sphere(1.0), 0.15)
    u1, v1 = imex_step(b, np.full(b.nA, us), np.full(b.nA, vs), p)
    assert np.abs(u1 - us).max() <= 1e-10 and np.abs(v1 - vs).max() <= 1e-10


def test_schnakenberg_pure_diffusion_eigenfunction():
    """gamma = 0, u0 = Y_2^1(cp): backward Euler multiplies by 1 / (1 + dt mu l(l+1))
    (Delta_S Y = -l(l+1) Y on the unit sphere), up to the O(h^2) of Delta_S^h."""
    p = SchnakenbergParams(gamma=0.0, mu1=1.0, mu2=2.0, dt=0.1)
    errs = []
    for h in (0.16, 0.1):
        b = Band(Sphere(1.0), h)
        Y = exact_sph(b, 2, 1)
        u1, v1 = imex_step(b, Y, Y, p)
        errs.append(max(np.abs(u1 - Y / (1 + 0.1 * 1.0 * 6)).max(), np.abs(v1 - Y / (1 + 0.1 * 2.0 * 6)).max()))
    assert errs[1] < 1e-2 and errs[0] / errs[1] > 0.8 * (0.16 / 0.1) ** 2


def test_schnakenberg_initial_state_recipe():
    """u = a + b, v = b/(a+b)^2 plus 1e-2 U[-1,1] (seed 3): bounds and independence of u, v noise."""
    p = SchnakenbergParams()
    b = Band(Sphere(1.0), 0.15)
    u, v = initial_state(b, p)
    assert np.all(np.abs(u - 1.0) <= 1e-2) and np.all(np.abs(v - 0.9) <= 1e-2)
    assert abs(np.corrcoef(u, v)[0, 1]) < 0.1
    # the state the noise is added to is the kinetics' fixed point (configs[4]: u = a + b,
    # v = b/(a+b)^2); with the default a + b = 1 the square cannot be seen, so a + b = 1.25
    q = SchnakenbergParams(a=0.25, b=1.0)
    u, v = initial_state(b, q)
    ru, rv = reaction(np.array([u.mean()]), np.array([v.mean()]), q)
    assert abs(ru[0]) < 5e-3 * q.gamma and abs(rv[0]) < 5e-3 * q.gamma
    assert abs(v.mean() - 0.64) < 1e-3


# ---------------------------------------------------------------- conventions found unpinned by tools/oracle_mutations.py
def test_real_sph_closed_forms_low_degree():
    """Reading R9 (real, orthonormal, +m = cos branch, -m = sin branch, no Condon-Shortley
    phase): the textbook Cartesian forms Y_1^1 = sqrt(3/4pi) x, Y_1^-1 = sqrt(3/4pi) y,
    Y_1^0 = sqrt(3/4pi) z, Y_2^2 = (1/4) sqrt(15/pi) (x^2 - y^2), Y_2^-2 = (1/2) sqrt(15/pi) x y,
    Y_2^1 = (1/2) sqrt(15/pi) x z on the unit sphere."""
    rng = np.random.default_rng(5)
    p = rng.normal(size=(200, 3))
    p /= np.linalg.norm(p, axis=1)[:, None]
    x, y, z = p.T
    c1 = math.sqrt(3.0 / (4.0 * math.pi))
    c2 = math.sqrt(15.0 / math.pi)
    for (l, m), want in {(1, 1): c1 * x, (1, -1): c1 * y, (1, 0): c1 * z, (2, 2): 0.25 * c2 * (x * x - y * y),
                         (2, -2): 0.5 * c2 * x * y, (2, 1): 0.5 * c2 * x * z}.items():
        assert np.allclose(real_sph(l, m, 3.0 * p), want, atol=1e-13), (l, m)


def test_torus_angles_invert_the_parametrisation():
    """Reading R10: ph = toroidal angle about the z axis, th = poloidal angle about the core
    circle.  Points built from ((R + r cos th) cos ph, (R + r cos th) sin ph, r sin th) give
    their angles back."""
    R, r = 1.0, 0.4
    th, ph = np.meshgrid(np.linspace(-3.0, 3.0, 13), np.linspace(-3.1, 3.1, 17), indexing="ij")
    th, ph = th.ravel(), ph.ravel()
    rho = R + r * np.cos(th)
    pts = np.stack([rho * np.cos(ph), rho * np.sin(ph), r * np.sin(th)], axis=1)
    th2, ph2 = torus_angles(pts, R)
    assert np.allclose(th2, th, atol=1e-12) and np.allclose(ph2, ph, atol=1e-12)


def test_rhs_torus_symmetries_and_zero_crossings():
    """configs[2]: f = cos(3 th) sin(2 ph) x modulation, modulation in [0.5, 1.5] (> 0), so
    the sign pattern of f is that of cos(3 th) sin(2 ph): odd under the quarter turn about z
    (ph -> ph + pi/2), even under z -> -z (th -> -th); 4 sign changes once around the outer
    equator (th = 0) and 6 once around the poloidal circle in the half plane x = y > 0."""
    h = 0.1
    b = Band(Torus(1.0, 0.4), h)
    ijk = b.active
    f = rhs_torus(b, 1, ijk)
    big = np.abs(f) > 0.05
    rot = np.stack([-ijk[:, 1], ijk[:, 0], ijk[:, 2]], axis=1)          # quarter turn about z
    refl = ijk * np.array([1, 1, -1])
    assert np.all(np.sign(rhs_torus(b, 1, rot)[big]) == -np.sign(f[big]))
    assert np.all(np.sign(rhs_torus(b, 1, refl)[big]) == np.sign(f[big]))
    assert 0.9 < np.abs(f).max() < 1.5

    def crossings(vals):
        sg = np.sign(vals[np.abs(vals) > 1e-6])
        return int(np.sum(sg != np.roll(sg, 1)))

    # outer equator: nodes of the plane z = 0 beyond the core circle by more than r/2
    rho = h * np.hypot(ijk[:, 0], ijk[:, 1])
    eq = (ijk[:, 2] == 0) & (rho > 1.0 + 0.2)
    order = np.argsort(np.arctan2(ijk[eq, 1], ijk[eq, 0]))
    assert crossings(f[eq][order]) == 4
    # poloidal circle: nodes of the half plane x = y > 0, ordered by their angle about the core circle
    pc = (ijk[:, 0] == ijk[:, 1]) & (ijk[:, 0] > 0)
    ang = np.arctan2(h * ijk[pc, 2], rho[pc] - 1.0)
    assert crossings(f[pc][np.argsort(ang)]) == 6


def test_rhs_noisy_sph_noise_level():
    """configs[3]: f = Y_10^5(cp(x)) + 1e-3 N(0,1): what is left after subtracting the
    harmonic has sample standard deviation 1e-3 (n ~ 1e4: +-1.5 %) and zero mean."""
    b = Band(Sphere(1.0), 0.1)
    d = rhs_noisy_sph(b, 10, 5, 2) - exact_sph(b, 10, 5)
    assert abs(d.std() / 1e-3 - 1.0) < 0.05 and abs(d.mean()) < 5e-5


def test_ras_subdomains_are_band_order_slabs():
    """Reading R8 (north_star 4: Morton-slab subdomains): subdomain s is the s-th contiguous
    range of the band order, so every band-order key of S~_s is below every key of S~_{s+1}."""
    b = Band(Sphere(1.0), 0.15)
    key = band_order_key(b.active)
    dis = disjoint_subdomains(b, 5)
    for s in range(4):
        assert key[dis[s]].max() < key[dis[s + 1]].min()


def test_arnoldi_fixed_happy_breakdown():
    """Reading R6: k GMRES steps stop early only on happy breakdown, and then the iterate is
    exact on the invariant subspace reached.  A = diag(2, 3, 5, 7): b = 4 e_1 spans a
    1-dimensional Krylov space (z = b/3 after one column), b = e_0 + e_2 a 2-dimensional
    one (z = (1/2, 0, 1/5, 0) after two)."""
    d = np.array([2.0, 3.0, 5.0, 7.0])
    A = lambda v: d * v  # noqa: E731
    z = arnoldi_fixed(A, np.array([0.0, 4.0, 0.0, 0.0]), 3)
    assert np.allclose(z, [0.0, 4.0 / 3.0, 0.0, 0.0], atol=1e-15)
    z = arnoldi_fixed(A, np.array([1.0, 0.0, 1.0, 0.0]), 4)
    assert np.allclose(z, [0.5, 0.0, 0.2, 0.0], atol=1e-14)


def test_gmres_initial_guess():
    """x0 is the starting iterate (restarted GMRES; cpm_solve's `u holds x0 on
    entry`): started at the solution GMRES returns it after 0 iterations; started elsewhere
    it still converges to the same solution, in fewer iterations from a nearby guess than
    from zero."""
    rng = np.random.default_rng(11)
    M = np.eye(30) * 4.0 + rng.normal(size=(30, 30)) * 0.3
    xs = rng.normal(size=30)
    b = M @ xs
    A = lambda v: M @ v  # noqa: E731
    x, st = gmres(A, b, x0=xs, restart=10, rtol=1e-12)
    assert st.iterations == 0 and st.converged and np.array_equal(x, xs)
    x0, st0 = gmres(A, b, restart=10, rtol=1e-12)
    x1, st1 = gmres(A, b, x0=xs + 1e-6 * rng.normal(size=30), restart=10, rtol=1e-12)
    assert st0.converged and st1.converged
    assert np.allclose(x0, xs, atol=1e-9) and np.allclose(x1, xs, atol=1e-9)
    assert st1.iterations < st0.iterations


def test_rhs_torus_modulation_worked_point():
    """Reading R10 (the input recipe of configs[2]): f = cos(3 th) sin(2 ph) (1 + sum_q a_q
    sin(k_q . cp)).  A lattice node on the diagonal x = y of the plane z = 0 outside the
    torus has cp = ((R + r)/sqrt2, (R + r)/sqrt2, 0), th = 0, ph = pi/4, so f is the
    modulation itself at that point, evaluated here from the coefficient table."""
    h = 0.1
    b = Band(Torus(1.0, 0.4), h)
    node = np.array([[11, 11, 0]])                     # |x| = 1.556 > R + r: outside, th = 0
    assert b.index_active(node)[0] >= 0
    s = 1.4 / math.sqrt(2.0)
    want = 1.0 + sum(a * math.sin((kx + ky) * s) for a, kx, ky, kz in seeded_inputs.smooth_modulation_coeffs(1))
    assert abs(want - 1.0) > 1e-3                      # the modulation is visible at this point
    assert abs(rhs_torus(b, 1, node)[0] - want) < 1e-13


def test_ras_inexact_local_solve_takes_k_steps():
    """north_star 4 / reading R6: the local solve is exactly k_inner GMRES steps from zero.
    With one subdomain and no overlap M(r) is that iterate for A z = r, so ||r - A M(r)||
    equals the least-squares minimum over span{r, A r, ..., A^(k-1) r} (explicit basis,
    independent lstsq) and is larger than the minimum over k + 1 vectors."""
    b = Band(Sphere(1.0), 0.16)
    A = shifted_operator(b, 1.0)
    r = seeded_inputs.uniform_pm1(4, b.active)
    k = 5
    z = RAS(b, A, nsub=1, overlap=0, k_inner=k, local="gmres")(r)
    res = np.linalg.norm(r - A @ z)

    def krylov_min(m):
        K = [r / np.linalg.norm(r)]
        for _ in range(m - 1):
            v = A @ K[-1]
            K.append(v / np.linalg.norm(v))
        AK = np.stack([A @ v for v in K], axis=1)
        y, *_ = np.linalg.lstsq(AK, r, rcond=None)
        return np.linalg.norm(r - AK @ y)

    mk, mk1 = krylov_min(k), krylov_min(k + 1)
    assert mk1 < 0.99 * mk                      # the two are distinguishable
    assert abs(res - mk) <= 1e-9 * mk
