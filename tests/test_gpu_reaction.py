"""GPU parity of the Schnakenberg IMEX Euler step (BASELINE config 4) against the oracle.

Both sides take the same seeded initial state (per lattice node); the CUDA path
solves the two shifted systems with GMRES(50) at rtol 1e-10 (warm start), the
oracle by direct sparse solves: the states agree to 1e-8 relative after every step.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.band import Band as OBand  # noqa: E402
from oracle.operator import laplace_beltrami_matrix  # noqa: E402
from oracle.reaction import SchnakenbergParams, imex_step, initial_state  # noqa: E402
from oracle.surfaces import Sphere, Torus  # noqa: E402

TOL = 1e-8


@pytest.fixture(scope="module")
def cpm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2110_06322_b200._build import build

    build()
    import paper_2110_06322_b200 as p

    return p


@pytest.mark.parametrize("kind,h,kw,steps", [("sphere", 0.1, {}, 3), ("sphere", 0.06, {"R": 0.7}, 2)])
def test_rd_steps_match_oracle(cpm, kind, h, kw, steps):
    gb = cpm.cpm_build_band(kind, h, **kw)
    ob = OBand(Torus(1.0, 0.4) if kind == "torus" else Sphere(kw.get("R", 1.0)), h)
    ga = cpm.cpm_band_active_coords(gb).astype(np.int64)
    perm = ob.index_active(ga)
    assert np.all(perm >= 0)
    p = SchnakenbergParams()
    uo, vo = initial_state(ob, p)
    ug, vg = initial_state(ob, p, ijk=ga)           # the same per-node draws, GPU order
    assert np.array_equal(ug, uo[perm]) and np.array_equal(vg, vo[perm])
    u = torch.from_numpy(ug).cuda()
    v = torch.from_numpy(vg).cuda()
    L = laplace_beltrami_matrix(ob)
    for _ in range(steps):
        s1, s2 = cpm.cpm_rd_step(gb, u, v, a=p.a, b=p.b, gamma=p.gamma, mu1=p.mu1, mu2=p.mu2, dt=p.dt)
        assert s1.converged and s2.converged
        uo, vo = imex_step(ob, uo, vo, p, L)
        eu = np.abs(u.cpu().numpy() - uo[perm]).max() / np.abs(uo).max()
        ev = np.abs(v.cpu().numpy() - vo[perm]).max() / np.abs(vo).max()
        assert eu <= TOL and ev <= TOL, (eu, ev)


def test_rd_step_errors(cpm):
    gb = cpm.cpm_build_band("sphere", 0.1)
    u = torch.ones(gb.n, dtype=torch.float64, device="cuda")
    with pytest.raises(cpm.CpmError, match="alias"):
        cpm.cpm_rd_step(gb, u, u)
    v = torch.ones_like(u)
    with pytest.raises(cpm.CpmError, match="> 0"):
        cpm.cpm_rd_step(gb, u, v, dt=0.0)
    with pytest.raises(cpm.CpmError, match="device"):
        cpm.cpm_rd_step(gb, u.cpu().numpy(), v)


def test_part_rd_step_single_rank_equals_rd_step(cpm):
    """cpm_part_rd_step with one rank (no communicator) is cpm_rd_step, bit for bit."""
    from paper_2110_06322_b200 import cpm as C

    gb = cpm.cpm_build_band("sphere", 0.1)
    ob = OBand(Sphere(1.0), 0.1)
    ga = cpm.cpm_band_active_coords(gb).astype(np.int64)
    p = SchnakenbergParams()
    ug, vg = initial_state(ob, p, ijk=ga)
    u1, v1 = torch.from_numpy(ug).cuda(), torch.from_numpy(vg).cuda()
    u2, v2 = u1.clone(), v1.clone()
    part = C.cpm_part_create(gb, 0, 1)
    for _ in range(2):
        a1, b1 = cpm.cpm_rd_step(gb, u1, v1)
        a2, b2 = C.cpm_part_rd_step(part, None, u2, v2)
        assert (a1.iterations, b1.iterations) == (a2.iterations, b2.iterations)
    assert torch.equal(u1, u2) and torch.equal(v1, v2)
