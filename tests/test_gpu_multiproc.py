"""The partitioned data plane run as SEVERAL PROCESSES (ranks) sharing one GPU,
through the host-staged transport (cpm_comm_init_host over a gloo group): every
halo exchange (operator and RAS overlap) and every Krylov allreduce of
cpm_part_apply / cpm_part_solve / cpm_part_ras_* goes between processes, exactly
the code path NCCL takes on a multi-GPU node except the NCCL calls themselves
(NCCL refuses two ranks on one device).  Checked against the single-process
cpm_apply / cpm_solve on the same band (VERDICT r1 missing #5)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import seeded_inputs
        import paper_2110_06322_b200 as cpm
        from paper_2110_06322_b200.distributed import DistributedCPM

        c = 1.0
        band = cpm.cpm_build_band("torus", 0.06, R=1.0, r=0.4)
        ga = cpm.cpm_band_active_coords(band).astype(np.int64)
        D = DistributedCPM(band, transport="host")
        lo, hi = D.lo, D.hi
        res = {"rank": rank, "lo": lo, "hi": hi}
        # one apply
        u = torch.from_numpy(seeded_inputs.uniform_pm1(0, ga)).cuda()
        yo = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
        D.apply(c, u[lo:hi].contiguous(), yo)
        res["y"] = yo.cpu().numpy()
        # plain GMRES(30) and RAS-FGMRES(30) (8 subdomains, overlap 4, 6 inner steps)
        f = torch.empty(band.n, dtype=torch.float64, device="cuda")
        cpm.cpm_eval_torus_rhs(band, seeded_inputs.smooth_modulation_coeffs(1), f)
        fo = f[lo:hi].contiguous()
        uo = torch.zeros_like(fo)
        st = D.solve(c, fo, uo, rtol=1e-10, restart=30)
        res["plain"] = (uo.cpu().numpy(), st.iterations, st.converged)
        ras = D.setup_ras(8, 4, 6, c)
        zr = torch.empty_like(fo)
        from paper_2110_06322_b200 import cpm as C

        C.cpm_part_ras_apply(ras, D.comm, fo, zr)
        res["z"] = zr.cpu().numpy()
        uo.zero_()
        st = D.solve(c, fo, uo, rtol=1e-10, restart=30, ras=ras)
        res["ras"] = (uo.cpu().numpy(), st.iterations, st.converged)
        # two partitioned Schnakenberg IMEX steps (config 4) on a sphere band
        from oracle.band import Band as OBand  # test infrastructure: the seeded initial state
        from oracle.reaction import SchnakenbergParams, initial_state
        from oracle.surfaces import Sphere

        sb = cpm.cpm_build_band("sphere", 0.1)
        sga = cpm.cpm_band_active_coords(sb).astype(np.int64)
        Ds = DistributedCPM(sb, transport="host")
        prm = SchnakenbergParams()
        ug, vg = initial_state(OBand(Sphere(1.0), 0.1), prm, ijk=sga)
        uu = torch.from_numpy(ug[Ds.lo:Ds.hi].copy()).cuda()
        vv = torch.from_numpy(vg[Ds.lo:Ds.hi].copy()).cuda()
        rd = []
        for _ in range(2):
            s1, s2 = Ds.rd_step(uu, vv, a=prm.a, b=prm.b, gamma=prm.gamma, mu1=prm.mu1, mu2=prm.mu2, dt=prm.dt)
            rd.append((uu.cpu().numpy().copy(), vv.cpu().numpy().copy(), s1.converged and s2.converged))
        res["rd"] = rd
        torch.cuda.synchronize()
        q.put(res)
    except Exception as e:  # pragma: no cover
        import traceback

        q.put({"rank": rank, "error": traceback.format_exc() + str(e)})
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def reference():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2110_06322_b200._build import build

    build()
    import seeded_inputs
    import paper_2110_06322_b200 as cpm

    c = 1.0
    band = cpm.cpm_build_band("torus", 0.06, R=1.0, r=0.4)
    ga = cpm.cpm_band_active_coords(band).astype(np.int64)
    u = torch.from_numpy(seeded_inputs.uniform_pm1(0, ga)).cuda()
    y = torch.empty_like(u)
    cpm.cpm_apply(band, c, u, y)
    f = torch.empty_like(u)
    cpm.cpm_eval_torus_rhs(band, seeded_inputs.smooth_modulation_coeffs(1), f)
    x = torch.zeros_like(u)
    st = cpm.cpm_solve(band, c, f, x, rtol=1e-10, restart=30)
    ras = cpm.cpm_ras_setup(band, 8, 4, 6, c)
    z = torch.empty_like(u)
    cpm.cpm_ras_apply(ras, f, z)
    xr = torch.zeros_like(u)
    sr = cpm.cpm_solve(band, c, f, xr, rtol=1e-10, restart=30, ras=ras)
    torch.cuda.synchronize()
    return dict(y=y.cpu().numpy(), x=x.cpu().numpy(), its=st.iterations, z=z.cpu().numpy(),
                xr=xr.cpu().numpy(), its_r=sr.iterations)


@pytest.mark.parametrize("world", [2, 4])
def test_partitioned_path_across_processes(reference, world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            r = q.get(timeout=600)
            assert "error" not in r, r.get("error")
            res[r["rank"]] = r
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.exitcode is None:
                p.kill()
    for p in procs:
        assert p.exitcode == 0
    ref = reference
    y = np.concatenate([res[r]["y"] for r in range(world)])
    assert np.array_equal(y, ref["y"])                      # the partitioned operator is bit-exact
    z = np.concatenate([res[r]["z"] for r in range(world)])
    assert np.abs(z - ref["z"]).max() <= 1e-12 * np.abs(ref["z"]).max()
    # the partitioned IMEX steps against the oracle (1e-8 per step)
    from oracle.band import Band as OBand
    from oracle.operator import laplace_beltrami_matrix
    from oracle.reaction import SchnakenbergParams, imex_step, initial_state
    from oracle.surfaces import Sphere
    import paper_2110_06322_b200 as cpm

    ob = OBand(Sphere(1.0), 0.1)
    sb = cpm.cpm_build_band("sphere", 0.1)
    perm = ob.index_active(cpm.cpm_band_active_coords(sb).astype(np.int64))
    prm = SchnakenbergParams()
    uo, vo = initial_state(ob, prm)
    L = laplace_beltrami_matrix(ob)
    for step in range(2):
        uo, vo = imex_step(ob, uo, vo, prm, L)
        ug = np.concatenate([res[r]["rd"][step][0] for r in range(world)])
        vg = np.concatenate([res[r]["rd"][step][1] for r in range(world)])
        assert all(res[r]["rd"][step][2] for r in range(world))
        assert np.abs(ug - uo[perm]).max() <= 1e-8 * np.abs(uo).max()
        assert np.abs(vg - vo[perm]).max() <= 1e-8 * np.abs(vo).max()
    for key, xk, itk in (("plain", "x", "its"), ("ras", "xr", "its_r")):
        x = np.concatenate([res[r][key][0] for r in range(world)])
        its = {res[r][key][1] for r in range(world)}
        assert len(its) == 1                                   # every rank took the same decisions
        assert all(res[r][key][2] for r in range(world))
        assert abs(its.pop() - ref[itk]) <= 1, key
        assert np.abs(x - ref[xk]).max() <= 1e-9 * np.abs(ref[xk]).max(), key
