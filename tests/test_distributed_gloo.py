"""Host logic of the multi-GPU path on CPU: world_size-2 gloo process group.
Checks the request all_to_all (who sends what to whom), slab bounds and the
NCCL-id broadcast plumbing — everything except the NCCL transport itself."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


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
        from paper_2110_06322_b200.distributed import (broadcast_uid, exchange_requests, request_counts,
                                                       slab_bounds)

        n = 1000
        bounds = slab_bounds(n, world)
        # synthetic halos: every rank asks for the 3 nodes on each side of its slab
        lo, hi = bounds[rank], bounds[rank + 1]
        halo = np.array(sorted({i for i in list(range(lo - 3, lo)) + list(range(hi, hi + 3)) if 0 <= i < n}),
                        dtype=np.int64)
        send, counts = exchange_requests(halo, bounds)
        uid = broadcast_uid(bytes(range(128)) if rank == 0 else None)
        q.put((rank, halo.tolist(), send.tolist(), counts.tolist(), request_counts(halo, bounds).tolist(),
               uid == bytes(range(128))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_requests_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, halo, send, counts, rc, uid_ok = q.get(timeout=120)
        res[r] = (halo, send, counts, rc, uid_ok)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2110_06322_b200.distributed import owners, slab_bounds

    bounds = slab_bounds(1000, world)
    for r in range(world):
        halo, send, counts, rc, uid_ok = res[r]
        assert uid_ok
        assert sum(counts) == len(send)
        # what r sends to q == what q requested from r, in q's order
        off = 0
        for qq in range(world):
            req = [a for a in res[qq][0] if owners(np.array([a]), bounds)[0] == r]
            assert send[off: off + counts[qq]] == req
            off += counts[qq]
        assert rc[r] == 0


def test_slab_bounds_match_oracle():
    from oracle.order import slab_bounds as osb
    from paper_2110_06322_b200.distributed import slab_bounds

    for n, R in [(10, 3), (4146590, 8), (7, 7)]:
        assert slab_bounds(n, R).tolist() == osb(n, R)


def _transport_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2110_06322_b200.distributed import host_transport_fns

        ar, a2a = host_transport_fns()
        buf = np.arange(5, dtype=np.float64) * (rank + 1)
        ar(buf)
        # rank r sends (r + 1) * 10 + q, repeated q + 1 times, to rank q != r
        sc = np.array([0 if q_ == rank else q_ + 1 for q_ in range(world)], dtype=np.int64)
        rc = np.array([0 if q_ == rank else rank + 1 for q_ in range(world)], dtype=np.int64)
        send = np.concatenate([np.full(sc[q_], (rank + 1) * 10.0 + q_) for q_ in range(world)])
        recv = np.empty(int(rc.sum()))
        a2a(send, sc, recv, rc)
        q.put((rank, buf.tolist(), recv.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_host_transport_callbacks_gloo(world):
    """The callbacks behind cpm_comm_init_host (distributed.host_transport_fns):
    in-place sum over the ranks, and the rank-ordered alltoallv blocks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_transport_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, buf, recv = q.get(timeout=120)
        res[r] = (buf, recv)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    tot = sum(r + 1 for r in range(world))
    for r in range(world):
        buf, recv = res[r]
        assert buf == [float(i * tot) for i in range(5)]
        want = []
        for src in range(world):
            if src != r:
                want += [(src + 1) * 10.0 + r] * (r + 1)
        assert recv == want
