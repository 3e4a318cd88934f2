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
