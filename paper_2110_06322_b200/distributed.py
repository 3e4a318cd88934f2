"""Multi-GPU plumbing (north_star item 5): one process per GPU, torch.distributed
for the set-up exchange, NCCL (inside libcpm.so) for the per-apply halo exchange
and the Krylov allreduces.

Set-up (once): every rank builds the same band, then its Morton-slab partition
(`cpm_part_create`).  A rank knows which halo nodes it RECEIVES (its sorted halo
list, grouped by owner); the owners learn what to SEND through one all_to_all of
the request lists (`exchange_requests`, host logic, any torch.distributed backend
— tested with gloo on CPU).  Rank 0's NCCL unique id is broadcast the same way.
"""
from __future__ import annotations

import numpy as np


def slab_bounds(n: int, nranks: int) -> np.ndarray:
    """Band-order slab bounds [floor(r n / R)] (reading R8), length nranks + 1."""
    return np.array([(r * n) // nranks for r in range(nranks + 1)], dtype=np.int64)


def owners(idx: np.ndarray, bounds: np.ndarray) -> np.ndarray:
    return np.searchsorted(bounds, idx, side="right") - 1


def request_counts(halo: np.ndarray, bounds: np.ndarray) -> np.ndarray:
    """How many of this rank's halo nodes each rank owns (halo sorted ascending)."""
    nr = len(bounds) - 1
    if halo.size and np.any(np.diff(halo) <= 0):
        raise ValueError("halo list must be strictly increasing")
    return np.bincount(owners(halo, bounds), minlength=nr).astype(np.int64)


def exchange_requests(halo: np.ndarray, bounds: np.ndarray, group=None):
    """all_to_all of halo requests -> (send_global, send_counts) for this rank.

    send_global lists, peer by peer in rank order, the owned global indices each
    peer requested, in that peer's halo order (= its receive order)."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    nr = dist.get_world_size(group)
    recv_counts = request_counts(halo, bounds)
    if recv_counts[rank] != 0:
        raise ValueError("a rank cannot request its own nodes")
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    rc = torch.from_numpy(recv_counts).to(dev)
    sc = torch.empty_like(rc)
    dist.all_to_all_single(sc, rc, group=group)
    send_counts = sc.cpu().numpy().astype(np.int64)
    src = torch.from_numpy(np.ascontiguousarray(halo, dtype=np.int64)).to(dev)
    dst = torch.empty(int(send_counts.sum()), dtype=torch.int64, device=dev)
    dist.all_to_all_single(dst, src, output_split_sizes=send_counts.tolist(),
                           input_split_sizes=recv_counts.tolist(), group=group)
    return dst.cpu().numpy(), send_counts


def broadcast_uid(uid: bytes | None, group=None) -> bytes:
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.zeros(128, dtype=torch.uint8, device=dev)
    if uid is not None:
        t.copy_(torch.frombuffer(bytearray(uid), dtype=torch.uint8))
    dist.broadcast(t, src=0, group=group)
    return bytes(t.cpu().numpy().tobytes())


def host_transport_fns(group=None):
    """(allreduce_sum, alltoallv) over a torch.distributed group on host tensors (gloo):
    the callbacks of cpm_comm_init_host (include/cpm.h)."""
    import torch
    import torch.distributed as dist

    def allreduce_sum(buf):
        t = torch.from_numpy(buf)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    def alltoallv(send, send_counts, recv, recv_counts):
        dist.all_to_all_single(torch.from_numpy(recv), torch.from_numpy(send),
                               output_split_sizes=[int(c) for c in recv_counts],
                               input_split_sizes=[int(c) for c in send_counts], group=group)

    return allreduce_sum, alltoallv


class DistributedCPM:
    """This rank's slab of a band, its communicator and the distributed ops.

    transport="nccl": NCCL inside libcpm.so (one GPU per rank); transport="host": the
    host-staged transport over `group` (gloo), which runs several ranks as processes
    sharing one GPU."""

    def __init__(self, band, group=None, transport="nccl"):
        import torch.distributed as dist

        from . import cpm

        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        self.band = band
        self.part = cpm.cpm_part_create(band, self.rank, self.nranks)
        bounds = slab_bounds(band.n, self.nranks)
        assert bounds[self.rank] == self.part.lo and bounds[self.rank + 1] == self.part.hi
        halo = cpm.cpm_part_halo_nodes(self.part)
        send, counts = exchange_requests(halo, bounds, group)
        cpm.cpm_part_set_send(self.part, send, counts)
        if transport == "host":
            ar, a2a = host_transport_fns(group)
            self.comm = cpm.cpm_comm_init_host(ar, a2a, self.rank, self.nranks)
        elif transport == "nccl":
            uid = cpm.cpm_comm_unique_id() if self.rank == 0 else None
            uid = broadcast_uid(uid, group)
            self.comm = cpm.cpm_comm_init(uid, self.rank, self.nranks)
        else:
            raise ValueError(f"unknown transport {transport!r}")

    @property
    def lo(self):
        return self.part.lo

    @property
    def hi(self):
        return self.part.hi

    def apply(self, c, u_owned, y_owned):
        from . import cpm

        return cpm.cpm_part_apply(self.part, self.comm, c, u_owned, y_owned)

    def setup_ras(self, n_sub, overlap, k_inner, c, group=None):
        """This rank's RAS subdomains (n_sub a multiple of the rank count) and the
        exchange plan of its RAS halo (the overlap reaching into other slabs)."""
        from . import cpm

        ras = cpm.cpm_part_ras_setup(self.part, n_sub, overlap, k_inner, c)
        halo = cpm.cpm_ras_halo_nodes(ras)
        send, counts = exchange_requests(halo, slab_bounds(self.band.n, self.nranks), group)
        cpm.cpm_ras_set_send(ras, send, counts)
        return ras

    def rd_step(self, u_owned, v_owned, **params):
        """One partitioned Schnakenberg IMEX step (cpm_part_rd_step) on the owned slices."""
        from . import cpm

        return cpm.cpm_part_rd_step(self.part, self.comm, u_owned, v_owned, **params)

    def solve(self, c, f_owned, u_owned, rtol=1e-10, restart=50, maxit=100000, ras=None):
        from . import cpm

        return cpm.cpm_part_solve(self.part, self.comm, c, f_owned, u_owned, rtol, restart, maxit, ras=ras)
