"""CPU tier: the multi-GPU exchange logic of paper_2510_01592_b200.slabs
(DistComm) with world_size 2 over gloo: halo planes land on the neighbour's
halo planes, the steppable lists are gathered to rank 0 in slab order."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_01592_b200.slabs import DistComm, split_x


class FakeSlab:
    """CPU stand-in: planes are byte tensors, one per window x."""

    def __init__(self, rank, x_begin, x_end, plane_bytes=48, bits_bytes=8):
        self.x_begin, self.x_end = x_begin, x_end
        self.planes = {x: (torch.full((plane_bytes,), (rank + 1) * 16 + (x % 16), dtype=torch.uint8)
                           if x_begin <= x < x_end else torch.zeros(plane_bytes, dtype=torch.uint8),
                           torch.full((bits_bytes,), x % 251, dtype=torch.uint8)
                           if x_begin <= x < x_end else torch.zeros(bits_bytes, dtype=torch.uint8))
                       for x in range(x_begin - 1, x_end + 1)}

    def plane(self, x):
        return self.planes[x]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ranges = split_x(10, world)
        a, b = ranges[rank]
        s = FakeSlab(rank, a, b)
        comm = DistComm(dist, device=None)
        comm.halo_exchange([s])
        res = {}
        if rank > 0:
            res["left_halo"] = s.plane(a - 1)[0][0].item()
            res["left_bits"] = s.plane(a - 1)[1][0].item()
        if rank + 1 < world:
            res["right_halo"] = s.plane(b)[0][0].item()
        # gather: rank r contributes r+1 entries
        n = rank + 1
        arrs = (torch.full((12 * n,), rank, dtype=torch.uint8), torch.full((24 * n,), 10 + rank, dtype=torch.uint8),
                torch.full((24 * n,), 20 + rank, dtype=torch.uint8))
        total, idx, mean, nrm = comm.gather_steppable([(n, arrs)])
        res["total"] = total
        if rank == 0:
            res["idx"] = idx.tolist()
            res["mean_first"] = mean[0].item()
            res["mean_last"] = mean[-1].item()
        pts = torch.arange(9, dtype=torch.float32) if rank == 0 else torch.zeros(3, dtype=torch.float32)
        res["frame"] = comm.broadcast_frame(pts).tolist()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_dist_comm_world2_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    # split_x(10, 2) = [(0,5), (5,10)]
    assert out[0]["right_halo"] == (1 + 1) * 16 + 5      # rank 1's plane x=5
    assert out[1]["left_halo"] == (0 + 1) * 16 + 4       # rank 0's plane x=4
    assert out[1]["left_bits"] == 4
    assert out[0]["total"] == out[1]["total"] == 3
    assert out[0]["idx"] == [0] * 12 + [1] * 24
    assert out[0]["mean_first"] == 10 and out[0]["mean_last"] == 11
    assert out[0]["frame"] == out[1]["frame"] == list(range(9))


def test_split_x_covers_window():
    for ex in (1, 7, 500, 2000):
        for w in (1, 2, 3, 8):
            if w > ex:
                continue
            r = split_x(ex, w)
            assert r[0][0] == 0 and r[-1][1] == ex
            assert all(a < b for a, b in r) and all(r[i][1] == r[i + 1][0] for i in range(w - 1))
