"""CPU tier: the multi-GPU exchange logic of paper_2510_01592_b200.slabs
(DistComm) with world_size 2 and 3 over gloo, checked against LocalComm (the
single-process virtual-slab exchanges) on the same data: halo planes land on
the neighbours' halo planes, plane counts and boundary triples are
all-gathered in slab order, the steppable halo lists fill every slab's
extended list, cluster members reach their owner in slab order, polygons are
gathered to rank 0 in slab order."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_01592_b200.slabs import MEMBER_REC_BYTES, DistComm, LocalComm, SlabLayout, split_x

EX = 12
W = 2


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


def plane_counts():
    return (np.arange(EX) * 7 % 5).astype(np.int32)


def ranges_for(world):
    return split_x(EX, world) if world < 3 else [(0, 5), (5, 6), (6, 12)]  # a slab thinner than W


def ext_lists(layout, k):
    """Extended list of slab k with only the own part filled: entry bytes = global ordinal."""
    lists = []
    for w in (12, 24, 24):
        t = torch.zeros(layout.n_ext(k) * w, dtype=torch.uint8)
        a, _ = layout.ranges[k]
        nl = layout.n_left(k)
        for j in range(layout.n_own(k)):
            o = int(layout.P[a]) + j
            t[(nl + j) * w:(nl + j + 1) * w] = (o * 3 + w) % 251
        lists.append(t)
    return lists


def triples_of(k):
    return torch.arange(3 * (k + 1), dtype=torch.int32).view(-1, 3) + 100 * k


def exports_of(layout, k):
    """Slab k sends (k - d) records to every lower slab d, tagged (k, d, i)."""
    counts = np.array([k - d if d < k else 0 for d in range(layout.n)], np.int64)
    rec = torch.zeros(int(counts.sum()) * MEMBER_REC_BYTES, dtype=torch.uint8)
    o = 0
    for d in range(layout.n):
        for i in range(int(counts[d])):
            rec[o * MEMBER_REC_BYTES:(o + 1) * MEMBER_REC_BYTES] = 10 * k + d + i
            o += 1
    return counts, rec


def run_exchanges(comm, slab_ids, world):
    layout = SlabLayout(ranges_for(world), plane_counts(), W)
    pc = plane_counts()
    counts = comm.allgather_plane_counts([torch.as_tensor(pc[a:b]) for a, b in
                                          [layout.ranges[k] for k in slab_ids]])
    ext = [ext_lists(layout, k) for k in slab_ids]
    comm.exchange_steppable(layout, ext)
    tri = comm.allgather_triples([triples_of(k) for k in slab_ids])
    recv = comm.exchange_members([exports_of(layout, k) for k in slab_ids])
    polys = comm.gather_polygons([[{"label": 100 * k + j} for j in range(k + 1)] for k in slab_ids])
    return {"counts": counts.tolist(), "ext": {k: [t.tolist() for t in e] for k, e in zip(slab_ids, ext)},
            "triples": tri.tolist(), "recv": {k: (r.tolist() if r is not None else None, n)
                                              for k, (r, n) in zip(slab_ids, recv)},
            "polys": polys}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = DistComm(dist, device=None)
        a, b = ranges_for(world)[rank]
        s = FakeSlab(rank, a, b)
        comm.halo_exchange([s])
        res = {}
        if rank > 0:
            res["left_halo"] = s.plane(a - 1)[0][0].item()
            res["left_bits"] = s.plane(a - 1)[1][0].item()
        if rank + 1 < world:
            res["right_halo"] = s.plane(b)[0][0].item()
        pts = torch.arange(9, dtype=torch.float32) if rank == 0 else torch.zeros(3, dtype=torch.float32)
        res["frame"] = comm.broadcast_frame(pts).tolist()
        res["ex"] = run_exchanges(comm, [rank], world)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_dist_comm_gloo_matches_local(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    rg = ranges_for(world)
    for r in range(world):
        a, b = rg[r]
        if r + 1 < world:
            assert out[r]["right_halo"] == (r + 2) * 16 + (b % 16)   # neighbour's plane x=b
        if r > 0:
            assert out[r]["left_halo"] == r * 16 + ((a - 1) % 16)     # neighbour's plane x=a-1
            assert out[r]["left_bits"] == (a - 1) % 251
        assert out[r]["frame"] == list(range(9))
    local = run_exchanges(LocalComm(world), list(range(world)), world)
    layout = SlabLayout(rg, plane_counts(), W)
    # every extended list is completely filled with the right global ordinals
    for k in range(world):
        for w, t in zip((12, 24, 24), local["ext"][k]):
            lo, _ = layout.ext(k)
            exp = [((int(layout.P[lo]) + e) * 3 + w) % 251 for e in range(layout.n_ext(k)) for _ in range(w)]
            assert t == exp
    for r in range(world):
        d = out[r]["ex"]
        assert d["counts"] == local["counts"] == plane_counts().tolist()
        assert d["ext"][r] == local["ext"][r]
        assert d["triples"] == local["triples"]
        assert d["recv"][r] == local["recv"][r]
    # members from higher slabs in slab order
    for d in range(world):
        rv, n = local["recv"][d]
        assert n == sum(k - d for k in range(d + 1, world))
    assert out[0]["ex"]["polys"] == local["polys"] == [{"label": 100 * k + j} for k in range(world)
                                                       for j in range(k + 1)]


def test_split_x_covers_window():
    for ex in (1, 7, 500, 2000):
        for w in (1, 2, 3, 8):
            if w > ex:
                continue
            r = split_x(ex, w)
            assert r[0][0] == 0 and r[-1][1] == ex
            assert all(a < b for a, b in r) and all(r[i][1] == r[i + 1][0] for i in range(w - 1))
