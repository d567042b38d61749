"""Spatial-slab decomposition of one large window across GPUs.

The window is split along x (the most significant axis of the reference's
flat index, voxel_grid.hpp:43-46), one slab per rank. Per frame:

1. every rank receives the frame (broadcast from rank 0);
2. clear_rays + integrate_frame on every slab (library): rays are clipped to
   the whole window and walked from their start with the reference's DDA, and
   only owned cells / points are kept -- bit-identical to one big grid;
3. halo exchange: each slab's first / last owned x-plane (cells + occupancy
   bits) is sent onto the halo planes of its neighbours (the 1-cell window of
   estimate_normals, segmentation.cpp:36-51);
4. estimate_normals + classify_steppable on owned voxels (library);
5. the steppable lists are gathered to rank 0 in slab order -- ordinals are
   x-major, so the concatenation IS the single-grid list -- and rank 0 runs
   build_adjacency .. make_polygon (vp_segment_steppable).

The same phase functions drive N virtual slabs in one process (LocalComm,
exchange = device copies; used by the single-GPU parity tests) or one slab
per rank under torch.distributed (DistComm: NCCL send/recv of the halo
planes, gather of the steppable lists).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import native
from .native import _p, _pose, check, lib, polygons_to_py


class DeviceBuffer:
    """Zero-copy torch view of library-owned device memory."""

    def __init__(self, ptr: int, nbytes: int, device: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}
        self.device = device

    def tensor(self):
        import torch
        return torch.as_tensor(self, device=f"cuda:{self.device}")


def split_x(extent_x: int, world: int):
    """Balanced contiguous x ranges [(x_begin, x_end)] for `world` slabs."""
    base, rem = divmod(extent_x, world)
    out, x = [], 0
    for r in range(world):
        w = base + (1 if r < rem else 0)
        out.append((x, x + w))
        x += w
    return out


class Slab:
    """One slab grid (vp_slab_create) owning window x in [x_begin, x_end)."""

    def __init__(self, res, window_extent, center, x_begin, x_end, device=0):
        ext = np.asarray(window_extent, np.int32)
        c = np.asarray(center, np.float64)
        self.h = C.c_void_p()
        self.x_begin, self.x_end, self.device = x_begin, x_end, device
        self.window_extent = tuple(int(v) for v in window_extent)
        check(lib().vp_slab_create(C.c_double(res), _p(ext, C.c_int32), _p(c, C.c_double),
                                   C.c_int32(x_begin), C.c_int32(x_end), C.c_int(device), C.byref(self.h)))

    def plane(self, window_x):
        cells, cb, bits, bb = C.c_void_p(), C.c_uint64(), C.c_void_p(), C.c_uint64()
        check(lib().vp_grid_plane(self.h, C.c_int32(window_x), C.byref(cells), C.byref(cb), C.byref(bits),
                                  C.byref(bb)))
        return (DeviceBuffer(cells.value, cb.value, self.device).tensor(),
                DeviceBuffer(bits.value, bb.value, self.device).tensor())

    def clear_integrate_device(self, pts_ptr, n, R, t):
        """clear_rays + integrate_frame (vp_update_frame; host or device points)."""
        R, t = _pose(R, t)
        cs, us = native.ClearStats(), native.UpdateStats()
        check(lib().vp_update_frame(self.h, C.c_void_p(pts_ptr), C.c_uint64(n), _p(R, C.c_double),
                                    _p(t, C.c_double), C.byref(cs), C.byref(us)))
        return (cs.voxels_cleared, cs.voxels_freed), (us.voxels_touched, us.points_discarded)

    def steppable(self, seg: native.SegParams):
        n = C.c_uint64()
        idx, mean, nrm = C.POINTER(C.c_int32)(), C.POINTER(C.c_double)(), C.POINTER(C.c_double)()
        check(lib().vp_slab_steppable(self.h, C.byref(seg), C.byref(n), C.byref(idx), C.byref(mean),
                                      C.byref(nrm)))
        S = n.value
        addr = lambda p: C.cast(p, C.c_void_p).value or 0  # noqa: E731
        return S, (DeviceBuffer(addr(idx), 12 * S, self.device).tensor(),
                   DeviceBuffer(addr(mean), 24 * S, self.device).tensor(),
                   DeviceBuffer(addr(nrm), 24 * S, self.device).tensor())

    def segment(self, params: native.PipelineParams, S, idx_t, mean_t, nrm_t):
        out = C.POINTER(native.Polygons)()
        check(lib().vp_segment_steppable(self.h, C.byref(params), C.c_uint64(S),
                                         C.c_void_p(idx_t.data_ptr() if S else 0),
                                         C.c_void_p(mean_t.data_ptr() if S else 0),
                                         C.c_void_p(nrm_t.data_ptr() if S else 0), C.c_int(1), C.byref(out)))
        return polygons_to_py(out)

    def counters(self):
        """vp_grid_counters: cleared freed touched discarded dropped occupied V S K fits padded
        inliers poolv newly surv_max overflow, as of the last call that read them back."""
        out = np.zeros(16, np.uint64)
        check(lib().vp_grid_counters(self.h, _p(out, C.c_uint64)))
        return out

    def close(self):
        if self.h:
            lib().vp_grid_destroy(self.h)
            self.h = None


class LocalComm:
    """N virtual slabs in one process: the exchanges are device copies."""

    def __init__(self, world):
        self.world = world

    def broadcast_frame(self, pts_t):
        return pts_t

    def halo_exchange(self, slabs):
        for r, s in enumerate(slabs):
            if r > 0:  # my first owned plane -> left neighbour's right halo
                dst = slabs[r - 1].plane(s.x_begin)
                src = s.plane(s.x_begin)
                dst[0].copy_(src[0])
                dst[1].copy_(src[1])
            if r + 1 < len(slabs):  # my last owned plane -> right neighbour's left halo
                dst = slabs[r + 1].plane(s.x_end - 1)
                src = s.plane(s.x_end - 1)
                dst[0].copy_(src[0])
                dst[1].copy_(src[1])

    def gather_steppable(self, parts):
        import torch
        S = sum(p[0] for p in parts)
        if S == 0:
            e = torch.empty(0, dtype=torch.uint8, device="cuda")
            return 0, e, e, e
        return S, torch.cat([p[1][0] for p in parts]), torch.cat([p[1][1] for p in parts]), \
            torch.cat([p[1][2] for p in parts])


class DistComm:
    """One slab per rank under torch.distributed (NCCL on B200s; gloo for CPU tests)."""

    def __init__(self, dist, device):
        self.dist = dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.device = device

    def broadcast_frame(self, pts_t):
        import torch
        n = torch.tensor([pts_t.numel() if self.rank == 0 else 0], dtype=torch.int64, device=pts_t.device)
        self.dist.broadcast(n, 0)
        if self.rank != 0:
            pts_t = torch.empty(int(n.item()), dtype=pts_t.dtype, device=pts_t.device)
        self.dist.broadcast(pts_t, 0)
        return pts_t

    def halo_exchange(self, slabs):
        (s,) = slabs
        ops = []
        P2P = self.dist.P2POp
        if self.rank > 0:
            mine, halo = s.plane(s.x_begin), s.plane(s.x_begin - 1)
            ops += [P2P(self.dist.isend, mine[0], self.rank - 1), P2P(self.dist.isend, mine[1], self.rank - 1),
                    P2P(self.dist.irecv, halo[0], self.rank - 1), P2P(self.dist.irecv, halo[1], self.rank - 1)]
        if self.rank + 1 < self.world:
            mine, halo = s.plane(s.x_end - 1), s.plane(s.x_end)
            ops += [P2P(self.dist.isend, mine[0], self.rank + 1), P2P(self.dist.isend, mine[1], self.rank + 1),
                    P2P(self.dist.irecv, halo[0], self.rank + 1), P2P(self.dist.irecv, halo[1], self.rank + 1)]
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()

    def gather_steppable(self, parts):
        import torch
        ((S, arrs),) = parts
        mine = torch.tensor([S], dtype=torch.int64, device=arrs[0].device)
        allc = [torch.zeros_like(mine) for _ in range(self.world)]
        self.dist.all_gather(allc, mine)
        counts = [int(c.item()) for c in allc]
        total = sum(counts)
        if self.rank != 0:
            for a in arrs:
                if S:
                    self.dist.send(a, 0)
            return total, None, None, None
        out = [torch.empty(total * w, dtype=torch.uint8, device=arrs[0].device) for w in (12, 24, 24)]
        off = 0
        for r, n in enumerate(counts):
            for o, a, w in zip(out, arrs, (12, 24, 24)):
                view = o[off * w:(off + n) * w]
                if n == 0:
                    continue
                if r == 0:
                    view.copy_(a)
                else:
                    self.dist.recv(view, r)
            off += n
        return total, out[0], out[1], out[2]


def slab_frame(slabs, comm, pts_t, R, t, params: native.PipelineParams):
    """One frame over the local slabs; returns the polygons on rank 0 (else None)."""
    import torch
    # the library runs on its own streams and returns synchronised; whatever
    # torch (or NCCL, which torch's stream waits on) produced is fenced with a
    # stream synchronise before the library reads it
    sync = torch.cuda.current_stream().synchronize if pts_t.is_cuda else (lambda: None)
    pts_t = comm.broadcast_frame(pts_t)
    sync()
    n = pts_t.numel() // 12 if pts_t.dtype.itemsize == 1 else pts_t.numel() // 3
    for s in slabs:
        s.clear_integrate_device(pts_t.data_ptr(), n, R, t)
    comm.halo_exchange(slabs)
    sync()
    parts = [s.steppable(params.seg) for s in slabs]
    S, idx, mean, nrm = comm.gather_steppable(parts)
    if idx is None:
        return None
    sync()
    return slabs[0].segment(params, S, idx, mean, nrm)
