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
5. per-plane steppable counts are all-gathered: ordinals are x-major, so every
   slab owns a contiguous global ordinal range and every plane's first ordinal
   is known everywhere (SlabLayout);
6. each slab receives the steppable voxels of the w planes either side of it
   (w = adjacency window, segmentation.cpp:89) and runs build_adjacency +
   label_components locally (library, vp_slab_label);
7. boundary-label merge: the slabs' boundary triples are all-gathered and a
   union-find over the boundary zone (replicated, on device) gives every
   owned voxel its canonical label = the component's minimum global ordinal
   (vp_slab_merge) -- the single-grid label, bit-exact;
8. cluster gather: members of clusters whose label lies in a lower slab are
   sent to that owner (vp_slab_export); each owner runs filter_clusters ..
   make_polygon on its clusters, members in global ordinal order
   (vp_slab_segment_owned);
9. polygons are gathered to rank 0 in slab order (= ascending label order).

The product path runs the whole sequence inside the library, one call per
rank and frame (vp_slab_frame, csrc/slab_frame.cu): the exchanges are
stream-ordered collectives of a communicator table -- the library's NCCL
communicator (nccl_comm: NVLink / NVSwitch between the GPUs of a node), the
in-process hub of vp_slab_frame_local (N virtual slabs on one GPU, one host
thread each), or TorchCommOps (any torch.distributed backend; the CPU-staged
gloo variant drives two processes on one GPU in the tests).

slab_frame() below is the same sequence written in Python over the
library's phase functions (LocalComm / DistComm); it is kept as an executable
model of the protocol for the gloo CPU tests (tests/test_slab_comm.py).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import native
from .native import _p, _pose, check, lib, polygons_to_py

MEMBER_REC_BYTES = 32  # vp_member_rec


class DeviceBuffer:
    """Zero-copy torch view of library-owned device memory."""

    def __init__(self, ptr: int, nbytes: int, device: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}
        self.device = device

    def tensor(self):
        import torch
        return torch.as_tensor(self, device=f"cuda:{self.device}")


def _dev_bytes(ptr, nbytes, device):
    import torch
    if nbytes == 0 or not ptr:
        return torch.empty(0, dtype=torch.uint8, device=f"cuda:{device}")
    return DeviceBuffer(ptr, nbytes, device).tensor()


def _addr(p):
    return C.cast(p, C.c_void_p).value or 0


def split_x(extent_x: int, world: int):
    """Balanced contiguous x ranges [(x_begin, x_end)] for `world` slabs."""
    base, rem = divmod(extent_x, world)
    out, x = [], 0
    for r in range(world):
        w = base + (1 if r < rem else 0)
        out.append((x, x + w))
        x += w
    return out


def adjacency_window(seg: native.SegParams, res: float) -> int:
    """w = max(1, ceil(distance_th / resolution)) (segmentation.cpp:89), from the library."""
    w = C.c_int32()
    check(lib().vp_adjacency_window(C.byref(seg), C.c_double(res), C.byref(w)))
    return w.value


class SlabLayout:
    """One frame's global view of the slabs (host arithmetic only; mirrors
    vp_slab_extend): P[x] = global ordinal of the first steppable voxel of
    window plane x, slab k owns ordinals [P[xb_k], P[xb_{k+1})), its extended
    list covers planes [max(0, xb_k - w), min(gex, xb_{k+1} + w))."""

    def __init__(self, ranges, plane_counts, w: int):
        self.ranges = [tuple(int(v) for v in r) for r in ranges]
        self.n = len(self.ranges)
        self.gex = self.ranges[-1][1]
        counts = np.asarray(plane_counts, np.int64)
        assert counts.shape == (self.gex,)
        self.P = np.zeros(self.gex + 1, np.int64)
        np.cumsum(counts, out=self.P[1:])
        self.w = int(w)
        self.x_begin = np.asarray([a for a, _ in self.ranges] + [self.gex], np.int32)
        self.counts_u32 = np.ascontiguousarray(counts, np.uint32)

    def ext(self, k):
        a, b = self.ranges[k]
        return max(0, a - self.w), min(self.gex, b + self.w)

    def n_own(self, k):
        a, b = self.ranges[k]
        return int(self.P[b] - self.P[a])

    def n_left(self, k):
        lo, _ = self.ext(k)
        return int(self.P[self.ranges[k][0]] - self.P[lo])

    def n_ext(self, k):
        lo, hi = self.ext(k)
        return int(self.P[hi] - self.P[lo])

    def transfers(self):
        """Halo lists: (src, dst, src_start, count, dst_start) -- entries of
        slab src's own list [src_start, +count) land at [dst_start, +count) of
        slab dst's extended list. Same list on every rank."""
        out = []
        for d in range(self.n):
            lo, hi = self.ext(d)
            for s in range(self.n):
                if s == d:
                    continue
                a, b = self.ranges[s]
                x0, x1 = max(lo, a), min(hi, b)
                if x0 >= x1:
                    continue
                cnt = int(self.P[x1] - self.P[x0])
                if cnt:
                    out.append((s, d, int(self.P[x0] - self.P[a]), cnt, int(self.P[x0] - self.P[lo])))
        return out

    def c_struct(self):
        lay = VpSlabLayout()
        lay.n_slabs = self.n
        lay.x_begin = _p(self.x_begin, C.c_int32)
        lay.plane_counts = _p(self.counts_u32, C.c_uint32)
        return lay


class VpSlabLayout(C.Structure):
    _fields_ = [("n_slabs", C.c_int32), ("x_begin", C.POINTER(C.c_int32)),
                ("plane_counts", C.POINTER(C.c_uint32))]


class Slab:
    """One slab grid (vp_slab_create) owning window x in [x_begin, x_end)."""

    def __init__(self, res, window_extent, center, x_begin, x_end, device=0):
        ext = np.asarray(window_extent, np.int32)
        c = np.asarray(center, np.float64)
        self.h = C.c_void_p()
        self.res = res
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
        """estimate_normals + classify_steppable on the owned voxels: (S, (idx, mean, normal) byte views)."""
        n = C.c_uint64()
        idx, mean, nrm = C.POINTER(C.c_int32)(), C.POINTER(C.c_double)(), C.POINTER(C.c_double)()
        check(lib().vp_slab_steppable(self.h, C.byref(seg), C.byref(n), C.byref(idx), C.byref(mean),
                                      C.byref(nrm)))
        S = n.value
        return S, (_dev_bytes(_addr(idx), 12 * S, self.device), _dev_bytes(_addr(mean), 24 * S, self.device),
                   _dev_bytes(_addr(nrm), 24 * S, self.device))

    def plane_counts(self):
        """Steppable voxels per owned plane (device uint32 view)."""
        import torch
        ptr = C.POINTER(C.c_uint32)()
        n = C.c_int32()
        check(lib().vp_slab_plane_counts(self.h, C.byref(ptr), C.byref(n)))
        return _dev_bytes(_addr(ptr), 4 * n.value, self.device).view(torch.int32)

    def extend(self, seg: native.SegParams, layout: SlabLayout):
        """Extended list buffers (idx 12 B, mean 24 B, normal 24 B per entry) with the own list in place."""
        lay = layout.c_struct()
        idx, mean, nrm = C.POINTER(C.c_int32)(), C.POINTER(C.c_double)(), C.POINTER(C.c_double)()
        n, lo, hi = C.c_uint64(), C.c_int32(), C.c_int32()
        check(lib().vp_slab_extend(self.h, C.byref(seg), C.byref(lay), C.byref(idx), C.byref(mean), C.byref(nrm),
                                   C.byref(n), C.byref(lo), C.byref(hi)))
        N = n.value
        k = layout.ranges.index((self.x_begin, self.x_end))
        self.n_own = layout.n_own(k)
        self.ext_lists = (_dev_bytes(_addr(idx), 12 * N, self.device), _dev_bytes(_addr(mean), 24 * N, self.device),
                          _dev_bytes(_addr(nrm), 24 * N, self.device))
        return self.ext_lists

    def label(self, seg: native.SegParams):
        """Local CCL on the extended list: (boundary triples as an int32 (n, 3) view, zone size)."""
        import torch
        t = C.POINTER(C.c_int32)()
        n, z = C.c_uint64(), C.c_uint64()
        check(lib().vp_slab_label(self.h, C.byref(seg), C.byref(t), C.byref(n), C.byref(z)))
        return _dev_bytes(_addr(t), 12 * n.value, self.device).view(torch.int32).view(-1, 3), z.value

    def merge(self, triples):
        """Canonical labels (global ordinals) of the owned entries (device int32 view)."""
        import torch
        out = C.POINTER(C.c_int32)()
        n = triples.shape[0] if triples is not None else 0
        check(lib().vp_slab_merge(self.h, C.c_void_p(triples.data_ptr() if n else 0), C.c_uint64(n),
                                  C.byref(out)))
        self._labels = _dev_bytes(_addr(out), 4 * self.n_own, self.device).view(torch.int32)
        return self._labels

    def merge_labels(self):
        """The labels of the last vp_slab_merge (device int32 view of the owned entries)."""
        return self._labels

    def export(self, n_slabs):
        """Members of clusters owned by lower slabs: (per-destination counts, 32-byte records view)."""
        counts = np.zeros(n_slabs, np.uint64)
        rec = C.c_void_p()
        check(lib().vp_slab_export(self.h, _p(counts, C.c_uint64), C.byref(rec)))
        tot = int(counts.sum())
        return counts.astype(np.int64), _dev_bytes(rec.value or 0, MEMBER_REC_BYTES * tot, self.device)

    def segment_owned(self, params: native.PipelineParams, recv, n_recv):
        out = C.POINTER(native.Polygons)()
        check(lib().vp_slab_segment_owned(self.h, C.byref(params), C.c_void_p(recv.data_ptr() if n_recv else 0),
                                          C.c_uint64(n_recv), C.byref(out)))
        return polygons_to_py(out)

    def segment_gathered(self, params: native.PipelineParams, S, idx_t, mean_t, nrm_t):
        """Segment a whole steppable list on this grid (vp_segment_steppable)."""
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


# ------------------------------------------------------------------ comms
class LocalComm:
    """N virtual slabs in one process: the exchanges are device copies."""

    def __init__(self, world):
        self.world = world
        self.rank = 0

    def slab_index(self, i):
        return i

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

    def allgather_plane_counts(self, counts):
        import torch
        return torch.cat(counts).cpu().numpy() if counts else np.zeros(0, np.int32)

    def exchange_steppable(self, layout, ext_lists):
        """ext_lists[k] = (idx, mean, normal) byte views of slab k's extended list."""
        for s, d, s0, cnt, d0 in layout.transfers():
            ls = layout.n_left(s)
            for src, dst, w in zip(ext_lists[s], ext_lists[d], (12, 24, 24)):
                dst[d0 * w:(d0 + cnt) * w].copy_(src[(ls + s0) * w:(ls + s0 + cnt) * w])

    def allgather_triples(self, parts):
        import torch
        return torch.cat(parts) if parts else None

    def exchange_members(self, exports):
        """exports[k] = (dest_counts, records): returns per slab the records
        received from the higher slabs, in slab order."""
        import torch
        out = []
        n = len(exports)
        offs = [np.concatenate([[0], np.cumsum(c)]) for c, _ in exports]
        for d in range(n):
            parts = []
            for s in range(d + 1, n):
                c = int(exports[s][0][d])
                if c:
                    o = int(offs[s][d])
                    parts.append(exports[s][1][o * MEMBER_REC_BYTES:(o + c) * MEMBER_REC_BYTES])
            recv = torch.cat(parts) if parts else None
            out.append((recv, sum(p.numel() for p in parts) // MEMBER_REC_BYTES))
        return out

    def gather_polygons(self, per_slab):
        return [p for polys in per_slab for p in polys]


class DistComm:
    """One slab per rank under torch.distributed (NCCL on B200s; gloo for CPU tests)."""

    def __init__(self, dist, device):
        self.dist = dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.device = device

    def slab_index(self, i):
        return self.rank

    def broadcast_frame(self, pts_t):
        import torch
        n = torch.tensor([pts_t.numel() if self.rank == 0 else 0], dtype=torch.int64, device=pts_t.device)
        self.dist.broadcast(n, 0)
        if self.rank != 0:
            pts_t = torch.empty(int(n.item()), dtype=pts_t.dtype, device=pts_t.device)
        self.dist.broadcast(pts_t, 0)
        return pts_t

    def _p2p(self, ops):
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()

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
        self._p2p(ops)

    def _allgather_var(self, t):
        """All-gather of 1-D tensors of different lengths, concatenated in rank order."""
        import torch
        n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
        ns = [torch.zeros_like(n) for _ in range(self.world)]
        self.dist.all_gather(ns, n)
        ns = [int(v.item()) for v in ns]
        m = max(ns)
        if m == 0:
            return t[:0]
        buf = torch.zeros(m, dtype=t.dtype, device=t.device)
        buf[:t.numel()] = t
        outs = [torch.empty_like(buf) for _ in range(self.world)]
        self.dist.all_gather(outs, buf)
        return torch.cat([o[:k] for o, k in zip(outs, ns)])

    def allgather_plane_counts(self, counts):
        (c,) = counts
        return self._allgather_var(c).cpu().numpy()

    def exchange_steppable(self, layout, ext_lists):
        (mine,) = ext_lists
        ops = []
        P2P = self.dist.P2POp
        ls = layout.n_left(self.rank)
        for s, d, s0, cnt, d0 in layout.transfers():
            if s == self.rank:
                for src, w in zip(mine, (12, 24, 24)):
                    ops.append(P2P(self.dist.isend, src[(ls + s0) * w:(ls + s0 + cnt) * w], d))
            elif d == self.rank:
                for dst, w in zip(mine, (12, 24, 24)):
                    ops.append(P2P(self.dist.irecv, dst[d0 * w:(d0 + cnt) * w], s))
        self._p2p(ops)

    def allgather_triples(self, parts):
        (t,) = parts
        return self._allgather_var(t.reshape(-1)).view(-1, 3)

    def exchange_members(self, exports):
        import torch
        ((counts, rec),) = exports
        mine = torch.as_tensor(np.asarray(counts, np.int64), device=rec.device if rec.numel() else self.device)
        allc = [torch.zeros_like(mine) for _ in range(self.world)]
        self.dist.all_gather(allc, mine)
        M = np.stack([a.cpu().numpy() for a in allc])  # M[s][d] = records s sends to d
        offs = np.concatenate([[0], np.cumsum(M[self.rank])])
        ops = []
        P2P = self.dist.P2POp
        for d in range(self.rank):  # my foreign members go to lower slabs
            c = int(M[self.rank][d])
            if c:
                o = int(offs[d])
                ops.append(P2P(self.dist.isend, rec[o * MEMBER_REC_BYTES:(o + c) * MEMBER_REC_BYTES], d))
        total = int(M[self.rank + 1:, self.rank].sum())
        recv = torch.empty(total * MEMBER_REC_BYTES, dtype=torch.uint8, device=mine.device)
        o = 0
        for s in range(self.rank + 1, self.world):
            c = int(M[s][self.rank])
            if c:
                ops.append(P2P(self.dist.irecv, recv[o * MEMBER_REC_BYTES:(o + c) * MEMBER_REC_BYTES], s))
                o += c
        self._p2p(ops)
        return [(recv if total else None, total)]

    def gather_polygons(self, per_slab):
        (polys,) = per_slab
        out = [None] * self.world if self.rank == 0 else None
        self.dist.gather_object(polys, out, dst=0)
        if self.rank != 0:
            return None
        return [p for part in out for p in part]


# ------------------------------------------------------------------ frame
def slab_frame(slabs, comm, pts_t, R, t, params: native.PipelineParams, stages=None):
    """One frame over the local slabs; returns the polygons on rank 0 (else None).
    `stages` (optional dict) receives per-phase counts for the bench."""
    import time

    import torch
    clock = [time.perf_counter()]

    def phase(name):  # wall time per phase (library calls return synchronised)
        if stages is not None:
            now = time.perf_counter()
            stages.setdefault("phase_ms", {})[name] = round(1e3 * (now - clock[0]), 3)
            clock[0] = now
    # the library runs on its own streams and returns synchronised; whatever
    # torch (or NCCL, which torch's stream waits on) produced is fenced with a
    # stream synchronise before the library reads it
    sync = torch.cuda.current_stream().synchronize if pts_t.is_cuda else (lambda: None)
    pts_t = comm.broadcast_frame(pts_t)
    sync()
    n = pts_t.numel() // 12 if pts_t.dtype.itemsize == 1 else pts_t.numel() // 3
    for s in slabs:
        s.clear_integrate_device(pts_t.data_ptr(), n, R, t)
    phase("broadcast+clear+integrate")
    if stages is not None:
        stages["c_map"] = slabs[0].counters()
    comm.halo_exchange(slabs)
    sync()
    seg = params.seg
    for s in slabs:
        s.steppable(seg)
    phase("halo planes+normals+classify")
    if stages is not None:
        stages["c_step"] = slabs[0].counters()
    counts = comm.allgather_plane_counts([s.plane_counts() for s in slabs])
    ranges = [s_range for s_range in _ranges(slabs, comm)]
    layout = SlabLayout(ranges, counts, adjacency_window(seg, slabs[0].res))
    phase("plane counts+layout")
    ext = [s.extend(seg, layout) for s in slabs]
    comm.exchange_steppable(layout, ext)
    sync()
    phase("halo lists")
    parts, zsize = [], 0
    for s in slabs:
        tr, zsize = s.label(seg)
        parts.append(tr)
    phase("local ccl")
    triples = comm.allgather_triples(parts)
    sync()
    for s in slabs:
        s.merge(triples)
    phase("label merge")
    exports = [s.export(layout.n) for s in slabs]
    recv = comm.exchange_members(exports)
    sync()
    phase("cluster gather")
    polys = [s.segment_owned(params, r, nr) for s, (r, nr) in zip(slabs, recv)]
    phase("fit+refine+polygon")
    if stages is not None:
        stages["c_seg"] = slabs[0].counters()
        stages.update(steppable=int(layout.P[-1]), zone=int(zsize), triples=int(triples.shape[0]),
                      exported=int(sum(int(c.sum()) for c, _ in exports)))
    out = comm.gather_polygons(polys)
    phase("polygon gather")
    return out


_RANGES_CACHE: dict = {}


def _ranges(slabs, comm):
    """x ranges of all slabs of the decomposition (all ranks for DistComm)."""
    if isinstance(comm, DistComm):
        key = (comm.world, slabs[0].window_extent[0])
        if key not in _RANGES_CACHE:
            import torch
            mine = torch.tensor([slabs[0].x_begin, slabs[0].x_end], dtype=torch.int64,
                                device=f"cuda:{slabs[0].device}" if comm.device is not None else "cpu")
            allr = [torch.zeros_like(mine) for _ in range(comm.world)]
            comm.dist.all_gather(allr, mine)
            _RANGES_CACHE[key] = [tuple(int(v) for v in a.tolist()) for a in allr]
        return _RANGES_CACHE[key]
    return [(s.x_begin, s.x_end) for s in slabs]


# ------------------------------------------------- library-orchestrated frame
class P2POp(C.Structure):
    _fields_ = [("peer", C.c_int32), ("send", C.c_int32), ("ptr", C.c_void_p), ("bytes", C.c_uint64)]


_BCAST = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32, C.c_void_p)
_ALLG = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)
_GROUP = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.POINTER(P2POp), C.c_void_p)


class CommOps(C.Structure):
    """vp_comm_ops: the communicator table vp_slab_frame runs its exchanges on."""
    _fields_ = [("ctx", C.c_void_p), ("rank", C.c_int32), ("nranks", C.c_int32),
                ("broadcast", _BCAST), ("allgather", _ALLG), ("group", _GROUP)]


def nccl_comm(dist, device: int) -> CommOps:
    """The library's NCCL communicator over the ranks of `dist` (one GPU each);
    the 128-byte unique id travels through dist (setup only)."""
    import torch
    rank, world = dist.get_rank(), dist.get_world_size()
    uid = np.zeros(128, np.uint8)
    if rank == 0:
        check(lib().vp_comm_nccl_unique_id(_p(uid, C.c_uint8)))
    t = torch.from_numpy(uid).to(f"cuda:{device}" if dist.get_backend() == "nccl" else "cpu")
    dist.broadcast(t, 0)
    uid = np.ascontiguousarray(t.cpu().numpy())
    ops = CommOps()
    check(lib().vp_comm_nccl_create(_p(uid, C.c_uint8), C.c_int32(world), C.c_int32(rank), C.c_int(device),
                                    C.byref(ops)))
    return ops


def nccl_comm_destroy(ops: CommOps) -> None:
    lib().vp_comm_nccl_destroy(C.byref(ops))


class TorchCommOps:
    """vp_comm_ops implemented with torch.distributed collectives. With a gloo
    group the device buffers are staged through host tensors (the library's
    stream is drained first); used to run real slabs in several processes on
    one GPU, where NCCL refuses duplicate devices."""

    def __init__(self, dist, device: int):
        import torch
        self.dist, self.device = dist, device
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self._torch = torch
        self.ops = CommOps()
        self.ops.ctx = None
        self.ops.rank, self.ops.nranks = self.rank, self.world
        # keep the callbacks alive as long as this object
        self._cb = (_BCAST(self._bcast), _ALLG(self._allgather), _GROUP(self._group))
        self.ops.broadcast, self.ops.allgather, self.ops.group = self._cb

    def _sync(self, stream):
        # the library's stream: its producers must be done before the copies
        self._torch.cuda.ExternalStream(stream, device=f"cuda:{self.device}").synchronize()

    def _d2h(self, ptr, nbytes):
        if not nbytes:
            return np.empty(0, np.uint8)
        return DeviceBuffer(ptr, nbytes, self.device).tensor().cpu().numpy()

    def _h2d(self, ptr, buf):
        if buf.nbytes:
            DeviceBuffer(ptr, buf.nbytes, self.device).tensor().copy_(self._torch.from_numpy(buf))
            self._torch.cuda.current_stream(self.device).synchronize()  # before the library stream reads it

    def _bcast(self, ctx, buf, nbytes, root, stream):
        try:
            self._sync(stream)
            h = self._d2h(buf, nbytes) if self.rank == root else np.empty(nbytes, np.uint8)
            t = self._torch.from_numpy(h)
            self.dist.broadcast(t, int(root))
            if self.rank != root:
                self._h2d(buf, t.numpy())
            return 0
        except Exception:  # noqa: BLE001 -- reported to the library as a failed collective
            return 1

    def _allgather(self, ctx, send, recv, nbytes, stream):
        try:
            self._sync(stream)
            t = self._torch.from_numpy(self._d2h(send, nbytes))
            outs = [self._torch.empty(nbytes, dtype=self._torch.uint8) for _ in range(self.world)]
            self.dist.all_gather(outs, t)
            self._h2d(recv, self._torch.cat(outs).numpy())
            return 0
        except Exception:  # noqa: BLE001
            return 1

    def _group(self, ctx, n, ops, stream):
        try:
            self._sync(stream)
            reqs, recvs = [], []
            for i in range(n):
                o = ops[i]
                if not o.bytes:
                    continue
                if o.send:
                    reqs.append(self.dist.isend(self._torch.from_numpy(self._d2h(o.ptr, o.bytes)), int(o.peer)))
                else:
                    t = self._torch.empty(int(o.bytes), dtype=self._torch.uint8)
                    reqs.append(self.dist.irecv(t, int(o.peer)))
                    recvs.append((o.ptr, t))
            for r in reqs:
                r.wait()
            for ptr, t in recvs:
                self._h2d(ptr, t.numpy())
            return 0
        except Exception:  # noqa: BLE001
            return 1


def frame(slab: Slab, ops, pts, n: int, R, t, params: native.PipelineParams):
    """One frame on this rank's slab (vp_slab_frame): rank 0 passes its points
    (numpy host array or a device tensor), the others None and the same n.
    Returns the window's polygons on rank 0, else None."""
    R, t = _pose(R, t)
    ops_s = ops.ops if isinstance(ops, TorchCommOps) else ops
    ptr = _points_ptr(pts)
    out = C.POINTER(native.Polygons)()
    check(lib().vp_slab_frame(slab.h, C.byref(ops_s), C.c_void_p(ptr), C.c_uint64(n), _p(R, C.c_double),
                              _p(t, C.c_double), C.byref(params), C.byref(out)))
    return polygons_to_py(out) if out else None


def frame_local(slabs_list, pts, R, t, params: native.PipelineParams):
    """One frame over N virtual slabs in this process (vp_slab_frame_local)."""
    R, t = _pose(R, t)
    arr = (C.c_void_p * len(slabs_list))(*[s.h.value for s in slabs_list])
    n = _points_len(pts)
    out = C.POINTER(native.Polygons)()
    check(lib().vp_slab_frame_local(arr, C.c_int32(len(slabs_list)), C.c_void_p(_points_ptr(pts)), C.c_uint64(n),
                                    _p(R, C.c_double), _p(t, C.c_double), C.byref(params), C.byref(out)))
    return polygons_to_py(out)


def _points_ptr(pts):
    if pts is None:
        return 0
    if hasattr(pts, "data_ptr"):
        return pts.data_ptr()
    return np.ascontiguousarray(pts, np.float32).ctypes.data


def _points_len(pts):
    if pts is None:
        return 0
    if hasattr(pts, "data_ptr"):
        return pts.numel() // 3 if pts.dtype.itemsize == 4 else pts.numel() // 12
    return len(pts)
