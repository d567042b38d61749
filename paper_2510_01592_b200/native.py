"""ctypes binding of the C ABI in include/voxplane_b200.h.

This is the Python harness's view of the product library
(`paper_2510_01592_b200/lib/libvoxplane_b200.so`, hand-written sm_100a
kernels + host runtime). There is no fallback: if the library is missing or
no B200 is visible, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VP_LIB") or os.path.join(PKG, "lib", "libvoxplane_b200.so")  # VP_LIB: experiments only

VP_OK, VP_EINVAL, VP_EEMPTY, VP_ENOMEM, VP_ECUDA, VP_ENODEV = range(6)


class VpError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"voxplane_b200 error {code}: {msg}")
        self.code = code


class InvalidArgument(VpError, ValueError):
    """std::invalid_argument in the reference."""


class SegParams(C.Structure):
    _fields_ = [("neighbor_radius", C.c_int32), ("min_neighbors", C.c_int32),
                ("max_angle_deg", C.c_double), ("adjacency_angle_deg", C.c_double),
                ("distance_th", C.c_double), ("min_cluster_size", C.c_int32),
                ("up", C.c_double * 3)]


class RansacParams(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("inlier_eps", C.c_double), ("seed", C.c_uint64),
                ("up", C.c_double * 3), ("execution", C.c_int32)]


class PipelineParams(C.Structure):
    _fields_ = [("seg", SegParams), ("ransac", RansacParams), ("refine", C.c_int32),
                ("min_polygon_area", C.c_double), ("refine_exact", C.c_int32)]


class UpdateStats(C.Structure):
    _fields_ = [("voxels_touched", C.c_uint64), ("points_discarded", C.c_uint64)]


class ClearStats(C.Structure):
    _fields_ = [("voxels_cleared", C.c_uint64), ("voxels_freed", C.c_uint64)]


class ShiftStats(C.Structure):
    _fields_ = [("shift", C.c_int32 * 3), ("voxels_dropped", C.c_uint64)]


class Plane(C.Structure):
    _fields_ = [("normal", C.c_double * 3), ("offset", C.c_double), ("inlier_count", C.c_int32),
                ("cluster_label", C.c_int32)]


class Polygon(C.Structure):
    _fields_ = [("plane", Plane), ("nverts", C.c_uint32), ("v2d", C.POINTER(C.c_double)),
                ("v3d", C.POINTER(C.c_double)), ("area", C.c_double)]


class Polygons(C.Structure):
    _fields_ = [("count", C.c_size_t), ("polys", C.POINTER(Polygon))]


class Occupied(C.Structure):
    _fields_ = [("count", C.c_size_t), ("idx", C.POINTER(C.c_int32)), ("mean", C.POINTER(C.c_double)),
                ("npts", C.POINTER(C.c_uint32)), ("status", C.POINTER(C.c_uint8))]


class Estimates(C.Structure):
    _fields_ = [("count", C.c_size_t), ("idx", C.POINTER(C.c_int32)), ("mean", C.POINTER(C.c_double)),
                ("normal", C.POINTER(C.c_double)), ("neighbor_count", C.POINTER(C.c_int32)),
                ("angle_to_up_deg", C.POINTER(C.c_double)), ("valid", C.POINTER(C.c_uint8))]


class Steppable(C.Structure):
    _fields_ = [("count", C.c_size_t), ("idx", C.POINTER(C.c_int32)), ("mean", C.POINTER(C.c_double)),
                ("normal", C.POINTER(C.c_double))]


class Fits(C.Structure):
    _fields_ = [("count", C.c_size_t), ("models", C.POINTER(Plane)), ("offsets", C.POINTER(C.c_uint64)),
                ("inliers", C.POINTER(C.c_double)), ("clusters_skipped_small", C.c_uint64),
                ("clusters_unfit", C.c_uint64)]


class FrameTiming(C.Structure):
    _fields_ = [("mapping_ms", C.c_double), ("classify_ms", C.c_double), ("cluster_ms", C.c_double),
                ("ransac_ms", C.c_double), ("hull_ms", C.c_double), ("total_ms", C.c_double),
                ("points", C.c_uint64), ("voxels", C.c_uint64), ("clusters", C.c_uint64)]


class RunOutputs(C.Structure):
    _fields_ = [("per_frame", C.POINTER(C.POINTER(Polygons))), ("timings", C.POINTER(FrameTiming)),
                ("traces", C.POINTER(C.POINTER(C.c_uint8))), ("trace_lens", C.POINTER(C.c_uint64))]


def default_params(seed: int = 0, refine: bool = True, min_area: float = 0.002,
                   refine_exact: bool = False) -> PipelineParams:
    """SegmentationParams / RansacParams / RunConfig / OutputConfig defaults."""
    p = PipelineParams()
    s = p.seg
    s.neighbor_radius, s.min_neighbors = 1, 3
    s.max_angle_deg = s.adjacency_angle_deg = 15.0
    s.distance_th, s.min_cluster_size = 0.05, 30
    s.up[:] = (0.0, 0.0, 1.0)
    r = p.ransac
    r.iterations, r.inlier_eps, r.seed, r.execution = 100, 0.01, seed, 0
    r.up[:] = (0.0, 0.0, 1.0)
    p.refine = 1 if refine else 0
    p.min_polygon_area = min_area
    p.refine_exact = 1 if refine_exact else 0
    return p


_lib = None


def lib():
    """Load the product library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        L.vp_last_error.restype = C.c_char_p
        L.vp_version.restype = C.c_char_p
        L.vp_pipeline_grid.restype = C.c_void_p
        L.vp_kernel_launch_count.restype = C.c_uint64
        L.vp_default_ablation_config.restype = None
        _lib = L
    return _lib


def check(rc):
    if rc != VP_OK:
        msg = lib().vp_last_error().decode(errors="replace")
        if rc == VP_EINVAL:
            raise InvalidArgument(rc, msg)
        raise VpError(rc, msg)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def _pose(R, t):
    R = np.ascontiguousarray(R, np.float64).reshape(9)
    t = np.ascontiguousarray(t, np.float64).reshape(3)
    return R, t


def polygons_to_py(pp) -> list[dict]:
    out = []
    P = pp.contents
    for i in range(P.count):
        q = P.polys[i]
        nv = q.nverts
        v2 = np.ctypeslib.as_array(q.v2d, (nv, 2)).copy() if nv else np.zeros((0, 2))
        v3 = np.ctypeslib.as_array(q.v3d, (nv, 3)).copy() if nv else np.zeros((0, 3))
        out.append(dict(normal=np.array(q.plane.normal[:]), offset=q.plane.offset,
                        inlier_count=q.plane.inlier_count, label=q.plane.cluster_label,
                        v2d=v2, v3d=v3, area=q.area))
    lib().vp_polygons_free(pp)
    return out


class Pipeline:
    """run_frames state on the device (vp_pipeline_*)."""

    def __init__(self, res, extent, start_center, params: PipelineParams | None = None, device=0):
        self.params = params or default_params()
        ext = np.asarray(extent, np.int32)
        c = np.asarray(start_center, np.float64)
        self.h = C.c_void_p()
        check(lib().vp_pipeline_create(C.c_double(res), _p(ext, C.c_int32), _p(c, C.c_double),
                                       C.byref(self.params), C.c_int(device), C.byref(self.h)))

    def frame(self, pts, R, t, want_polygons=True):
        pts = np.ascontiguousarray(pts, np.float32)
        R, t = _pose(R, t)
        out = C.POINTER(Polygons)()
        tm = FrameTiming()
        check(lib().vp_pipeline_frame(self.h, _p(pts, C.c_float), C.c_uint64(len(pts)),
                                      _p(R, C.c_double), _p(t, C.c_double),
                                      C.byref(out) if want_polygons else None, C.byref(tm)))
        return (polygons_to_py(out) if want_polygons else None), tm

    def frame_ptr(self, pts_host_ptr: int, n: int, R, t, want_polygons=True, want_timing=True):
        """vp_pipeline_frame on a raw host pointer (e.g. pinned memory); the
        stage timings (FrameTiming, six event queries) only when wanted."""
        R, t = _pose(R, t)
        out = C.POINTER(Polygons)()
        tm = FrameTiming()
        check(lib().vp_pipeline_frame(self.h, C.c_void_p(pts_host_ptr), C.c_uint64(n),
                                      _p(R, C.c_double), _p(t, C.c_double),
                                      C.byref(out) if want_polygons else None,
                                      C.byref(tm) if want_timing else None))
        return (polygons_to_py(out) if want_polygons else None), (tm if want_timing else None)

    def run(self, frames, device_ptrs=None, want_polygons=True, timings=False):
        """vp_pipeline_run: run_frames over a list of Frames (host arrays), or
        over device pointers: device_ptrs = [(ptr, n), ...] with frames giving poses."""
        nf = len(frames)
        R = np.ascontiguousarray(np.stack([np.asarray(f.rotation, np.float64).reshape(9) for f in frames]))
        t = np.ascontiguousarray(np.stack([np.asarray(f.translation, np.float64).reshape(3) for f in frames]))
        ptrs = (C.c_void_p * max(nf, 1))()
        ns = np.zeros(max(nf, 1), np.uint64)
        keep = []
        if device_ptrs is not None:
            for k, (ptr, n) in enumerate(device_ptrs):
                ptrs[k] = ptr
                ns[k] = n
        else:
            for k, f in enumerate(frames):
                a = np.ascontiguousarray(f.points, np.float32)
                keep.append(a)
                ptrs[k] = a.ctypes.data
                ns[k] = len(a)
        out = C.POINTER(Polygons)()
        tms = (FrameTiming * max(nf, 1))()
        check(lib().vp_pipeline_run(self.h, C.c_size_t(nf), ptrs, _p(ns, C.c_uint64), _p(R, C.c_double),
                                    _p(t, C.c_double), C.c_int(1 if device_ptrs is not None else 0),
                                    C.byref(out) if want_polygons else None, tms if timings else None))
        polys = polygons_to_py(out) if want_polygons else None
        return (polys, [tms[k] for k in range(nf)]) if timings else polys

    def run_frames(self, frames, device_ptrs=None, per_frame=True, timings=True, traces=False):
        """vp_pipeline_run_frames: the pipelined run with per-frame outputs.
        Returns dict(polygons=final, per_frame=[...], timings=[...], traces=[bytes])."""
        nf = len(frames)
        R = np.ascontiguousarray(np.stack([np.asarray(f.rotation, np.float64).reshape(9) for f in frames]))
        t = np.ascontiguousarray(np.stack([np.asarray(f.translation, np.float64).reshape(3) for f in frames]))
        ptrs = (C.c_void_p * max(nf, 1))()
        ns = np.zeros(max(nf, 1), np.uint64)
        keep = []
        if device_ptrs is not None:
            for k, (ptr, n) in enumerate(device_ptrs):
                ptrs[k] = ptr
                ns[k] = n
        else:
            for k, f in enumerate(frames):
                a = np.ascontiguousarray(f.points, np.float32)
                keep.append(a)
                ptrs[k] = a.ctypes.data
                ns[k] = len(a)
        ex = RunOutputs()
        pf = (C.POINTER(Polygons) * max(nf, 1))()
        tms = (FrameTiming * max(nf, 1))()
        trs = (C.POINTER(C.c_uint8) * max(nf, 1))()
        tls = (C.c_uint64 * max(nf, 1))()
        if per_frame:
            ex.per_frame = C.cast(pf, C.POINTER(C.POINTER(Polygons)))
        if timings:
            ex.timings = C.cast(tms, C.POINTER(FrameTiming))
        if traces:
            ex.traces = C.cast(trs, C.POINTER(C.POINTER(C.c_uint8)))
            ex.trace_lens = C.cast(tls, C.POINTER(C.c_uint64))
        out = C.POINTER(Polygons)()
        check(lib().vp_pipeline_run_frames(self.h, C.c_size_t(nf), ptrs, _p(ns, C.c_uint64), _p(R, C.c_double),
                                           _p(t, C.c_double), C.c_int(1 if device_ptrs is not None else 0),
                                           C.byref(out), C.byref(ex)))
        res = dict(polygons=polygons_to_py(out))
        if per_frame:
            res["per_frame"] = [polygons_to_py(pf[k]) for k in range(nf)]
        if timings:
            res["timings"] = [tms[k] for k in range(nf)]
        if traces:
            tr = []
            for k in range(nf):
                tr.append(C.string_at(trs[k], tls[k]))
                lib().vp_free(trs[k])
            res["traces"] = tr
        return res

    def run_ptrs(self, ptr_array, n_array, R_array, t_array, device_ptrs, want_polygons, convert=True):
        """Low-overhead vp_pipeline_run on prebuilt ctypes arrays (bench).
        convert=False returns the C result (vp_polygons*) as the ABI hands it
        over; polygons_to_py() turns it into dicts and frees it."""
        out = C.POINTER(Polygons)()
        check(lib().vp_pipeline_run(self.h, C.c_size_t(len(n_array)), ptr_array, _p(n_array, C.c_uint64),
                                    _p(R_array, C.c_double), _p(t_array, C.c_double),
                                    C.c_int(1 if device_ptrs else 0),
                                    C.byref(out) if want_polygons else None, None))
        if not want_polygons:
            return None
        return polygons_to_py(out) if convert else out

    def reset(self, start_center):
        c = np.ascontiguousarray(start_center, np.float64)
        check(lib().vp_pipeline_reset(self.h, _p(c, C.c_double)))

    def counters(self):
        out = np.zeros(16, np.uint64)
        check(lib().vp_pipeline_counters(self.h, _p(out, C.c_uint64)))
        return out

    def frame_device(self, pts_dev_ptr: int, n: int, R, t, want_polygons=False):
        R, t = _pose(R, t)
        out = C.POINTER(Polygons)()
        tm = FrameTiming()
        check(lib().vp_pipeline_frame_device(self.h, C.c_void_p(pts_dev_ptr), C.c_uint64(n),
                                             _p(R, C.c_double), _p(t, C.c_double),
                                             C.byref(out) if want_polygons else None, C.byref(tm)))
        return (polygons_to_py(out) if want_polygons else None), tm

    def frame_trace_raw(self, pts, R, t) -> bytes:
        pts = np.ascontiguousarray(pts, np.float32)
        R, t = _pose(R, t)
        buf = C.POINTER(C.c_uint8)()
        n = C.c_uint64()
        check(lib().vp_pipeline_frame_trace(self.h, _p(pts, C.c_float), C.c_uint64(len(pts)),
                                            _p(R, C.c_double), _p(t, C.c_double), C.byref(buf),
                                            C.byref(n)))
        data = C.string_at(buf, n.value)
        lib().vp_free(buf)
        return data

    def frame_trace(self, pts, R, t):
        from .trace import parse_trace
        return parse_trace(self.frame_trace_raw(pts, R, t))

    @property
    def grid(self) -> "Grid":
        return Grid._borrow(lib().vp_pipeline_grid(self.h))

    def close(self):
        if self.h:
            lib().vp_pipeline_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Grid:
    """VoxelGrid (voxel_grid.hpp:17-91) on the device."""

    def __init__(self, res, extent, center, device=0):
        ext = np.asarray(extent, np.int32)
        c = np.asarray(center, np.float64)
        self.h = C.c_void_p()
        self.owned = True
        check(lib().vp_grid_create(C.c_double(res), _p(ext, C.c_int32), _p(c, C.c_double),
                                   C.c_int(device), C.byref(self.h)))

    @classmethod
    def _borrow(cls, h):
        g = cls.__new__(cls)
        g.h = C.c_void_p(h)
        g.owned = False
        return g

    def info(self):
        o = np.zeros(3)
        e = np.zeros(3, np.int32)
        r = C.c_double()
        n = C.c_uint64()
        check(lib().vp_grid_info(self.h, _p(o, C.c_double), _p(e, C.c_int32), C.byref(r), C.byref(n)))
        return dict(origin=o, extent=e, resolution=r.value, occupied_count=n.value)

    def integrate_frame(self, pts, R, t):
        pts = np.ascontiguousarray(pts, np.float32)
        R, t = _pose(R, t)
        st = UpdateStats()
        check(lib().vp_integrate_frame(self.h, _p(pts, C.c_float), C.c_uint64(len(pts)),
                                       _p(R, C.c_double), _p(t, C.c_double), C.byref(st)))
        return st.voxels_touched, st.points_discarded

    def clear_rays(self, pts, R, t):
        pts = np.ascontiguousarray(pts, np.float32)
        R, t = _pose(R, t)
        st = ClearStats()
        check(lib().vp_clear_rays(self.h, _p(pts, C.c_float), C.c_uint64(len(pts)),
                                  _p(R, C.c_double), _p(t, C.c_double), C.byref(st)))
        return st.voxels_cleared, st.voxels_freed

    def recenter(self, c):
        c = np.ascontiguousarray(c, np.float64)
        st = ShiftStats()
        check(lib().vp_recenter(self.h, _p(c, C.c_double), C.byref(st)))
        return tuple(st.shift[:]), st.voxels_dropped

    def merge_point(self, idx, p):
        i = np.asarray(idx, np.int32)
        q = np.asarray(p, np.float64)
        check(lib().vp_merge_point(self.h, _p(i, C.c_int32), _p(q, C.c_double)))

    def cell(self, idx):
        i = np.asarray(idx, np.int32)
        s = np.zeros(3)
        n = C.c_uint32()
        st = C.c_uint8()
        check(lib().vp_get_cell(self.h, _p(i, C.c_int32), _p(s, C.c_double), C.byref(n), C.byref(st)))
        return s, n.value, st.value

    def set_status(self, idx, status):
        i = np.asarray(idx, np.int32)
        check(lib().vp_set_status(self.h, _p(i, C.c_int32), C.c_uint8(status)))

    def occupied_voxels(self):
        o = C.POINTER(Occupied)()
        check(lib().vp_occupied_voxels(self.h, C.byref(o)))
        O = o.contents
        n = O.count
        res = dict(idx=np.ctypeslib.as_array(O.idx, (n, 3)).copy() if n else np.zeros((0, 3), np.int32),
                   mean=np.ctypeslib.as_array(O.mean, (n, 3)).copy() if n else np.zeros((0, 3)),
                   count=np.ctypeslib.as_array(O.npts, (n,)).copy() if n else np.zeros(0, np.uint32),
                   status=np.ctypeslib.as_array(O.status, (n,)).copy() if n else np.zeros(0, np.uint8))
        lib().vp_occupied_free(o)
        return res

    def estimate_normals(self, seg: SegParams):
        e = C.POINTER(Estimates)()
        check(lib().vp_estimate_normals(self.h, C.byref(seg), C.byref(e)))
        E = e.contents
        n = E.count

        def arr(p, shape, dt):
            return np.ctypeslib.as_array(p, shape).copy() if n else np.zeros(shape, dt)
        res = dict(idx=arr(E.idx, (n, 3), np.int32), mean=arr(E.mean, (n, 3), float),
                   normal=arr(E.normal, (n, 3), float), neighbor_count=arr(E.neighbor_count, (n,), np.int32),
                   angle=arr(E.angle_to_up_deg, (n,), float), valid=arr(E.valid, (n,), np.uint8))
        lib().vp_estimates_free(e)
        return res

    def segment(self, params: PipelineParams):
        out = C.POINTER(Polygons)()
        tm = FrameTiming()
        check(lib().vp_segment(self.h, C.byref(params), C.byref(out), C.byref(tm)))
        return polygons_to_py(out), tm

    def close(self):
        if self.h and self.owned:
            lib().vp_grid_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def label_components(st_idx, st_mean, st_normal, seg: SegParams, res: float, device=0):
    n = len(st_idx)
    s = Steppable()
    idx = np.ascontiguousarray(st_idx, np.int32)
    mean = np.ascontiguousarray(st_mean, np.float64)
    nrm = np.ascontiguousarray(st_normal, np.float64)
    s.count = n
    s.idx, s.mean, s.normal = _p(idx, C.c_int32), _p(mean, C.c_double), _p(nrm, C.c_double)
    labels = np.zeros(n, np.int32)
    check(lib().vp_label_components(C.byref(s), C.byref(seg), C.c_double(res), C.c_int(device),
                                    _p(labels, C.c_int32)))
    return labels


def fit_planes(labels, offsets, means, rp: RansacParams, device=0):
    labels = np.ascontiguousarray(labels, np.int32)
    offsets = np.ascontiguousarray(offsets, np.uint64)
    means = np.ascontiguousarray(means, np.float64)
    f = C.POINTER(Fits)()
    check(lib().vp_fit_planes(C.c_size_t(len(labels)), _p(labels, C.c_int32), _p(offsets, C.c_uint64),
                              _p(means, C.c_double), C.byref(rp), C.c_int(device), C.byref(f)))
    F = f.contents
    n = F.count
    offs = np.ctypeslib.as_array(F.offsets, (n + 1,)).copy()
    tot = int(offs[-1]) if n else 0
    inl = np.ctypeslib.as_array(F.inliers, (tot, 3)).copy() if tot else np.zeros((0, 3))
    models = [dict(normal=np.array(F.models[i].normal[:]), offset=F.models[i].offset,
                   inlier_count=F.models[i].inlier_count, label=F.models[i].cluster_label,
                   inliers=inl[offs[i]:offs[i + 1]]) for i in range(n)]
    stats = (F.clusters_skipped_small, F.clusters_unfit)
    lib().vp_fits_free(f)
    return models, stats


class Stream:
    """VXPF frame stream read into pinned host memory (vp_stream_open)."""

    def __init__(self, path: str):
        self.h = C.c_void_p()
        check(lib().vp_stream_open(str(path).encode(), C.byref(self.h)))

    def __len__(self):
        L = lib()
        L.vp_stream_count.restype = C.c_uint64
        return int(L.vp_stream_count(self.h))

    def frame(self, i):
        xyz = C.POINTER(C.c_float)()
        n = C.c_uint64()
        R = np.zeros(9)
        t = np.zeros(3)
        check(lib().vp_stream_frame(self.h, C.c_uint64(i), C.byref(xyz), C.byref(n), _p(R, C.c_double),
                                    _p(t, C.c_double)))
        pts = np.ctypeslib.as_array(xyz, (n.value, 3)).copy() if n.value else np.zeros((0, 3), np.float32)
        return pts, R.reshape(3, 3), t

    def replay(self, pl: "Pipeline", first=0, count=None):
        """run_frames over the stream (vp_pipeline_replay): the last frame's polygons."""
        count = len(self) - first if count is None else count
        out = C.POINTER(Polygons)()
        check(lib().vp_pipeline_replay(pl.h, self.h, C.c_uint64(first), C.c_uint64(count), C.byref(out), None))
        return out

    def close(self):
        if self.h:
            lib().vp_stream_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def write_frames_binary(path, frames):
    """write_frames_binary (frame_io.cpp:74-89) through the library."""
    n = len(frames)
    pts = [np.ascontiguousarray(f.points, np.float32) for f in frames]
    ptrs = (C.c_void_p * max(n, 1))(*[p.ctypes.data for p in pts])
    cnt = np.asarray([len(p) for p in pts], np.uint64)
    R = np.ascontiguousarray(np.stack([np.asarray(f.rotation, np.float64).reshape(9) for f in frames]))
    t = np.ascontiguousarray(np.stack([np.asarray(f.translation, np.float64) for f in frames]))
    check(lib().vp_write_frames_binary(str(path).encode(), C.c_size_t(n), ptrs, _p(cnt, C.c_uint64),
                                       _p(R, C.c_double), _p(t, C.c_double)))


def write_polygons(path, polys_ptr):
    """write_polygons (polygon_io.cpp:30-47) of a vp_polygons_t* through the library."""
    check(lib().vp_write_polygons(str(path).encode(), polys_ptr))


def polygons_struct(polys):
    """A vp_polygons_t view of polygon dicts (normal, offset, label, inlier_count,
    v3d, area); returns (struct, keep-alive list)."""
    arr = (Polygon * max(len(polys), 1))()
    keep = [arr]
    for q, p in zip(arr, polys):
        v = np.ascontiguousarray(p["v3d"], np.float64).reshape(-1, 3)
        v2 = np.ascontiguousarray(p.get("v2d", np.zeros((len(v), 2))), np.float64).reshape(-1, 2)
        keep += [v, v2]
        q.plane.normal[:] = tuple(float(x) for x in p["normal"])
        q.plane.offset = p["offset"]
        q.plane.inlier_count = p["inlier_count"]
        q.plane.cluster_label = p["label"]
        q.nverts = len(v)
        q.area = p["area"]
        q.v3d = v.ctypes.data_as(C.POINTER(C.c_double))
        q.v2d = v2.ctypes.data_as(C.POINTER(C.c_double))
    return Polygons(len(polys), arr), keep


def scene_truth(kind: int, device=0):
    """build_scene's ground-truth polygons (scene_sim.cpp:23-30, 43-114): the
    corner sets through make_polygon on the device."""
    planes = np.zeros(16 * 4)
    corners = np.zeros(16 * 12)
    n = C.c_size_t()
    if lib().vp_scene_truth(C.c_int(kind), _p(planes, C.c_double), _p(corners, C.c_double), C.byref(n)) != 0:
        raise ValueError(f"unknown scene kind {kind}")
    models = [dict(normal=tuple(planes[4 * r:4 * r + 3]), offset=planes[4 * r + 3], inlier_count=0, label=r)
              for r in range(n.value)]
    return make_polygons(models, [corners[12 * r:12 * r + 12].reshape(4, 3) for r in range(n.value)], device=device)


class IoUReport(C.Structure):
    _fields_ = [("truth_count", C.c_uint64), ("detected_count", C.c_uint64), ("matched", C.c_uint64),
                ("unmatched_truth", C.c_uint64), ("unmatched_detected", C.c_uint64), ("mean_iou", C.c_double),
                ("area_weighted_iou", C.c_double)]


class PlaneMatch(C.Structure):
    _fields_ = [("detected_id", C.c_int32), ("truth_id", C.c_int32), ("iou", C.c_double)]


def match_planes(detected, truth, raster_res=0.005, report_path=None, device=0):
    """match_planes (metrics.cpp:114-160) + optional write_iou_report; returns
    (report dict, [(truth_id, detected_id, iou)])."""
    d, kd = polygons_struct(detected)
    t, kt = polygons_struct(truth)
    rep = IoUReport()
    m = (PlaneMatch * max(1, min(len(detected), len(truth))))()
    check(lib().vp_match_planes(C.byref(d), C.byref(t), C.c_double(raster_res), C.c_int(device), C.byref(rep), m))
    if report_path:
        check(lib().vp_write_iou_report(str(report_path).encode(), C.byref(rep), m))
    return ({k: getattr(rep, k) for k, _ in IoUReport._fields_},
            [(m[i].truth_id, m[i].detected_id, m[i].iou) for i in range(rep.matched)])


class HeightMap:
    """The 2.5-D height-map baseline (heightmap.hpp:10-55) on the GPU."""

    def __init__(self, res, extent, center=(0.0, 0.0), device=0):
        e = np.asarray(extent, np.int32)
        c = np.asarray(center, np.float64)
        self.extent = tuple(int(v) for v in extent)
        self.h = C.c_void_p()
        check(lib().vp_heightmap_create(C.c_double(res), _p(e, C.c_int32), _p(c, C.c_double), C.c_int(device),
                                        C.byref(self.h)))

    def integrate(self, pts, R, t):
        """hm_integrate (heightmap.cpp:26-38)."""
        pts = np.ascontiguousarray(pts, np.float32)
        R, t = _pose(R, t)
        check(lib().vp_hm_integrate(self.h, _p(pts, C.c_float), C.c_uint64(len(pts)), _p(R, C.c_double),
                                    _p(t, C.c_double)))

    def cells(self):
        n = self.extent[0] * self.extent[1]
        h = np.zeros(n)
        v = np.zeros(n, np.uint8)
        check(lib().vp_hm_cells(self.h, _p(h, C.c_double), _p(v, C.c_uint8)))
        return h.reshape(self.extent), v.reshape(self.extent).astype(bool)

    def segment(self, params: PipelineParams):
        """hm_segment (heightmap.cpp:40-89) + run_frames' area filter (params.min_polygon_area)."""
        out = C.POINTER(Polygons)()
        check(lib().vp_hm_segment(self.h, C.byref(params), C.byref(out)))
        return polygons_to_py(out)

    def regions(self):
        """(visit sequence, root per cell) of the last segment()."""
        n = self.extent[0] * self.extent[1]
        visit = np.zeros(n, np.uint32)
        root = np.zeros(n, np.int32)
        nv = C.c_uint64()
        check(lib().vp_hm_regions(self.h, _p(visit, C.c_uint32), _p(root, C.c_int32), C.byref(nv)))
        return visit[:nv.value], root.reshape(self.extent)

    def close(self):
        if self.h:
            lib().vp_heightmap_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class AblationConfig(C.Structure):
    _fields_ = [("cluster_counts", C.POINTER(C.c_int32)), ("n_counts", C.c_int32), ("trials", C.c_int32),
                ("points_min", C.c_int32), ("points_max", C.c_int32), ("seed", C.c_uint64),
                ("iterations", C.c_int32), ("inlier_eps", C.c_double), ("device", C.c_int32)]


class AblationRow(C.Structure):
    _fields_ = [("clusters", C.c_int32), ("trials", C.c_int32), ("parallel_ms", C.c_double),
                ("serial_ms", C.c_double), ("parallel_median_ms", C.c_double), ("serial_median_ms", C.c_double)]


def ablation_config(counts=(1, 2, 4, 8, 16), **kw):
    """AblationConfig (pipeline.hpp:65-74) defaults, overridden by keywords."""
    c = AblationConfig()
    lib().vp_default_ablation_config(C.byref(c))
    c._counts = np.ascontiguousarray(counts, np.int32)  # keep alive
    c.cluster_counts = _p(c._counts, C.c_int32)
    c.n_counts = len(counts)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def run_ablation(cfg: AblationConfig, csv_path: str | None = None):
    """run_ablation (pipeline.cpp:304-381) on the device; optional write_ablation_csv."""
    rows = (AblationRow * max(cfg.n_counts, 1))()
    check(lib().vp_run_ablation(C.byref(cfg), rows))
    if csv_path:
        check(lib().vp_write_ablation_csv(csv_path.encode(), rows, C.c_size_t(cfg.n_counts)))
    return [dict(clusters=r.clusters, trials=r.trials, parallel_ms=r.parallel_ms, serial_ms=r.serial_ms,
                 parallel_median_ms=r.parallel_median_ms, serial_median_ms=r.serial_median_ms)
            for r in rows[:cfg.n_counts]]


def ablation_clusters(cfg: AblationConfig, trial: int, count: int):
    """The synthetic clusters of one (trial, count): array (count, M, 3)."""
    m = C.c_int32()
    pts = C.POINTER(C.c_double)()
    check(lib().vp_ablation_clusters(C.byref(cfg), C.c_int32(trial), C.c_int32(count), C.byref(m), C.byref(pts)))
    out = np.ctypeslib.as_array(pts, (count, m.value, 3)).copy()
    lib().vp_free(pts)
    return out


def make_polygons(planes, inlier_sets, directions=16, device=0):
    n = len(planes)
    arr = (Plane * max(n, 1))()
    for i, p in enumerate(planes):
        arr[i].normal[:] = tuple(p["normal"])
        arr[i].offset = p["offset"]
        arr[i].inlier_count = p.get("inlier_count", 0)
        arr[i].cluster_label = p.get("label", -1)
    offs = np.zeros(n + 1, np.uint64)
    offs[1:] = np.cumsum([len(s) for s in inlier_sets])
    pts = np.ascontiguousarray(np.concatenate(inlier_sets) if n else np.zeros((0, 3)), np.float64)
    out = C.POINTER(Polygons)()
    check(lib().vp_make_polygons(C.c_size_t(n), arr, _p(offs, C.c_uint64), _p(pts, C.c_double),
                                 C.c_int(directions), C.c_int(device), C.byref(out)))
    return polygons_to_py(out)


def refine_planes(fits_models, up=(0.0, 0.0, 1.0), exact=False, device=0):
    """refine_plane for a list of dict(normal, offset, inlier_count, label, inliers)."""
    n = len(fits_models)
    f = Fits()
    models = (Plane * max(n, 1))()
    for i, m in enumerate(fits_models):
        models[i].normal[:] = tuple(m["normal"])
        models[i].offset = m["offset"]
        models[i].inlier_count = m["inlier_count"]
        models[i].cluster_label = m["label"]
    offs = np.zeros(n + 1, np.uint64)
    offs[1:] = np.cumsum([len(m["inliers"]) for m in fits_models])
    pts = np.ascontiguousarray(np.concatenate([m["inliers"] for m in fits_models]) if n else np.zeros((0, 3)))
    f.count = n
    f.models = C.cast(models, C.POINTER(Plane))
    f.offsets = _p(offs, C.c_uint64)
    f.inliers = _p(pts, C.c_double)
    out = (Plane * max(n, 1))()
    u = np.asarray(up, np.float64)
    check(lib().vp_refine_planes(C.byref(f), _p(u, C.c_double), C.c_int(1 if exact else 0),
                                 C.c_int(device), out))
    return [(np.array(out[i].normal[:]), out[i].offset) for i in range(n)]


def set_ccl_mode(mode: int) -> None:
    """0 = hook + forward-window unions (default), 1 = neighbour sampling + giant
    skip, 2 = hook + giant skip (identical labels)."""
    check(lib().vp_set_ccl_mode(C.c_int(mode)))


def kernel_launch_count() -> int:
    return int(lib().vp_kernel_launch_count())
