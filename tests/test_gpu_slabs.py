"""GPU tier: spatial slabs as N virtual slabs on one device.

A fixed window driven with clear_rays + integrate_frame per frame and then
segmented must give the same steppable list (bit-exact) and the same polygons
whether it lives in one grid or in N slab grids with halo exchange and the
distributed segmentation (local CCL + boundary-label merge + cluster gather
to the owning slab) -- the multi-GPU path's correctness argument, checked on
1 GPU. The merged labels must equal the single-grid canonical labels."""
import numpy as np
import pytest
import torch

from paper_2510_01592_b200 import native, scenes, slabs
from paper_2510_01592_b200.trace import format_polygons

pytestmark = pytest.mark.gpu

RES = 0.01
EXTENT = (300, 200, 150)        # x in [-1.5, 1.5), y in [-1, 1), z in [-0.25, 1.25)
CENTER = (0.0, 0.0, 0.5)


def one_grid(frames, params):
    g = native.Grid(RES, EXTENT, CENTER)
    polys = None
    for f in frames:
        pts = np.ascontiguousarray(f.points, np.float32)
        R, t = f.rotation.reshape(9), f.translation
        cs, us = native.ClearStats(), native.UpdateStats()
        native.check(native.lib().vp_update_frame(g.h, native._p(pts, native.C.c_float),
                                                  native.C.c_uint64(len(pts)),
                                                  native._p(np.ascontiguousarray(R), native.C.c_double),
                                                  native._p(np.ascontiguousarray(t), native.C.c_double),
                                                  native.C.byref(cs), native.C.byref(us)))
        polys, _ = g.segment(params)
    return g, polys


def steppable_normals(g, params):
    from ctypes import POINTER, byref, c_size_t, c_int32
    st = POINTER(native.Steppable)()
    objs = POINTER(c_int32)()
    nobj = c_size_t()
    native.check(native.lib().vp_classify_steppable(g.h, byref(params.seg), byref(st), byref(objs), byref(nobj)))
    S = st.contents.count
    nrm = np.ctypeslib.as_array(st.contents.normal, (S, 3)).copy()
    native.lib().vp_steppable_free(st)
    native.lib().vp_free(objs)
    return nrm


def steppable_of_grid(g, params):
    from ctypes import POINTER, byref, c_size_t, c_int32
    st = POINTER(native.Steppable)()
    objs = POINTER(c_int32)()
    nobj = c_size_t()
    native.check(native.lib().vp_classify_steppable(g.h, byref(params.seg), byref(st), byref(objs), byref(nobj)))
    S = st.contents.count
    idx = np.ctypeslib.as_array(st.contents.idx, (S, 3)).copy()
    mean = np.ctypeslib.as_array(st.contents.mean, (S, 3)).copy()
    native.lib().vp_steppable_free(st)
    native.lib().vp_free(objs)
    return idx, mean


@pytest.mark.parametrize("ranges", [[(0, 300)], [(0, 150), (150, 300)], [(0, 37), (37, 150), (150, 151), (151, 300)],
                                    [(0, 100), (100, 102), (102, 104), (104, 200), (200, 300)],
                                    [(a, a + 38) for a in range(0, 266, 38)] + [(266, 300)]])
def test_virtual_slabs_equal_one_grid(ranges):
    check_slabs(ranges, scenes.stair_frames(10))


@pytest.mark.parametrize("ranges", [[(0, 150), (150, 300)], [(0, 100), (100, 102), (102, 104), (104, 200), (200, 300)]])
def test_virtual_slabs_lidar(ranges):
    """Incoherent rays: the slab walk's brick-mask path (owned-range marking,
    rays dropped once they left the slab) against the one-grid walk."""
    check_slabs(ranges, scenes.lidar_stair_frames(6))


def check_slabs(ranges, frames):
    params = native.default_params(seed=5, refine_exact=True)
    g, ref_polys = one_grid(frames, params)
    ref_idx, ref_mean = steppable_of_grid(g, params)
    sl = [slabs.Slab(RES, EXTENT, CENTER, a, b) for a, b in ranges]
    comm = slabs.LocalComm(len(sl))
    polys = None
    for f in frames:
        pts = torch.from_numpy(np.ascontiguousarray(f.points)).cuda()
        polys = slabs.slab_frame(sl, comm, pts, f.rotation, f.translation, params)
    # the merged labels of the last frame (kept by each slab) == single-grid canonical labels
    labels = np.concatenate([s.merge_labels().cpu().numpy() for s in sl])
    parts = [s.steppable(params.seg) for s in sl]
    S = sum(p[0] for p in parts)
    idx = torch.cat([p[1][0] for p in parts]).cpu().numpy().view(np.int32).reshape(S, 3)
    mean = torch.cat([p[1][1] for p in parts]).cpu().numpy().view(np.float64).reshape(S, 3)
    assert np.array_equal(idx, ref_idx) and mean.tobytes() == ref_mean.tobytes()
    ref_labels = native.label_components(ref_idx, ref_mean, steppable_normals(g, params), params.seg, RES)
    assert np.array_equal(labels, ref_labels)
    assert len(ref_polys) >= 3
    assert format_polygons(polys) == format_polygons(ref_polys)


def check_slabs_library(ranges, frames, device_points=True):
    """The library-orchestrated frame (vp_slab_frame_local: one host thread per
    slab, the exchanges as device copies) gives the one-grid polygons."""
    params = native.default_params(seed=5, refine_exact=True)
    _, ref_polys = one_grid(frames, params)
    sl = [slabs.Slab(RES, EXTENT, CENTER, a, b) for a, b in ranges]
    polys = None
    for f in frames:
        pts = torch.from_numpy(np.ascontiguousarray(f.points)).cuda() if device_points else f.points
        polys = slabs.frame_local(sl, pts, f.rotation, f.translation, params)
    assert len(ref_polys) >= 3
    assert format_polygons(polys) == format_polygons(ref_polys)
    for s in sl:
        s.close()


@pytest.mark.parametrize("ranges", [[(0, 300)], [(0, 150), (150, 300)], [(0, 37), (37, 150), (150, 151), (151, 300)],
                                    [(a, a + 38) for a in range(0, 266, 38)] + [(266, 300)]])
def test_library_slab_frame_equals_one_grid(ranges):
    check_slabs_library(ranges, scenes.stair_frames(10))


def test_library_slab_frame_lidar_host_points():
    check_slabs_library([(0, 100), (100, 102), (102, 104), (104, 200), (200, 300)], scenes.lidar_stair_frames(6),
                        device_points=False)


def test_library_slab_frame_reports_bad_layout():
    # x ranges that do not tile the window: every slab thread fails, the first error is reported
    params = native.default_params(seed=5)
    sl = [slabs.Slab(RES, EXTENT, CENTER, 0, 100), slabs.Slab(RES, EXTENT, CENTER, 120, 300)]
    f = scenes.stair_frames(1)[0]
    with pytest.raises(native.InvalidArgument, match="tile the window"):
        slabs.frame_local(sl, f.points, f.rotation, f.translation, params)


def test_slab_window_is_fixed():
    s = slabs.Slab(RES, EXTENT, CENTER, 0, 100)
    from ctypes import byref
    st = native.ShiftStats()
    c = np.array([0.5, 0.0, 0.5])
    rc = native.lib().vp_recenter(s.h, native._p(c, native.C.c_double), byref(st))
    assert rc == native.VP_EINVAL
