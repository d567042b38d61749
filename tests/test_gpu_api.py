"""GPU tier: the per-stage C ABI against the oracle and the reference's own
unit-test cases (proj/tests/test_voxel_grid.cpp, test_segmentation.cpp,
test_plane_fit.cpp, test_polygonize.cpp)."""
import ctypes as C

import numpy as np
import pytest

from cpu_oracles import CpuSession
from paper_2510_01592_b200 import native

pytestmark = pytest.mark.gpu

I3 = np.eye(3)


def small_grid(res=0.01, n=40):
    # test_voxel_grid.cpp:15-18: window [0, n*res)^3
    return native.Grid(res, (n, n, n), (0.5 * n * res,) * 3)


def test_single_point_fills_empty_voxel():
    g = small_grid()
    p = np.array([[0.105, 0.003, 0.002]], np.float32)
    touched, disc = g.integrate_frame(p, I3, np.zeros(3))
    assert (touched, disc) == (1, 0)
    occ = g.occupied_voxels()
    assert occ["count"].tolist() == [1]
    assert occ["idx"].tolist() == [[10, 0, 0]]
    assert np.array_equal(occ["mean"][0], p[0].astype(np.float64))


def test_nan_and_out_of_bounds_are_discarded():
    g = small_grid()
    pts = np.array([[np.nan, 0.1, 0.1], [0.1, 0.1, 0.1], [5.0, 0.1, 0.1], [-0.001, 0.1, 0.1]], np.float32)
    touched, disc = g.integrate_frame(pts, I3, np.zeros(3))
    assert (touched, disc) == (1, 3)


def test_invalid_rotation_raises():
    g = small_grid()
    R = np.diag([1.0, 1.0, 2.0])
    with pytest.raises(native.InvalidArgument):
        g.integrate_frame(np.zeros((1, 3), np.float32), R, np.zeros(3))
    with pytest.raises(native.InvalidArgument):
        g.clear_rays(np.zeros((1, 3), np.float32), R, np.zeros(3))


def test_axis_ray_frees_exactly_interior_cells():
    # test_voxel_grid.cpp:157-169: ray from cell 0 to cell 10 along x frees 1..9
    g = small_grid()
    fill = np.array([[0.005 + 0.01 * i, 0.055, 0.055] for i in range(11)], np.float32)
    g.integrate_frame(fill, I3, np.zeros(3))
    sensor = np.array([0.005, 0.055, 0.055])
    end = np.array([[0.105 - 0.005, 0.0, 0.0]], np.float32)  # sensor-frame offset
    cleared, freed = g.clear_rays(end, I3, sensor)
    assert cleared == 9 and freed == 9
    idx = g.occupied_voxels()["idx"].tolist()
    assert idx == [[0, 5, 5], [10, 5, 5]]


def test_shared_voxels_freed_once():
    g = small_grid()
    fill = np.array([[0.005 + 0.01 * i, 0.055, 0.055] for i in range(11)], np.float32)
    g.integrate_frame(fill, I3, np.zeros(3))
    ends = np.array([[0.1, 0.0, 0.0], [0.1, 0.0, 0.0004], [0.1, 0.0004, 0.0]], np.float32)
    cleared, freed = g.clear_rays(ends, I3, np.array([0.005, 0.055, 0.055]))
    assert freed == 9 and cleared == 9


def test_random_rays_match_oracle_grid_state():
    rng = np.random.default_rng(7)
    p = native.default_params()
    g = native.Pipeline(0.01, (40, 40, 40), (0.2, 0.2, 0.2), p)
    o = CpuSession("oracle", 0.01, (40, 40, 40), (0.2, 0.2, 0.2), p)
    for k in range(6):
        pts = rng.uniform(-0.25, 0.25, (400, 3)).astype(np.float32)
        t = np.array([0.2, 0.2, 0.2]) + rng.uniform(-0.004, 0.004, 3)
        a = g.frame_trace_raw(pts, I3, t)
        b = o.frame_raw(pts, I3, t)
        assert a == b, f"frame {k}"


@pytest.mark.parametrize("dense", [3000, 20000])
def test_dense_voxels_fold_in_index_order(dense):
    # voxels with > 128 points (k_integrate_fold_dense: shared-memory sort up to
    # 16384 points, ordered stream beyond) must fold in ascending point index
    rng = np.random.default_rng(dense)
    parts = [rng.uniform(0.25, 0.30, (dense, 3)), rng.uniform([0.10, 0.15, 0.20], [0.15, 0.20, 0.25], (700, 3)),
             rng.uniform(0.35, 0.40, (150, 3)), rng.uniform(0.0, 0.5, (60, 3))]
    pts = np.concatenate(parts).astype(np.float32)
    pts = pts[rng.permutation(len(pts))]
    p = native.default_params()
    g = native.Pipeline(0.05, (10, 10, 10), (0.25, 0.25, 0.25), p)
    o = CpuSession("oracle", 0.05, (10, 10, 10), (0.25, 0.25, 0.25), p)
    t = np.array([0.26, 0.27, 0.28])
    for k in range(2):
        assert g.frame_trace_raw(pts, I3, t) == o.frame_raw(pts, I3, t), f"frame {k}"


def test_c1_frame_bit_exact():
    # BASELINE configs[0]: Stair5 640x480 at 0.05 m (~160 points per voxel)
    from paper_2510_01592_b200 import scenes
    wl = scenes.workload("c1")
    f = wl.frames[0]
    p = native.default_params(seed=wl.seed, refine_exact=True)
    g = native.Pipeline(wl.resolution, wl.extent, f.translation, p)
    o = CpuSession("oracle", wl.resolution, wl.extent, f.translation, p)
    assert g.frame_trace_raw(f.points, f.rotation, f.translation) == o.frame_raw(f.points, f.rotation, f.translation)


def test_recenter_shift_and_drop():
    # test_voxel_grid.cpp:225-237: shift (3,0,0) moves cell (10,5,5) to (7,5,5)
    g = small_grid()
    g.integrate_frame(np.array([[0.105, 0.055, 0.055], [0.015, 0.055, 0.055]], np.float32), I3, np.zeros(3))
    shift, dropped = g.recenter((0.2 + 0.03, 0.2, 0.2))
    assert shift == (3, 0, 0) and dropped == 1
    occ = g.occupied_voxels()
    assert occ["idx"].tolist() == [[7, 5, 5]]
    s, n, st = g.cell((7, 5, 5))
    assert n == 1 and abs(s[0] - np.float32(0.105)) < 1e-12
    shift, dropped = g.recenter((0.2 + 0.03 + 1.0, 0.2, 0.2))
    assert dropped == 1 and g.occupied_voxels()["idx"].shape[0] == 0


def test_recenter_commutes_with_integrate():
    rng = np.random.default_rng(3)
    pts = rng.uniform(-0.2, 0.2, (2000, 3)).astype(np.float32)
    t0 = np.array([0.2, 0.2, 0.2])
    a = small_grid()
    a.clear_rays(pts, I3, t0)
    a.integrate_frame(pts, I3, t0)
    a.recenter((0.2 + 0.05, 0.2 - 0.02, 0.2 + 0.07))
    ma = a.occupied_voxels()
    # oracle order: integrate, recenter
    p = native.default_params()
    o = CpuSession("oracle", 0.01, (40, 40, 40), (0.2, 0.2, 0.2), p)
    # the oracle session recenters on a global-cell change; drive it with two frames
    o.frame_raw(pts, I3, t0)
    t = o.frame(np.zeros((0, 3), np.float32), I3, np.array([0.25, 0.18, 0.27]))
    assert t.shift == (5, -2, 7)
    assert np.array_equal(ma["idx"], t.occ_idx) and ma["mean"].tobytes() == t.occ_mean.tobytes()


def test_occupied_voxels_lexicographic():
    rng = np.random.default_rng(1)
    g = small_grid()
    g.integrate_frame(rng.uniform(0, 0.4, (3000, 3)).astype(np.float32), I3, np.zeros(3))
    idx = g.occupied_voxels()["idx"].astype(np.int64)
    flat = (idx[:, 0] * 40 + idx[:, 1]) * 40 + idx[:, 2]
    assert np.all(np.diff(flat) > 0)


def test_empty_grid_normals_raise():
    g = small_grid()
    with pytest.raises(native.VpError) as e:
        g.estimate_normals(native.default_params().seg)
    assert e.value.code == native.VP_EEMPTY


def test_horizontal_patch_normals():
    # test_segmentation.cpp:49-70: a flat patch gives +z normals, angle 0
    g = small_grid()
    xs, ys = np.meshgrid(np.arange(5, 30) * 0.01 + 0.005, np.arange(5, 30) * 0.01 + 0.005)
    pts = np.stack([xs.ravel(), ys.ravel(), np.full(xs.size, 0.105)], 1).astype(np.float32)
    g.integrate_frame(pts, I3, np.zeros(3))
    est = g.estimate_normals(native.default_params().seg)
    inner = (est["neighbor_count"] == 9)
    assert inner.sum() > 100
    assert np.allclose(est["normal"][inner], [0, 0, 1], atol=1e-6)
    assert np.all(est["angle"][inner] < 1e-3)


def random_steppable(rng, n, spread):
    idx = rng.integers(0, spread, (n, 3)).astype(np.int32)
    idx = np.unique(idx, axis=0)
    flat = (idx[:, 0].astype(np.int64) * 10000 + idx[:, 1]) * 10000 + idx[:, 2]
    idx = idx[np.argsort(flat)]
    mean = (idx + 0.5) * 0.01 + rng.normal(0, 0.003, idx.shape)
    nrm = np.tile([0.0, 0.0, 1.0], (len(idx), 1)) + rng.normal(0, 0.15, idx.shape)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    return idx, mean, nrm


@pytest.fixture(params=[0, 1, 2, 3, 4], ids=["pairs_ccl", "sampling_ccl", "hook_giant_ccl", "hook_rows_ccl", "hook_union_ccl"])
def ccl_mode(request):
    native.set_ccl_mode(request.param)
    yield request.param
    native.set_ccl_mode(0)


@pytest.mark.parametrize("seed", range(6))
def test_label_components_matches_oracle(seed, ccl_mode):
    rng = np.random.default_rng(seed)
    idx, mean, nrm = random_steppable(rng, 3000 if seed < 3 else 12000, 30)
    seg = native.default_params().seg
    got = native.label_components(idx, mean, nrm, seg, 0.01)
    L = CpuSession.load("oracle")
    exp = np.zeros(len(idx), np.int32)
    L.oracle_label_components(C.c_size_t(len(idx)), idx.ctypes.data_as(C.POINTER(C.c_int32)),
                              mean.ctypes.data_as(C.POINTER(C.c_double)),
                              nrm.ctypes.data_as(C.POINTER(C.c_double)), C.byref(seg), C.c_double(0.01),
                              exp.ctypes.data_as(C.POINTER(C.c_int32)))
    assert np.array_equal(got, exp)


def test_label_components_widest_window_and_limit():
    """w = ceil(distance_th / res) = 15 (a window row of 31 cells, the widest one
    bitmap span holds) matches the oracle; w > 15 fails loudly."""
    rng = np.random.default_rng(7)
    idx, mean, nrm = random_steppable(rng, 2000, 40)
    seg = native.default_params().seg
    seg.distance_th = 0.149
    got = native.label_components(idx, mean, nrm, seg, 0.01)
    L = CpuSession.load("oracle")
    exp = np.zeros(len(idx), np.int32)
    L.oracle_label_components(C.c_size_t(len(idx)), idx.ctypes.data_as(C.POINTER(C.c_int32)),
                              mean.ctypes.data_as(C.POINTER(C.c_double)),
                              nrm.ctypes.data_as(C.POINTER(C.c_double)), C.byref(seg), C.c_double(0.01),
                              exp.ctypes.data_as(C.POINTER(C.c_int32)))
    assert np.array_equal(got, exp)
    seg.distance_th = 0.2
    with pytest.raises(native.InvalidArgument):
        native.label_components(idx, mean, nrm, seg, 0.01)


def planar_steppable(rng):
    """~300k voxels: a 520 x 520 noisy floor with holes, a raised 200 x 120 table
    patch and clutter -- a giant component plus many small ones."""
    fx, fy = np.meshgrid(np.arange(520), np.arange(520), indexing="ij")
    keep = rng.random(fx.shape) > 0.12
    fz = 40 + (rng.random(fx.shape) < 0.2).astype(int)
    floor = np.stack([fx[keep], fy[keep], fz[keep]], 1)
    tx, ty = np.meshgrid(np.arange(100, 300), np.arange(50, 170), indexing="ij")
    table = np.stack([tx.ravel(), ty.ravel(), np.full(tx.size, 115)], 1)
    clutter = np.stack([rng.integers(0, 520, 4000), rng.integers(0, 520, 4000), rng.integers(60, 110, 4000)], 1)
    idx = np.unique(np.concatenate([floor, table, clutter]).astype(np.int32), axis=0)
    mean = (idx + 0.5) * 0.01 + rng.normal(0, 0.002, idx.shape)
    nrm = np.tile([0.0, 0.0, 1.0], (len(idx), 1)) + rng.normal(0, 0.05, idx.shape)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    return idx, mean, nrm


def test_label_components_large_planar_matches_oracle(ccl_mode):
    # the sampling CCL's giant-component path at scale (C5 has ~1M steppable voxels)
    rng = np.random.default_rng(11)
    idx, mean, nrm = planar_steppable(rng)
    seg = native.default_params().seg
    got = native.label_components(idx, mean, nrm, seg, 0.01)
    L = CpuSession.load("oracle")
    exp = np.zeros(len(idx), np.int32)
    L.oracle_label_components(C.c_size_t(len(idx)), idx.ctypes.data_as(C.POINTER(C.c_int32)),
                              mean.ctypes.data_as(C.POINTER(C.c_double)),
                              nrm.ctypes.data_as(C.POINTER(C.c_double)), C.byref(seg), C.c_double(0.01),
                              exp.ctypes.data_as(C.POINTER(C.c_int32)))
    assert len(np.unique(exp)) > 100
    assert np.array_equal(got, exp)


def test_two_clusters_labels():
    # test_segmentation.cpp:235-248: two separated patches -> labels {0, 5}
    idx = np.array([[0, 0, 0], [0, 0, 1], [0, 1, 0], [1, 0, 0], [1, 1, 0],
                    [20, 20, 0], [20, 21, 0], [21, 20, 0]], np.int32)
    mean = (idx + 0.5) * 0.01
    nrm = np.tile([0.0, 0.0, 1.0], (len(idx), 1))
    got = native.label_components(idx, mean, nrm, native.default_params().seg, 0.01)
    assert sorted(set(got.tolist())) == [0, 5]


def oracle_fit(labels, offsets, means, rp):
    L = CpuSession.load("oracle")
    nc = len(labels)
    models = (native.Plane * max(nc, 1))()
    fitted = np.zeros(nc, np.uint8)
    inl = np.zeros((offsets[-1], 3))
    nin = np.zeros(nc, np.uint64)
    sk, uf = C.c_uint64(), C.c_uint64()
    L.oracle_fit_planes(C.c_size_t(nc), labels.ctypes.data_as(C.POINTER(C.c_int32)),
                        offsets.ctypes.data_as(C.POINTER(C.c_uint64)), means.ctypes.data_as(C.POINTER(C.c_double)),
                        C.byref(rp), models, fitted.ctypes.data_as(C.POINTER(C.c_uint8)),
                        inl.ctypes.data_as(C.POINTER(C.c_double)), nin.ctypes.data_as(C.POINTER(C.c_uint64)),
                        C.byref(sk), C.byref(uf))
    out = []
    for c in range(nc):
        if fitted[c]:
            m = models[c]
            out.append(dict(normal=np.array(m.normal[:]), offset=m.offset, inlier_count=m.inlier_count,
                            label=m.cluster_label, inliers=inl[offsets[c]:offsets[c] + nin[c]]))
    return out, (sk.value, uf.value)


def test_fit_planes_matches_oracle_bitwise():
    rng = np.random.default_rng(11)
    sizes = [2, 40, 1, 500, 3, 2000, 75]
    means, labels, offs = [], [], [0]
    for c, m in enumerate(sizes):
        n = rng.normal(size=3)
        n /= np.linalg.norm(n)
        pts = rng.uniform(-0.5, 0.5, (m, 3))
        pts -= np.outer(pts @ n, n)
        pts += np.outer(rng.normal(0, 0.004, m), n) + rng.uniform(-1, 1, 3)
        if c == 4:  # collinear -> every sample degenerate (unfit)
            pts = np.outer(np.linspace(0, 1, m), [1.0, 2.0, 3.0])
        means.append(pts)
        labels.append(c * 7 + 1)
        offs.append(offs[-1] + m)
    means = np.concatenate(means)
    labels = np.array(labels, np.int32)
    offs = np.array(offs, np.uint64)
    rp = native.default_params(seed=99).ransac
    got, gstats = native.fit_planes(labels, offs, means, rp)
    exp, estats = oracle_fit(labels, offs, means, rp)
    assert gstats == estats == (2, 1)
    assert len(got) == len(exp)
    for a, b in zip(got, exp):
        assert (a["label"], a["inlier_count"]) == (b["label"], b["inlier_count"])
        assert a["normal"].tobytes() == b["normal"].tobytes() and a["offset"] == b["offset"]
        assert a["inliers"].tobytes() == b["inliers"].tobytes()


def test_refine_exact_and_tree():
    rng = np.random.default_rng(5)
    fits = []
    for m in (3, 10, 1000, 30000):
        pts = rng.uniform(-0.5, 0.5, (m, 3))
        pts[:, 2] = 0.3 + 0.01 * pts[:, 0] + rng.normal(0, 0.002, m)
        fits.append(dict(normal=np.array([0, 0, 1.0]), offset=0.3, inlier_count=m, label=m, inliers=pts))
    L = CpuSession.load("oracle")
    ex = native.refine_planes(fits, exact=True)
    tr = native.refine_planes(fits, exact=False)
    for f, (ne, oe), (nt, ot) in zip(fits, ex, tr):
        init = native.Plane()
        init.normal[:] = tuple(f["normal"])
        init.offset = f["offset"]
        out = native.Plane()
        pts = np.ascontiguousarray(f["inliers"])
        L.oracle_refine_plane(C.c_size_t(len(pts)), pts.ctypes.data_as(C.POINTER(C.c_double)), C.byref(init),
                              np.array([0, 0, 1.0]).ctypes.data_as(C.POINTER(C.c_double)), C.byref(out))
        assert ne.tobytes() == np.array(out.normal[:]).tobytes() and oe == out.offset
        assert np.arccos(np.clip(ne @ nt, -1, 1)) <= 1e-4 and abs(oe - ot) <= 1e-4


def _oracle_polygon(L, pl, pts):
    P = native.Plane()
    P.normal[:] = tuple(pl["normal"])
    P.offset = pl["offset"]
    v2 = np.zeros(2 * len(pts))
    v3 = np.zeros(3 * len(pts))
    area = C.c_double()
    pts = np.ascontiguousarray(pts, float)
    nv = L.oracle_make_polygon(C.byref(P), C.c_size_t(len(pts)), pts.ctypes.data_as(C.POINTER(C.c_double)),
                               16, v2.ctypes.data_as(C.POINTER(C.c_double)),
                               v3.ctypes.data_as(C.POINTER(C.c_double)), C.byref(area))
    return nv, v2[:2 * nv], v3[:3 * nv], area.value


def test_make_polygon_large_fits_vs_oracle():
    """Fits above the wide-pass threshold (16 384 inliers: chunked extremes
    and keep test over the grid) next to small ones, with exact ties: lattice
    points put many points on the same extreme line (key-reduction and
    lexicographic tie-breaks), duplicated points, and survivor sets on both
    sides of the rank-sort (512) and shared-memory (1024) limits."""
    rng = np.random.default_rng(21)
    L = CpuSession.load("oracle")
    planes, sets = [], []

    def add(pts, normal=(0, 0, 1.0), offset=0.0):
        n = np.asarray(normal, float)
        planes.append(dict(normal=n / np.linalg.norm(n), offset=offset, inlier_count=len(pts), label=len(planes)))
        sets.append(np.ascontiguousarray(pts, float))

    g = np.stack(np.meshgrid(np.arange(150), np.arange(140), indexing="ij"), -1).reshape(-1, 2) * 0.01
    add(np.c_[g, np.zeros(len(g))])                                   # 21 000-point lattice square
    disk = g[((g - 0.7) ** 2).sum(1) < 0.49]
    add(np.c_[disk, np.full(len(disk), 0.3)], offset=0.3)             # lattice disk: hundreds of survivors
    add(np.r_[np.c_[g, np.zeros(len(g))], np.c_[g, np.zeros(len(g))]])  # every point twice
    add(rng.normal(size=(70000, 3)), normal=(0.3, -0.2, 0.9), offset=0.1)
    add(rng.uniform(-1, 1, (150000, 3)), normal=(1.0, 0.0, 0.0))
    add(rng.normal(size=(300, 3)))                                    # a small fit beside them
    theta = rng.uniform(0, 2 * np.pi, 40000)
    add(np.c_[np.cos(theta), np.sin(theta), np.zeros(40000)])         # points on a circle: every point survives
    got = native.make_polygons(planes, sets)
    assert len(got) == len(planes)
    for pl, pts, gp in zip(planes, sets, got):
        nv, v2, v3, area = _oracle_polygon(L, pl, pts)
        assert len(gp["v2d"]) == nv
        if nv:
            assert gp["v2d"].tobytes() == v2.tobytes()
            assert gp["v3d"].tobytes() == v3.tobytes()
            assert gp["area"] == area


def test_make_polygon_square_and_vs_oracle():
    # test_polygonize.cpp:105-117: unit square -> CCW from the lex-min vertex, area 1
    sq = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [0.5, 0.5, 0], [0.25, 0.75, 0]], float)
    plane = dict(normal=np.array([0, 0, 1.0]), offset=0.0, inlier_count=6, label=0)
    poly = native.make_polygons([plane], [sq])[0]
    assert poly["v3d"].shape == (4, 3) and abs(poly["area"] - 1.0) < 1e-12
    rng = np.random.default_rng(9)
    L = CpuSession.load("oracle")
    planes, sets = [], []
    for k in range(40):
        m = int(rng.integers(3, 6000))
        n = rng.normal(size=3)
        n /= np.linalg.norm(n)
        if n[2] < 0:
            n = -n
        pts = rng.normal(size=(m, 3)) if k % 3 else rng.uniform(-1, 1, (m, 3))
        planes.append(dict(normal=n, offset=float(rng.uniform(-1, 1)), inlier_count=m, label=k))
        sets.append(pts)
    sets.append(np.outer(np.linspace(0, 1, 10), [1, 0, 0.0]))   # collinear -> nullopt
    planes.append(dict(normal=np.array([0, 0, 1.0]), offset=0.0, inlier_count=10, label=99))
    got = native.make_polygons(planes, sets)
    assert len(got) == len(planes)
    for pl, pts, g in zip(planes, sets, got):
        P = native.Plane()
        P.normal[:] = tuple(pl["normal"])
        P.offset = pl["offset"]
        v2 = np.zeros(2 * len(pts))
        v3 = np.zeros(3 * len(pts))
        area = C.c_double()
        pts = np.ascontiguousarray(pts, float)
        nv = L.oracle_make_polygon(C.byref(P), C.c_size_t(len(pts)), pts.ctypes.data_as(C.POINTER(C.c_double)),
                                   16, v2.ctypes.data_as(C.POINTER(C.c_double)),
                                   v3.ctypes.data_as(C.POINTER(C.c_double)), C.byref(area))
        assert len(g["v2d"]) == nv
        if nv:
            assert g["v2d"].tobytes() == v2[:2 * nv].tobytes()
            assert g["v3d"].tobytes() == v3[:3 * nv].tobytes()
            assert g["area"] == area.value
