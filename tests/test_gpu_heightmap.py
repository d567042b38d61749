"""GPU tier: the height-map baseline (heightmap.cpp)
against the reference's own unit cases (proj/tests/test_heightmap.cpp) and its
golden end-to-end output: the baseline run of test_pipeline.cpp:183-192
replayed from the reference's emitted stream must write
pipe_baseline/polygons_final.txt byte for byte."""
import math

import numpy as np
import pytest

from paper_2510_01592_b200 import native
from paper_2510_01592_b200.frames import read_frames
from paper_2510_01592_b200.trace import format_polygons
from workloads import GOLDEN, golden_text

pytestmark = pytest.mark.gpu

I3 = np.eye(3)


def small_map():
    # test_heightmap.cpp:16-19: 0.01 m, 120 x 120 around the origin
    return native.HeightMap(0.01, (120, 120), (0.0, 0.0))


def cell_of(hm, x, y):
    return int(math.floor((x + 0.6) / 0.01)), int(math.floor((y + 0.6) / 0.01))


def test_point_writes_its_height():
    hm = small_map()
    hm.integrate(np.array([[0.1, 0.1, 0.3]], np.float32), I3, np.zeros(3))
    h, v = hm.cells()
    i, j = cell_of(hm, 0.1, 0.1)
    assert v[i, j] and abs(h[i, j] - 0.3) < 1e-6 and v.sum() == 1


def test_latest_measurement_wins():
    hm = small_map()
    hm.integrate(np.array([[0.05, 0.05, 0.0]], np.float32), I3, np.zeros(3))
    hm.integrate(np.array([[0.05, 0.05, 0.5]], np.float32), I3, np.zeros(3))
    i, j = cell_of(hm, 0.05, 0.05)
    assert abs(hm.cells()[0][i, j] - 0.5) < 1e-6  # the overhang overwrote the floor
    # same cell, same frame: the last point of the stream wins (also among many)
    pts = np.array([[0.05, 0.05, 0.2]] * 1000 + [[0.05, 0.05, 0.1]], np.float32)
    hm.integrate(pts, I3, np.zeros(3))
    assert abs(hm.cells()[0][i, j] - 0.1) < 1e-6


def test_empty_and_out_of_bounds_change_nothing():
    hm = small_map()
    hm.integrate(np.zeros((0, 3), np.float32), I3, np.zeros(3))
    hm.integrate(np.array([[9.0, 9.0, 1.0], [np.nan, 0.0, 0.0]], np.float32), I3, np.zeros(3))
    assert not hm.cells()[1].any()


def floor_points(stage=False):
    pts = []
    for x in range(120):
        for y in range(120):
            wx, wy = -0.6 + 0.01 * (x + 0.5), -0.6 + 0.01 * (y + 0.5)
            on = stage and 0.1 < wx < 0.5 and -0.2 < wy < 0.2
            pts.append((wx, wy, 0.2 if on else 0.0))
    return np.array(pts, np.float32)


def test_flat_floor_one_covering_polygon():
    hm = small_map()
    hm.integrate(floor_points(), I3, np.zeros(3))
    p = native.default_params(seed=3, min_area=-math.inf)
    polys = hm.segment(p)
    assert len(polys) == 1
    assert abs(polys[0]["area"] - 1.44) < 0.05 * 1.44 and abs(polys[0]["normal"][2] - 1.0) < 1e-6


def test_single_stage_two_regions():
    hm = small_map()
    hm.integrate(floor_points(stage=True), I3, np.zeros(3))
    polys = hm.segment(native.default_params(seed=4, min_area=-math.inf))
    assert len(polys) == 2
    assert sorted(round(p["offset"], 3) for p in polys) == [0.0, 0.2]


def test_baseline_run_reproduces_golden():
    # test_pipeline.cpp:183-192: tiny_config with run.baseline = true, 4 frames;
    # the map is a fixed window around the scene origin (pipeline.cpp:167-170)
    frames = read_frames(f"{GOLDEN}/baseline_frames.bin")
    assert len(frames) == 4
    hm = native.HeightMap(0.01, (140, 140), (0.0, 0.0))
    p = native.default_params(seed=77, refine_exact=True)
    polys = None
    for f in frames:
        hm.integrate(f.points, f.rotation, f.translation)
        polys = hm.segment(p)
    assert format_polygons(polys) == golden_text("pipe_baseline")


def py_regions(h, v, dth):
    """heightmap.cpp:44-79 restated: BFS region growing, seeds lexicographic."""
    import collections
    ex, ey = v.shape
    region = -np.ones((ex, ey), np.int64)
    order = []
    for x in range(ex):
        for y in range(ey):
            if not v[x, y] or region[x, y] >= 0:
                continue
            lab = x * ey + y
            q = collections.deque([(x, y)])
            region[x, y] = lab
            while q:
                cx, cy = q.popleft()
                order.append(cx * ey + cy)
                for sx, sy in ((1, 0), (-1, 0), (0, 1), (0, -1)):
                    nx, ny = cx + sx, cy + sy
                    if 0 <= nx < ex and 0 <= ny < ey and v[nx, ny] and region[nx, ny] < 0 \
                            and abs(h[nx, ny] - h[cx, cy]) < dth:
                        region[nx, ny] = lab
                        q.append((nx, ny))
    return order, region


@pytest.mark.parametrize("seed,ex,ey,tx,ty", [(0, 90, 70, 17, 13), (1, 90, 70, 17, 13), (2, 90, 70, 17, 13),
                                              (3, 320, 280, 400, 400)])
def test_regions_and_bfs_order_match_restatement(seed, ex, ey, tx, ty):
    # terraced random map with holes: many regions, long BFS fronts; the flat
    # 320 x 280 case is one region whose fronts reach thousands of (cell, step)
    # pairs per level (several passes of the block-wide BFS kernel per level)
    rng = np.random.default_rng(seed)
    xs, ys = np.meshgrid(np.arange(ex), np.arange(ey), indexing="ij")
    z = 0.03 * ((xs // tx + ys // ty) % 4) + rng.normal(0, 0.004, xs.shape)
    keep = rng.random(xs.shape) > 0.15
    pts = np.stack([(xs + 0.5) * 0.01, (ys + 0.5) * 0.01, z], -1)[keep].astype(np.float32)
    hm = native.HeightMap(0.01, (ex, ey), (ex * 0.005, ey * 0.005))
    hm.integrate(pts, I3, np.zeros(3))
    p = native.default_params(seed=seed, min_area=-math.inf)
    p.seg.distance_th = 0.02
    hm.segment(p)
    h, v = hm.cells()
    visit, root = hm.regions()
    order, region = py_regions(h, v, 0.02)
    assert np.array_equal(np.where(v, root, -1), np.where(v, region, -1))
    by_gpu, by_py = {}, {}
    for c in visit:
        by_gpu.setdefault(int(root.reshape(-1)[c]), []).append(int(c))
    for c in order:
        by_py.setdefault(int(region.reshape(-1)[c]), []).append(int(c))
    assert len(by_py) > (20 if tx < ex else 0) and by_gpu == by_py
