"""GPU tier: the B200 pipeline against the CPU oracle, stage by stage.

Bit-exact bar (integer / index / FP64-ordered work): occupancy, sums, counts,
statuses, occupied list, normals, steppable list, canonical labels, clusters,
RANSAC candidates / winners / inlier sets. With refine_exact the refine sums are
sequential too, so the whole trace (and the golden files) must be byte-equal.
With the default tree-reduced refine the tolerance of north_star applies:
plane normals within 1e-4 rad, offsets within 1e-4 m, hull vertices within
1e-5 m (symmetric Hausdorff).
"""
import numpy as np
import pytest

from cpu_oracles import CpuSession
from paper_2510_01592_b200 import native, scenes
from paper_2510_01592_b200.trace import format_polygons, parse_trace
from workloads import golden_text, run_config

pytestmark = pytest.mark.gpu

NORMAL_TOL = 1e-4   # rad
OFFSET_TOL = 1e-4   # m
VERTEX_TOL = 1e-5   # m


def sessions(name_or_frames, res=None, ext=None, seed=None, exact=True, params=None):
    if isinstance(name_or_frames, str):
        frames, res, ext, seed, _ = run_config(name_or_frames)
    else:
        frames = name_or_frames
    p = params or native.default_params(seed=seed, refine_exact=exact)
    gpu = native.Pipeline(res, ext, frames[0].translation, p)
    ora = CpuSession("oracle", res, ext, frames[0].translation, p)
    return frames, gpu, ora


def diff_sections(a, b):
    """Names of trace fields that differ (for diagnostics)."""
    out = []
    for k in ("cleared", "freed", "touched", "discarded", "recentered", "shift", "dropped", "origin",
              "occupied_count", "skipped", "unfit"):
        if getattr(a, k) != getattr(b, k):
            out.append(f"{k}: gpu={getattr(a, k)} oracle={getattr(b, k)}")
    for k in ("occ_idx", "occ_mean", "occ_count", "occ_status", "normal", "ncount", "valid", "st_idx",
              "st_mean", "st_normal", "labels"):
        x, y = getattr(a, k), getattr(b, k)
        if x.shape != y.shape:
            out.append(f"{k}: shape {x.shape} vs {y.shape}")
        elif x.tobytes() != y.tobytes():
            bad = np.nonzero((x != y).reshape(len(x), -1).any(axis=1))[0]
            out.append(f"{k}: {len(bad)} rows differ, first {bad[:5].tolist()}")
    if a.clusters != b.clusters:
        out.append(f"clusters: {a.clusters[:6]} vs {b.clusters[:6]}")
    if len(a.fits) != len(b.fits):
        out.append(f"fits: {len(a.fits)} vs {len(b.fits)}")
    else:
        for i, (x, y) in enumerate(zip(a.fits, b.fits)):
            if (x["inlier_count"], x["label"]) != (y["inlier_count"], y["label"]) or \
                    x["normal"].tobytes() != y["normal"].tobytes() or x["offset"] != y["offset"] or \
                    x["inliers"].tobytes() != y["inliers"].tobytes():
                out.append(f"fit {i} differs")
    return out


def check_bit_exact(frames, gpu, ora):
    for i, f in enumerate(frames):
        a = gpu.frame_trace_raw(f.points, f.rotation, f.translation)
        b = ora.frame_raw(f.points, f.rotation, f.translation)
        if a != b:
            d = diff_sections(parse_trace(a), parse_trace(b))
            pytest.fail(f"frame {i}: trace differs: {d}")
    return parse_trace(a)


@pytest.mark.parametrize("name", ["t1", "smallobs"])
def test_trace_bit_exact_and_golden(name):
    frames, gpu, ora = sessions(name)
    last = check_bit_exact(frames, gpu, ora)
    assert format_polygons(last.polygons) == golden_text(run_config(name)[4])


@pytest.mark.parametrize("name", ["stair", "rosette"])
def test_golden_files_reproduced(name):
    frames, res, ext, seed, run = run_config(name)
    gpu = native.Pipeline(res, ext, frames[0].translation, native.default_params(seed=seed, refine_exact=True))
    polys = None
    for f in frames:
        polys, _ = gpu.frame(f.points, f.rotation, f.translation)
    assert format_polygons(polys) == golden_text(run)


@pytest.mark.parametrize("ccl_mode", [0, 1, 2, 3, 4], ids=["pairs_ccl", "sampling_ccl", "hook_giant_ccl", "hook_rows_ccl", "hook_union_ccl"])
def test_stair_every_stage_bit_exact(ccl_mode):
    native.set_ccl_mode(ccl_mode)
    try:
        frames, gpu, ora = sessions("stair")
        check_bit_exact(frames[:12], gpu, ora)
    finally:
        native.set_ccl_mode(0)


def test_ccl_pair_table_overflow_falls_back_to_full_union():
    # k_ccl_pairs lists cross-tree root pairs in a table; when it overflows the
    # full union runs instead (VP_CCL_PAIR_CAP forces a 2-slot table)
    import os
    import subprocess
    import sys
    code = ("import sys; sys.path[:0] = ['tests', '.']; "
            "import test_gpu_parity as t; "
            "frames, gpu, ora = t.sessions('stair'); t.check_bit_exact(frames[:8], gpu, ora); print('ok')")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, VP_CCL_PAIR_CAP="2"))
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-3000:]


def many_patch_frame(n_side=47, spacing=0.08):
    """One synthetic frame of n_side^2 separate 3x3-voxel floor patches
    (2 points per voxel) seen from 0.5 m above: every patch is its own
    steppable cluster (spacing > distance_th)."""
    from types import SimpleNamespace
    pts = []
    for i in range(n_side):
        for j in range(n_side):
            cx, cy = -1.9 + spacing * i, -1.9 + spacing * j
            for dx in (-1, 0, 1):
                for dy in (-1, 0, 1):
                    for q in (-0.002, 0.002):
                        pts.append((cx + 0.01 * dx + q, cy + 0.01 * dy - q, 0.004 + q))
    t = np.array([0.0, 0.0, 0.5])  # the window is centred on the first pose: z in [-0.1, 1.1)
    pts = np.asarray(pts, np.float64) - t
    return SimpleNamespace(points=np.ascontiguousarray(pts, np.float32), rotation=np.eye(3), translation=t)


def test_more_clusters_than_initial_capacity():
    # 2209 clusters in one frame (> the 2048 the buffers start with): the
    # cluster-sized buffers grow and the chain re-runs; the trace (clusters,
    # RANSAC fits, inlier sets, refined planes, polygons) equals the oracle's
    f = many_patch_frame()
    p = native.default_params(seed=3, refine_exact=True, min_area=1e-6)
    p.seg.min_cluster_size = 5
    frames, gpu, ora = sessions([f, f], 0.01, (400, 400, 120), 3, params=p)
    t = check_bit_exact(frames, gpu, ora)
    assert len(t.clusters) == 47 * 47 and len(t.fits) > 2048 and len(t.polygons) > 2048


def test_more_clusters_than_capacity_pipelined():
    # the same frames through vp_pipeline_run: the overflowing frame's chain is
    # grown and re-run when its slot is harvested; traces equal the frame path
    f = many_patch_frame()
    p = native.default_params(seed=3, refine_exact=True, min_area=1e-6)
    p.seg.min_cluster_size = 5
    frames = [f, f, f]
    a = native.Pipeline(0.01, (400, 400, 120), f.translation, p)
    out = a.run_frames(frames, traces=True)
    b = native.Pipeline(0.01, (400, 400, 120), f.translation, p)
    for k, fr in enumerate(frames):
        assert out["traces"][k] == b.frame_trace_raw(fr.points, fr.rotation, fr.translation), f"frame {k}"


def hausdorff(a, b):
    d = np.linalg.norm(a[:, None, :] - b[None, :, :], axis=2)
    return max(d.min(axis=1).max(), d.min(axis=0).max())


def check_tolerance(ta, tb):
    # everything up to the RANSAC fits is bit-exact in either refine mode
    assert diff_sections(ta, tb) == []
    for (na, oa), (nb, ob) in zip(ta.refined, tb.refined):
        ang = np.arccos(np.clip(np.dot(na, nb), -1.0, 1.0))
        assert ang <= NORMAL_TOL and abs(oa - ob) <= OFFSET_TOL
    assert [(p["label"], p["inlier_count"]) for p in ta.polygons] == \
           [(p["label"], p["inlier_count"]) for p in tb.polygons]
    for pa, pb in zip(ta.polygons, tb.polygons):
        assert hausdorff(pa["v3d"], pb["v3d"]) <= VERTEX_TOL
        assert abs(pa["area"] - pb["area"]) <= 1e-4 * max(1.0, pb["area"])


@pytest.mark.parametrize("name", ["t1", "stair"])
def test_tree_refine_within_tolerance(name):
    frames, gpu, ora = sessions(name, exact=False)
    for f in frames:
        ta = gpu.frame_trace(f.points, f.rotation, f.translation)
        tb = ora.frame(f.points, f.rotation, f.translation)
        check_tolerance(ta, tb)


def test_stepping_stones_reduced_window_bit_exact():
    # C2 scene and sensor, 0.01 m, a 240^3 window so the oracle stays fast
    wl = scenes.workload("c2", frames=8)
    frames, gpu, ora = sessions(wl.frames, 0.01, (240, 240, 240), 2025)
    last = check_bit_exact(frames, gpu, ora)
    assert len(last.polygons) >= 2


def test_c2_full_size_first_frames_bit_exact():
    # BASELINE configs[1] at its full 500^3 window: first frames vs the oracle
    wl = scenes.workload("c2", frames=30)
    frames, gpu, ora = sessions(wl.frames[:3], 0.01, (500, 500, 500), 2025)
    check_bit_exact(frames, gpu, ora)


def test_c2_full_stream_properties_and_determinism():
    # size-independent properties over the whole 30-frame stream at 500^3:
    # run-to-run bitwise determinism, label canonicality, polygon invariants.
    wl = scenes.workload("c2")
    p = native.default_params(seed=2025)
    runs = []
    for _ in range(2):
        gpu = native.Pipeline(0.01, (500, 500, 500), wl.frames[0].translation, p)
        traces = [gpu.frame_trace_raw(f.points, f.rotation, f.translation) for f in wl.frames]
        runs.append(traces)
        gpu.close()
    assert runs[0] == runs[1]
    t = parse_trace(runs[0][-1])
    assert t.occupied_count == len(t.occ_idx)
    flat = (t.occ_idx[:, 0].astype(np.int64) * 500 + t.occ_idx[:, 1]) * 500 + t.occ_idx[:, 2]
    assert np.all(np.diff(flat) > 0)                    # lexicographic order
    lab = t.labels
    assert np.all(lab <= np.arange(len(lab)))           # label = component minimum ordinal
    assert np.all(lab[lab] == lab)                      # roots are fixed points
    labels = [p["label"] for p in t.polygons]
    assert labels == sorted(labels) and len(labels) >= 6
    for poly in t.polygons:
        assert poly["area"] >= 0.002
        v = poly["v2d"]
        a, b = np.roll(v, -1, 0) - v, np.roll(v, -2, 0) - np.roll(v, -1, 0)
        cr = a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0]
        assert np.all(cr > 0)                           # strictly convex, CCW


@pytest.mark.parametrize("name", ["t1", "stair"])
def test_pipelined_run_equals_per_frame(name):
    # vp_pipeline_run overlaps consecutive frames; outputs must equal the
    # frame-by-frame path and the golden file (exact refine)
    frames, res, ext, seed, run = run_config(name)
    p = native.default_params(seed=seed, refine_exact=True)
    a = native.Pipeline(res, ext, frames[0].translation, p)
    polys_run = a.run(frames)
    b = native.Pipeline(res, ext, frames[0].translation, p)
    for f in frames:
        polys_frame, _ = b.frame(f.points, f.rotation, f.translation)
    assert format_polygons(polys_run) == format_polygons(polys_frame) == golden_text(run)
    oa, ob = a.grid.occupied_voxels(), b.grid.occupied_voxels()
    for k in oa:
        assert oa[k].tobytes() == ob[k].tobytes()


def test_pipelined_run_c2_matches_frames_and_device_inputs():
    import torch
    wl = scenes.workload("c2", frames=12)
    p = native.default_params(seed=wl.seed)
    a = native.Pipeline(wl.resolution, wl.extent, wl.frames[0].translation, p)
    dev = [torch.from_numpy(f.points).cuda() for f in wl.frames]
    polys_dev, tms = a.run(wl.frames, device_ptrs=[(d.data_ptr(), len(d)) for d in dev], timings=True)
    assert all(t.total_ms > 0 for t in tms)
    b = native.Pipeline(wl.resolution, wl.extent, wl.frames[0].translation, p)
    polys_host = b.run(wl.frames)
    c = native.Pipeline(wl.resolution, wl.extent, wl.frames[0].translation, p)
    for f in wl.frames:
        polys_frame, _ = c.frame(f.points, f.rotation, f.translation)
    assert format_polygons(polys_dev) == format_polygons(polys_host) == format_polygons(polys_frame)
    # a second run continues from the map state, like further run_frames iterations
    more = scenes.workload("c2", frames=30).frames[12:16]
    a2 = a.run(more, device_ptrs=None)
    for f in more:
        polys_frame, _ = c.frame(f.points, f.rotation, f.translation)
    assert format_polygons(a2) == format_polygons(polys_frame)


def test_pipelined_run_regrows_capacities():
    """LiDAR frames of ~1 M points: the occupancy bound of the frames in
    flight exceeds the initial 4 M-voxel capacity, so vp_pipeline_run grows
    every segmentation context mid-run and re-captures its graphs; the result
    must still equal the frame-by-frame path."""
    import torch
    wl = scenes.workload("c4", frames=8)
    p = native.default_params(seed=wl.seed)
    a = native.Pipeline(wl.resolution, wl.extent, wl.frames[0].translation, p)
    dev = [torch.from_numpy(f.points).cuda() for f in wl.frames]
    assert sum(len(d) for d in dev[:5]) > (1 << 22)  # frames in flight + the known occupancy
    polys_run = a.run(wl.frames, device_ptrs=[(d.data_ptr(), len(d)) for d in dev])
    b = native.Pipeline(wl.resolution, wl.extent, wl.frames[0].translation, p)
    for f in wl.frames:
        polys_frame, _ = b.frame(f.points, f.rotation, f.translation)
    assert format_polygons(polys_run) == format_polygons(polys_frame)
