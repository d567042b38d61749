"""GPU tier: plane IoU scoring (metrics.cpp:19-185)
against the reference's golden IoU reports: the final polygons of the
reference's own test runs, scored against build_scene's ground truth
(scene_sim.cpp:23-30, 43-114), must produce its iou_report.txt byte for byte;
plus a closed-form unit case."""
import numpy as np
import pytest

from paper_2510_01592_b200 import native, scenes
from paper_2510_01592_b200.frames import read_frames
from workloads import GOLDEN, run_config

pytestmark = pytest.mark.gpu


def golden_report(run):
    return open(f"{GOLDEN}/{run}.iou_report.txt").read()


def final_polygons(name):
    frames, res, ext, seed, _ = run_config(name)
    pl = native.Pipeline(res, ext, frames[0].translation, native.default_params(seed=seed, refine_exact=True))
    polys = None
    for f in frames:
        polys, _ = pl.frame(f.points, f.rotation, f.translation)
    return polys


@pytest.mark.parametrize("name,run,kind", [("t1", "pipe_t1", scenes.SMALL_OBSTACLE),
                                           ("smallobs", "pipe_smallobs", scenes.SMALL_OBSTACLE),
                                           ("stair", "pipe_stair", scenes.STAIR5),
                                           ("rosette", "pipe_rosette", scenes.SMALL_OBSTACLE)])
def test_iou_report_reproduces_golden(tmp_path, name, run, kind):
    truth = native.scene_truth(kind)
    native.match_planes(final_polygons(name), truth, report_path=tmp_path / "iou_report.txt")
    assert (tmp_path / "iou_report.txt").read_text() == golden_report(run)


def test_baseline_iou_report_reproduces_golden(tmp_path):
    frames = read_frames(f"{GOLDEN}/baseline_frames.bin")
    hm = native.HeightMap(0.01, (140, 140), (0.0, 0.0))
    p = native.default_params(seed=77, refine_exact=True)
    for f in frames:
        hm.integrate(f.points, f.rotation, f.translation)
        polys = hm.segment(p)
    native.match_planes(polys, native.scene_truth(scenes.SMALL_OBSTACLE), report_path=tmp_path / "r.txt")
    assert (tmp_path / "r.txt").read_text() == golden_report("pipe_baseline")


def square(x0, y0, s, z=0.0, label=0):
    v = np.array([[x0, y0, z], [x0 + s, y0, z], [x0 + s, y0 + s, z], [x0, y0 + s, z]])
    return dict(normal=np.array([0.0, 0.0, 1.0]), offset=z, inlier_count=0, label=label, v3d=v, area=s * s)


def test_iou_closed_form_and_gate():
    # two unit squares overlapping by half: IoU = 0.5 / 1.5 (raster 0.005 m is exact here)
    rep, m = native.match_planes([square(0.5, 0.0, 1.0)], [square(0.0, 0.0, 1.0)])
    assert rep["matched"] == 1 and abs(m[0][2] - 1.0 / 3.0) < 1e-9
    # a wall is gated out by the 20 degree normal test
    wall = square(0.0, 0.0, 1.0)
    wall["normal"] = np.array([1.0, 0.0, 0.0])
    rep, m = native.match_planes([wall], [square(0.0, 0.0, 1.0)])
    assert rep["matched"] == 0 and rep["unmatched_truth"] == 1 and rep["mean_iou"] == 0.0
