"""The reference's own test runs (proj/tests/test_pipeline.cpp) as frame
streams, rendered by the library's frame source (pinned to the reference's
render_frame by test_oracle.py), plus the golden polygon files they produced."""
import os

from paper_2510_01592_b200 import scenes
from paper_2510_01592_b200.frames import read_frames

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_text(run):
    return open(os.path.join(GOLDEN, f"{run}.polygons_final.txt")).read()


def tiny_fixture_frames():
    return read_frames(os.path.join(GOLDEN, "tiny_frames.bin"))


def run_config(name):
    """(frames, resolution, extent, seed, golden run dir) of a reference test run."""
    if name == "t1":  # test_pipeline.cpp:15-26, :168-181
        return tiny_fixture_frames(), 0.01, (140, 140, 140), 77, "pipe_t1"
    if name == "smallobs":  # :55-62
        sensor = scenes.SensorSpec(width=160, height=120)
        poses = scenes.default_trajectory(scenes.SMALL_OBSTACLE, 10, 20.0)
        return scenes.render(scenes.stock_scene(scenes.SMALL_OBSTACLE), sensor, poses, 77), 0.01, (140, 140, 140), 77, "pipe_smallobs"
    if name == "stair":  # :77-88
        return scenes.stair_frames(25), 0.01, (200, 200, 200), 5, "pipe_stair"
    if name == "rosette":  # :110-121
        sensor = scenes.SensorSpec(kind=1, pattern=scenes.rosette_pattern(12000))
        poses = scenes.default_trajectory(scenes.SMALL_OBSTACLE, 30, 20.0)
        return scenes.render(scenes.stock_scene(scenes.SMALL_OBSTACLE), sensor, poses, 5), 0.01, (200, 200, 200), 5, "pipe_rosette"
    raise ValueError(name)
