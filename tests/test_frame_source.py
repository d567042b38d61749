"""GPU tier: the device frame source (render_frame on the GPU, SURVEY §8(f)
row 1) against the host frame source, which test_oracle.py pins to the
reference's render_frame byte for byte. Same hit set and order; points equal
to the byte unless an ulp of the device log/cos survives the f32 rounding,
which these streams never show."""
import numpy as np
import pytest

from paper_2510_01592_b200 import scenes

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,frames", [("c2", 3), ("c3", 2), ("c4", 1), ("c5", 1)])
def test_device_frames_equal_host_frames(name, frames):
    w = scenes.workload_spec(name, frames)
    host = scenes.render(w.scene, w.sensor, w.poses, w.seed)
    src = scenes.DeviceFrameSource(w.scene, w.sensor, w.seed)
    for i, (pose, h) in enumerate(zip(w.poses, host)):
        d = src.render(pose, i)
        assert d.rotation.tobytes() == h.rotation.tobytes() and d.translation.tobytes() == h.translation.tobytes()
        assert d.points.shape == h.points.shape, f"frame {i}: {len(d.points)} vs {len(h.points)} hits"
        diff = np.nonzero((d.points != h.points).any(axis=1))[0]
        assert len(diff) == 0, f"frame {i}: {len(diff)} of {len(h.points)} points differ, first {diff[:5]}"


def test_device_frames_drive_the_pipeline_identically():
    from paper_2510_01592_b200 import native
    from paper_2510_01592_b200.trace import format_polygons
    w = scenes.workload_spec("c2", 4)
    host = scenes.render(w.scene, w.sensor, w.poses, w.seed)
    src = scenes.DeviceFrameSource(w.scene, w.sensor, w.seed)
    p = native.default_params(seed=w.seed)
    a = native.Pipeline(w.resolution, w.extent, host[0].translation, p)
    b = native.Pipeline(w.resolution, w.extent, host[0].translation, p)
    for i, (pose, h) in enumerate(zip(w.poses, host)):
        pa, _ = a.frame(h.points, h.rotation, h.translation)
        ptr, n, R, t = src.render_ptr(pose, i)
        b.frame_device(ptr, n, R, t)
    pb, _ = b.frame(np.zeros((0, 3), np.float32), R, t)  # flush: an empty frame at the same pose
    pa, _ = a.frame(np.zeros((0, 3), np.float32), R, t)
    assert format_polygons(pa) == format_polygons(pb)
