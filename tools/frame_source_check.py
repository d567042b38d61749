"""Device vs host frame source: mismatch counts and render times."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_01592_b200 import scenes  # noqa: E402

for name, nf in (("c2", 30), ("c4", 4), ("c5", 2)):
    w = scenes.workload_spec(name, nf)
    t0 = time.time()
    host = scenes.render(w.scene, w.sensor, w.poses, w.seed)
    th = time.time() - t0
    src = scenes.DeviceFrameSource(w.scene, w.sensor, w.seed)
    src.render_ptr(w.poses[0], 0)
    torch.cuda.synchronize()
    bad = tot = 0
    t0 = time.time()
    for i, pose in enumerate(w.poses):
        src.render_ptr(pose, i)
    td = time.time() - t0
    for i, (pose, h) in enumerate(zip(w.poses, host)):
        d = src.render(pose, i)
        tot += len(h.points)
        if d.points.shape != h.points.shape:
            print(name, i, "hit count differs", d.points.shape, h.points.shape)
            continue
        bad += int((d.points != h.points).any(axis=1).sum())
    print(f"{name}: {len(host)} frames, {tot} points, {bad} differ; host render {1e3 * th / len(host):.1f} ms/frame "
          f"(all cores), device {1e3 * td / len(host):.3f} ms/frame")
