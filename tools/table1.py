"""Table I at scale: the voxel-map pipeline against the
2.5-D height-map baseline (heightmap.cpp:26-89) on the same streams, both on
the GPU: frames/s and plane IoU of the final polygons against build_scene's
ground truth (metrics.cpp:114-160, scored on the device).

Streams: the stock Stair5 and Overhang scenes (scene_sim.cpp:43-114) seen by
the C2 sensor (640x480 pinhole, 6 m) along their default trajectories, 30
frames at 30 Hz; 0.01 m voxels in a 500^3 window, a 500^2 height map.
usage: python tools/table1.py [--frames 30] [--out profiles/r01_table1.txt]"""
import argparse
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_01592_b200 import native, scenes  # noqa: E402


def voxel_run(frames, params, reps=3):
    pl = native.Pipeline(0.01, (500, 500, 500), frames[0].translation, params)
    dev = [torch.from_numpy(np.ascontiguousarray(f.points)).cuda() for f in frames]
    ptrs = [(d.data_ptr(), len(f.points)) for d, f in zip(dev, frames)]
    polys, best = None, None
    for _ in range(reps):
        pl.reset(frames[0].translation)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        polys = pl.run(frames, device_ptrs=ptrs, want_polygons=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return len(frames) / best, polys


def heightmap_run(frames, params, reps=3):
    c = frames[0].translation
    polys, best = None, None
    for _ in range(reps):
        hm = native.HeightMap(0.01, (500, 500), (float(c[0]), float(c[1])))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for f in frames:  # run_frames' baseline branch: integrate, then segment every frame
            hm.integrate(f.points, f.rotation, f.translation)
            polys = hm.segment(params)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
        hm.close()
    return len(frames) / best, polys


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=30)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    sensor = scenes.SensorSpec(width=640, height=480, max_range=6.0)
    lines = ["# Table I at scale: GPU voxel pipeline vs GPU height-map baseline, same streams "
             f"({a.frames} frames, 640x480, 0.01 m); frames/s = whole stream incl. per-frame segmentation, "
             "IoU = final polygons vs build_scene truth (device raster 5 mm)",
             f"{'scene':10s} {'method':10s} {'frames/s':>9s} {'polygons':>8s} {'matched':>7s} "
             f"{'mean IoU':>8s} {'area-w IoU':>10s}"]
    for name, kind in (("stair5", scenes.STAIR5), ("overhang", scenes.OVERHANG)):
        frames = scenes.render(scenes.stock_scene(kind), sensor,
                               scenes.default_trajectory(kind, a.frames, 30.0), 2025)
        params = native.default_params(seed=2025)
        truth = native.scene_truth(kind)
        for method, fn in (("voxel", voxel_run), ("heightmap", heightmap_run)):
            fps, polys = fn(frames, params)
            rep, _ = native.match_planes(polys, truth)
            lines.append(f"{name:10s} {method:10s} {fps:9.1f} {len(polys):8d} {rep['matched']:7d} "
                         f"{rep['mean_iou']:8.3f} {rep['area_weighted_iou']:10.3f}")
            print(lines[-1], flush=True)
    if a.out:
        with open(a.out, "w") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
