"""Where a single frame's latency goes (one frame in flight, C2 frames 2..29):
library latency (points H2D start -> polygons in host memory) vs the device
span of the frame graph (FrameTiming.total_ms) and the H2D copy alone."""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_01592_b200 import native, scenes  # noqa: E402

wl = scenes.workload("c2")
pl = native.Pipeline(wl.resolution, wl.extent, wl.frames[0].translation, native.default_params(seed=wl.seed))
host = [torch.from_numpy(f.points).pin_memory() for f in wl.frames]
dev = [torch.empty_like(h, device="cuda") for h in host]
L = native.lib()
L.vp_pipeline_latency_ms.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
lat, dspan, h2d, parts = [], [], [], []
ms = C.c_double()
for rep in range(2):
    pl.reset(wl.frames[0].translation)
    for k, f in enumerate(wl.frames):
        polys, tm = pl.frame_ptr(host[k].data_ptr(), len(f.points), f.rotation, f.translation, want_polygons=True)
        native.check(L.vp_pipeline_latency_ms(pl.h, C.byref(ms)))
        if rep == 1 and k >= 2:
            lat.append(ms.value)
            dspan.append(tm.total_ms)
            parts.append((tm.mapping_ms, tm.classify_ms, tm.cluster_ms, tm.ransac_ms, tm.hull_ms))
s = torch.cuda.Stream()
for k in range(2, 30):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record()
        dev[k].copy_(host[k], non_blocking=True)
        e1.record()
    e1.synchronize()
    h2d.append(e0.elapsed_time(e1))
print(f"latency p50 {statistics.median(lat):.4f} ms, device span p50 {statistics.median(dspan):.4f} ms, "
      f"points H2D p50 {statistics.median(h2d):.4f} ms ({len(wl.frames[5].points) * 12 / 1e6:.2f} MB)")
names = ("mapping", "classify", "cluster", "ransac", "refine+hull")
print("device stages p50 (ms): " + ", ".join(f"{n} {statistics.median(p[i] for p in parts):.4f}" for i, n in enumerate(names)))
