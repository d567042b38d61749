"""e2e gap probe: C2 stream with device vs pinned-host points, with and without
the final polygons (median of 4 runs, frames/s)."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2510_01592_b200 import native, scenes
wl = scenes.workload("c2")
fr = wl.frames; nf = len(fr)
pl = native.Pipeline(wl.resolution, wl.extent, fr[0].translation, native.default_params(seed=wl.seed))
L = native.lib(); L.vp_pipeline_stream.restype = C.c_void_p
stream = torch.cuda.ExternalStream(L.vp_pipeline_stream(pl.h))
R = np.ascontiguousarray(np.stack([f.rotation.reshape(9) for f in fr]), np.float64)
t = np.ascontiguousarray(np.stack([f.translation for f in fr]), np.float64)
n = np.asarray([len(f.points) for f in fr], np.uint64)
dev = [torch.from_numpy(f.points).cuda() for f in fr]
host = [torch.from_numpy(f.points).pin_memory() for f in fr]
dp = (C.c_void_p * nf)(*[d.data_ptr() for d in dev]); hp = (C.c_void_p * nf)(*[h.data_ptr() for h in host])
start = np.ascontiguousarray(fr[0].translation, np.float64)
def run(ptrs, devp, want):
    ts = []
    for _ in range(6):
        L.vp_pipeline_reset(pl.h, start.ctypes.data_as(C.POINTER(C.c_double))); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream); raw = pl.run_ptrs(ptrs, n, R, t, device_ptrs=devp, want_polygons=want, convert=False); e1.record(stream); e1.synchronize()
        if want: native.polygons_to_py(raw)
        ts.append(e0.elapsed_time(e1))
    return nf / (np.median(ts[2:]) / 1e3)
for name, ptrs, devp, want in [("dev nopoly", dp, True, False), ("dev poly", dp, True, True), ("host nopoly", hp, False, False), ("host poly", hp, False, True)]:
    print(name, round(run(ptrs, devp, want), 1))
