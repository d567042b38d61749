"""Phase timestamps of k_poly_fused (build with -DVP_POLY_PROFILE, run with
VP_LIB=<that build>): per fit, ns from the fit's start to each phase end."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_01592_b200 import native, scenes  # noqa: E402

from paper_2510_01592_b200 import slabs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
if name == "c5":  # one slab over the C5 window, library-orchestrated frames
    wl = scenes.workload("c5", frames=int(sys.argv[2]) if len(sys.argv) > 2 else 6)
    sl = slabs.Slab(wl.resolution, wl.extent, scenes.C5_CENTER, 0, wl.extent[0])
    p = native.default_params(seed=wl.seed)
    for f in wl.frames:
        polys = slabs.frame_local([sl], torch.from_numpy(f.points).cuda(), f.rotation, f.translation, p)
    print("polygons", len(polys), "counters", sl.counters())
else:
    wl = scenes.workload("c2", frames=12)
    pl = native.Pipeline(wl.resolution, wl.extent, wl.frames[0].translation, native.default_params(seed=wl.seed))
    dev = [torch.from_numpy(f.points).cuda() for f in wl.frames]
    for f, d in zip(wl.frames, dev):
        pl.frame_device(d.data_ptr(), len(f.points), f.rotation, f.translation)
out = np.zeros((64, 20), np.uint64)
native.lib().vp_debug_poly_times(out.ctypes.data_as(C.POINTER(C.c_ulonglong)))
names = ["start", "ext+sync", "inner+sync", "keep+sync", "sort", "uniq+chains", "area+lift", "end sync", "proj", "extloop", "warpred", "ctared", "basis"]
for f in range(64):
    if out[f, 0] == 0:
        break
    t = out[f].astype(np.int64) - int(out[f, 0])
    print(f, f"n={int(out[f, 13])} surv={int(out[f, 14])}", " ".join(f"{n}={v / 1e3:.1f}" for n, v in zip(names[1:], t[1:13])),
          f"uniq={t[15] / 1e3:.1f} chains={t[16] / 1e3:.1f}")

if hasattr(native.lib(), "vp_debug_chain_stats"):
    cs = np.zeros(4, np.uint64)
    native.lib().vp_debug_chain_stats(cs.ctypes.data_as(C.POINTER(C.c_ulonglong)))
    print(f"half chains: {int(cs[1])} points, {int(cs[0])} pop tests, {int(cs[2])} cycles "
          f"({cs[2] / max(cs[1], 1):.0f} cycles/point, {cs[2] / max(cs[0], 1):.0f} cycles/test)")
