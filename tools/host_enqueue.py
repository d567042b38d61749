"""Is the pipelined run host-bound? Wall time of vp_pipeline_run over the C2
stream (device inputs) against the device span measured with CUDA events, and
the host time spent enqueueing (the call returns after the last harvest)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_01592_b200 import native, scenes  # noqa: E402

wl = scenes.workload("c2")
pl = native.Pipeline(wl.resolution, wl.extent, wl.frames[0].translation, native.default_params(seed=wl.seed))
dev = [torch.from_numpy(f.points).cuda() for f in wl.frames]
ptrs = (C.c_void_p * len(dev))(*[d.data_ptr() for d in dev])
n = np.asarray([len(f.points) for f in wl.frames], np.uint64)
R = np.ascontiguousarray(np.stack([f.rotation.reshape(9) for f in wl.frames]))
t = np.ascontiguousarray(np.stack([f.translation for f in wl.frames]))
L = native.lib()
for rep in range(4):
    pl.reset(wl.frames[0].translation)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h0 = time.perf_counter()
    native.check(L.vp_pipeline_run(pl.h, C.c_size_t(len(dev)), ptrs, native._p(n, C.c_uint64),
                                   native._p(R, C.c_double), native._p(t, C.c_double), 1, None, None))
    h1 = time.perf_counter()
    e1.record()
    e1.synchronize()
    print(f"rep {rep}: host wall {1e3 * (h1 - h0):.3f} ms, device (events around the call) "
          f"{e0.elapsed_time(e1):.3f} ms for {len(dev)} frames")
