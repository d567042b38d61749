"""Stage spans of a pipelined C2 run (VP_PIPE_STATS); --host: pinned host frames."""
import ctypes as C
import os
import sys

os.environ["VP_PIPE_STATS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_01592_b200 import native, scenes  # noqa: E402

wl = scenes.workload("c2")
pl = native.Pipeline(wl.resolution, wl.extent, wl.frames[0].translation, native.default_params(seed=wl.seed))
dev = [torch.from_numpy(f.points).cuda() for f in wl.frames]
host = [torch.from_numpy(f.points).pin_memory() for f in wl.frames]
use_host = "--host" in sys.argv  # pinned host frames (H2D inside the call, copy-ahead)
ptrs = (C.c_void_p * len(dev))(*[(h if use_host else d).data_ptr() for h, d in zip(host, dev)])
n = np.asarray([len(f.points) for f in wl.frames], np.uint64)
R = np.ascontiguousarray(np.stack([f.rotation.reshape(9) for f in wl.frames]))
t = np.ascontiguousarray(np.stack([f.translation for f in wl.frames]))
for rep in range(2):
    pl.reset(wl.frames[0].translation)
    tm = (native.FrameTiming * len(dev))()
    native.check(native.lib().vp_pipeline_run(pl.h, C.c_size_t(len(dev)), ptrs, native._p(n, C.c_uint64),
                                              native._p(R, C.c_double), native._p(t, C.c_double),
                                              0 if use_host else 1, None, tm))
    print("rep", rep, "frame total_ms:", [round(x.total_ms, 3) for x in tm][:10], file=sys.stderr)
