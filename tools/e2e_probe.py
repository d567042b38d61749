"""e2e gap probe: the C2 stream through vp_pipeline_run with device-resident
vs pinned-host points, with and without the final polygons (frames/s,
median of the last 4 of 6 runs).
usage: python tools/e2e_probe.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_01592_b200 import native, scenes  # noqa: E402


def main():
    wl = scenes.workload("c2")
    fr = wl.frames
    nf = len(fr)
    pl = native.Pipeline(wl.resolution, wl.extent, fr[0].translation, native.default_params(seed=wl.seed))
    L = native.lib()
    L.vp_pipeline_stream.restype = C.c_void_p
    stream = torch.cuda.ExternalStream(L.vp_pipeline_stream(pl.h))
    R = np.ascontiguousarray(np.stack([f.rotation.reshape(9) for f in fr]), np.float64)
    t = np.ascontiguousarray(np.stack([f.translation for f in fr]), np.float64)
    n = np.asarray([len(f.points) for f in fr], np.uint64)
    dev = [torch.from_numpy(f.points).cuda() for f in fr]
    host = [torch.from_numpy(f.points).pin_memory() for f in fr]
    dev_ptrs = (C.c_void_p * nf)(*[d.data_ptr() for d in dev])
    host_ptrs = (C.c_void_p * nf)(*[h.data_ptr() for h in host])
    start = np.ascontiguousarray(fr[0].translation, np.float64)

    def rate(ptrs, device_ptrs, want_polygons):
        ms = []
        for _ in range(6):
            L.vp_pipeline_reset(pl.h, start.ctypes.data_as(C.POINTER(C.c_double)))
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            raw = pl.run_ptrs(ptrs, n, R, t, device_ptrs=device_ptrs, want_polygons=want_polygons, convert=False)
            e1.record(stream)
            e1.synchronize()
            if want_polygons:
                native.polygons_to_py(raw)
            ms.append(e0.elapsed_time(e1))
        return nf / (np.median(ms[2:]) / 1e3)

    for name, ptrs, device_ptrs, want in (("device, no polygons", dev_ptrs, True, False),
                                          ("device, polygons", dev_ptrs, True, True),
                                          ("host, no polygons", host_ptrs, False, False),
                                          ("host, polygons", host_ptrs, False, True)):
        print(f"{name:22s} {rate(ptrs, device_ptrs, want):9.1f} frames/s", flush=True)


if __name__ == "__main__":
    main()
