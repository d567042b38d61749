"""Per-kernel device time of one pass over a workload's stream (serialised
launches with CUDA events; shares only) and the wall time of a normal pass
(usage: python tools/stream_profile.py --workload c1)."""
import argparse
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_01592_b200 import native, scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c1")
    ap.add_argument("--frames", type=int, default=0)
    a = ap.parse_args()
    wl = scenes.workload(a.workload, frames=a.frames or None)
    pl = native.Pipeline(wl.resolution, wl.extent, wl.frames[0].translation, native.default_params(seed=wl.seed))
    dev = [torch.from_numpy(f.points).cuda() for f in wl.frames]
    L = native.lib()
    for rep in range(3):
        pl.reset(wl.frames[0].translation)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for f, d in zip(wl.frames, dev):
            pl.frame_device(d.data_ptr(), len(f.points), f.rotation, f.translation)
        torch.cuda.synchronize()
        print(f"pass {rep}: {1e3 * (time.perf_counter() - t0) / len(wl.frames):.3f} ms/frame (frame-by-frame API)")
    pl.reset(wl.frames[0].translation)
    L.vp_profile_enable(1)
    for f, d in zip(wl.frames, dev):
        pl.frame_device(d.data_ptr(), len(f.points), f.rotation, f.translation)
    names = (C.c_char_p * 128)()
    ms = (C.c_double * 128)()
    calls = (C.c_uint64 * 128)()
    nk = L.vp_profile_read(names, ms, calls, 128)
    L.vp_profile_enable(0)
    prof = sorted(((names[i].decode(), ms[i], calls[i]) for i in range(nk)), key=lambda r: -r[1])
    tot = sum(r[1] for r in prof)
    nf = len(wl.frames)
    print(f"{a.workload}: {nf} frames, kernel sum {tot / nf:.3f} ms/frame")
    for n, m, c in prof[:20]:
        print(f"  {n:24s} {1e3 * m / nf:9.1f} us/frame  {c / nf:.1f} launches/frame  {100 * m / tot:5.1f}%")
    print("counters", pl.counters())


if __name__ == "__main__":
    main()
