"""Per-kernel device time of a workload's frame stream (the library's event
profile: one kernel at a time, so shares, not pipelined spans).
usage: python tools/kernel_profile.py --workload c4 [--frames 10] [--top 20]"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2510_01592_b200 import native, scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--frames", type=int, default=10)
    ap.add_argument("--top", type=int, default=20)
    a = ap.parse_args()
    wl = scenes.workload(a.workload, frames=a.frames)
    pl = native.Pipeline(wl.resolution, wl.extent, wl.frames[0].translation, native.default_params(seed=wl.seed))
    dev = [torch.from_numpy(f.points).cuda() for f in wl.frames]
    L = native.lib()
    for f, d in zip(wl.frames[:2], dev[:2]):  # warm-up (allocations, graphs)
        pl.frame_device(d.data_ptr(), len(f.points), f.rotation, f.translation)
    pl.reset(wl.frames[0].translation)
    torch.cuda.synchronize()
    L.vp_profile_enable(1)
    for f, d in zip(wl.frames, dev):
        pl.frame_device(d.data_ptr(), len(f.points), f.rotation, f.translation)
    names = (C.c_char_p * 128)()
    ms = (C.c_double * 128)()
    calls = (C.c_uint64 * 128)()
    nk = L.vp_profile_read(names, ms, calls, 128)
    L.vp_profile_enable(0)
    rows = sorted(((ms[i], calls[i], names[i].decode()) for i in range(nk)), reverse=True)
    tot = sum(r[0] for r in rows)
    nf = len(wl.frames)
    print(f"{a.workload}: {nf} frames, {sum(len(f.points) for f in wl.frames) / nf:.0f} points/frame, "
          f"{tot / nf:.3f} ms/frame serialised")
    for t, c, n in rows[:a.top]:
        print(f"{n:28s} {1e3 * t / nf:9.1f} us/frame {100 * t / tot:5.1f}%  calls {c}")


if __name__ == "__main__":
    main()
