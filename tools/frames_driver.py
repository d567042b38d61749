"""Run N frames of a workload through the pipeline with device-resident inputs
(for ncu captures: the kernels of frame k can be selected with -s/-c)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_01592_b200 import native, scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--frames", type=int, default=30)
    ap.add_argument("--counters", action="store_true")
    a = ap.parse_args()
    wl = scenes.workload(a.workload)
    pl = native.Pipeline(wl.resolution, wl.extent, wl.frames[0].translation, native.default_params(seed=wl.seed))
    dev = [torch.from_numpy(f.points).cuda() for f in wl.frames]
    names = "cleared freed touched discarded dropped occupied V S K fits padded inliers poolv newly surv_max overflow".split()
    for k in range(a.frames):
        f = wl.frames[k % len(wl.frames)]
        if k and k % len(wl.frames) == 0:
            pl.reset(wl.frames[0].translation)
        _, tm = pl.frame_device(dev[k % len(dev)].data_ptr(), len(f.points), f.rotation, f.translation)
        if a.counters:
            c = pl.counters()
            print(k, len(f.points), " ".join(f"{n}={int(v)}" for n, v in zip(names, c)),
                  f"total_ms={tm.total_ms:.3f}", flush=True)


if __name__ == "__main__":
    main()
