"""C5 probe: the 2000x2000x300 window over K virtual slabs on one GPU.

Prints per-frame wall time of each phase and checks that 1 and K virtual
slabs give identical polygons (usage: python tools/c5_probe.py --frames 6 --slabs 1 4).
--library: the library-orchestrated frame (vp_slab_frame_local, one host
thread per virtual slab) instead of the Python model of the protocol.
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2510_01592_b200 import native, scenes, slabs  # noqa: E402
from paper_2510_01592_b200.trace import format_polygons  # noqa: E402


def run(wl, k, params, library=False):
    ranges = slabs.split_x(wl.extent[0], k)
    ss = [slabs.Slab(wl.resolution, wl.extent, scenes.C5_CENTER, a, b) for a, b in ranges]
    comm = slabs.LocalComm(k)
    out = None
    for i, f in enumerate(wl.frames):
        pts = torch.from_numpy(f.points).cuda()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if library:
            out = slabs.frame_local(ss, pts, f.rotation, f.translation, params)
            torch.cuda.synchronize()
            print(f"library slabs={k} frame {i}: {len(f.points)} pts, {len(out)} polygons, "
                  f"{1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
            continue
        st = {}
        out = slabs.slab_frame(ss, comm, pts, f.rotation, f.translation, params, stages=st)
        torch.cuda.synchronize()
        print(f"slabs={k} frame {i}: {len(f.points)} pts, {len(out)} polygons, {1e3 * (time.perf_counter() - t0):.2f} ms"
              f" | steppable {st['steppable']} zone {st['zone']} exported {st['exported']} | {st['phase_ms']}",
              flush=True)
    for s in ss:
        s.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=6)
    ap.add_argument("--slabs", type=int, nargs="+", default=[1, 4])
    ap.add_argument("--library", action="store_true")
    a = ap.parse_args()
    wl = scenes.workload("c5", frames=a.frames)
    params = native.default_params(seed=wl.seed)
    outs = [format_polygons(run(wl, k, params, a.library)) for k in a.slabs]
    print("identical:", all(o == outs[0] for o in outs))


if __name__ == "__main__":
    main()
