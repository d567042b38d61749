"""CCL cross-check on a C5 steppable list: the slab path's merged labels, the
library's label_components in both CCL modes and the C oracle's
label_components must agree (usage: python tools/ccl_check.py --frames 8)."""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from cpu_oracles import CpuSession  # noqa: E402
from paper_2510_01592_b200 import native, scenes, slabs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=8)
    ap.add_argument("--slabs", type=int, default=1)
    a = ap.parse_args()
    wl = scenes.workload("c5", frames=a.frames)
    params = native.default_params(seed=wl.seed)
    ranges = slabs.split_x(wl.extent[0], a.slabs)
    ss = [slabs.Slab(wl.resolution, wl.extent, scenes.C5_CENTER, lo, hi) for lo, hi in ranges]
    comm = slabs.LocalComm(len(ss))
    for f in wl.frames:
        pts = torch.from_numpy(f.points).cuda()
        slabs.slab_frame(ss, comm, pts, f.rotation, f.translation, params)
    labels = np.concatenate([s.merge_labels().cpu().numpy() for s in ss])
    parts = [s.steppable(params.seg) for s in ss]
    S = sum(p[0] for p in parts)
    idx = torch.cat([p[1][0] for p in parts]).cpu().numpy().view(np.int32).reshape(S, 3)
    mean = torch.cat([p[1][1] for p in parts]).cpu().numpy().view(np.float64).reshape(S, 3)
    nrm = torch.cat([p[1][2] for p in parts]).cpu().numpy().view(np.float64).reshape(S, 3)
    print("steppable", S, "slab-path components", len(np.unique(labels)))
    out = {}
    for mode in (0, 1):
        native.set_ccl_mode(mode)
        out[mode] = native.label_components(idx, mean, nrm, params.seg, wl.resolution)
        print(f"mode {mode}: components {len(np.unique(out[mode]))}, "
              f"differs from slab path at {(out[mode] != labels).sum()}")
    native.set_ccl_mode(0)
    L = CpuSession.load("oracle")
    exp = np.zeros(S, np.int32)
    seg = params.seg
    L.oracle_label_components(C.c_size_t(S), idx.ctypes.data_as(C.POINTER(C.c_int32)),
                              mean.ctypes.data_as(C.POINTER(C.c_double)),
                              nrm.ctypes.data_as(C.POINTER(C.c_double)), C.byref(seg), C.c_double(wl.resolution),
                              exp.ctypes.data_as(C.POINTER(C.c_int32)))
    print(f"oracle: components {len(np.unique(exp))}; mode0 diff {(out[0] != exp).sum()}, "
          f"mode1 diff {(out[1] != exp).sum()}, slab diff {(labels != exp).sum()}")
    bad = np.nonzero(out[0] != exp)[0]
    if len(bad):
        print("first bad:", bad[:10].tolist(), "mode0", out[0][bad[:10]].tolist(), "oracle", exp[bad[:10]].tolist())


if __name__ == "__main__":
    main()
