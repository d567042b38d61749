"""Time the CCL variants (vp_set_ccl_mode 0/1/2) on the C2 stream and a C5
steppable list; every variant must give the same labels."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_01592_b200 import native, scenes  # noqa: E402


def main():
    wl = scenes.workload("c2")
    L = native.lib()
    for mode in (0, 1, 2):
        native.set_ccl_mode(mode)
        pl = native.Pipeline(wl.resolution, wl.extent, wl.frames[0].translation, native.default_params(seed=2025))
        L.vp_profile_enable(1)
        for f in wl.frames:
            pl.frame(f.points, f.rotation, f.translation, want_polygons=False)
        names = (C.c_char_p * 128)()
        ms = (C.c_double * 128)()
        calls = (C.c_uint64 * 128)()
        nk = L.vp_profile_read(names, ms, calls, 128)
        L.vp_profile_enable(0)
        prof = {names[i].decode(): ms[i] / 30 * 1e3 for i in range(nk) if b"ccl" in names[i]}
        print(f"C2 mode {mode}: ccl us/frame", {k: round(v, 1) for k, v in prof.items()},
              "total", round(sum(prof.values()), 1), flush=True)
        pl.close()
    # C5 steppable list (8 frames, one slab): label_components per mode
    from paper_2510_01592_b200 import slabs
    w5 = scenes.workload("c5", frames=8)
    params = native.default_params(seed=2025)
    native.set_ccl_mode(0)
    s = slabs.Slab(w5.resolution, w5.extent, scenes.C5_CENTER, 0, w5.extent[0])
    comm = slabs.LocalComm(1)
    for f in w5.frames:
        slabs.slab_frame([s], comm, torch.from_numpy(f.points).cuda(), f.rotation, f.translation, params)
    S, (idx, mean, nrm) = s.steppable(params.seg)
    idx = idx.cpu().numpy().view(np.int32).reshape(S, 3)
    mean = mean.cpu().numpy().view(np.float64).reshape(S, 3)
    nrm = nrm.cpu().numpy().view(np.float64).reshape(S, 3)
    ref = None
    for mode in (0, 1, 2):
        native.set_ccl_mode(mode)
        native.label_components(idx, mean, nrm, params.seg, 0.01)  # warm
        L.vp_profile_enable(1)
        lab = native.label_components(idx, mean, nrm, params.seg, 0.01)
        names = (C.c_char_p * 128)()
        ms = (C.c_double * 128)()
        calls = (C.c_uint64 * 128)()
        nk = L.vp_profile_read(names, ms, calls, 128)
        L.vp_profile_enable(0)
        prof = {names[i].decode(): ms[i] * 1e3 for i in range(nk) if b"ccl" in names[i]}
        ref = lab if ref is None else ref
        print(f"C5 S={S} mode {mode}: same={np.array_equal(lab, ref)} ccl us",
              {k: round(v, 1) for k, v in prof.items()}, "total", round(sum(prof.values()), 1), flush=True)
    native.set_ccl_mode(0)


if __name__ == "__main__":
    main()
