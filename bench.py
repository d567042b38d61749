"""Benchmark: segmentation update rate of the full per-frame update
(clear -> integrate -> recenter -> normals/classify -> CCL -> RANSAC -> refine
-> hull) on BASELINE.json configs[1] (C2: Stair5 + stepping stones, 30-frame
640x480 depth stream, 0.01 m voxels, 500^3 window), one B200 per rank.

A step = one pass over the 30-frame stream from an empty map (the map is reset
between steps, untimed, together with an L2 flush). `value` = frames/s with
every frame already resident in HBM (device time, CUDA events on the
library's stream, max over ranks); a step is one vp_pipeline_run call
(run_frames: consecutive frames overlap on the device, outputs identical to
the frame-by-frame API). `e2e` = the same call with pinned-host inputs (H2D
inside) and the final polygons read back.

--impl reference times the reference's own CPU implementation (oracle/_ref:
the unmodified /root/reference sources) on the host cores over a bounded
sample of the same stream.

N > 1 (default C5, BASELINE configs[4]): one 2000x2000x300 window split into
x-slabs across the ranks, each frame one vp_slab_frame call
per rank (csrc/slab_frame.cu: frame broadcast, halo planes, halo steppable
lists, boundary-label merge, cluster gather to the owning slab and the
polygon gather, all over the library's NCCL communicator; strong scaling).
--workload c2 with N > 1 runs independent replicas of the per-robot C2 stream
(weak scaling, no data-path collective: the fallback where slabbing does not
apply).

At N = 1 the line also carries secondary `configs` (C1, C3, C4 and C5 as one
slab) measured the same way.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "segmentation update rate (Hz, ms/frame) at 0.01 m; points/s integrated; HBM GB/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


C2_WORKLOAD = "C2: stair5+stepping stones, 30x640x480 depth frames, 0.01 m, 500^3"


def c2_config(nf, npoints, world):
    """`config` of the C2 line -- identical in both arms (same frames, same step)."""
    return {"workload": C2_WORKLOAD, "frames_per_step": nf, "points_per_step": int(npoints),
            "resolution_m": 0.01, "extent": [500, 500, 500], "seed": 2025,
            "step": "one pass over the 30-frame stream from an empty map",
            "l2": "B200 arm: 256 MiB write between steps (> 126 MB L2)",
            "parallelism": f"replicas x{world}" if world > 1 else "single"}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) > 8 for i in range(4)
                          if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# --------------------------------------------------------------- workload
def load_workload(name):
    from paper_2510_01592_b200 import scenes
    t = time.time()
    wl = scenes.workload(name)
    log(f"[bench] workload {name}: {len(wl.frames)} frames, {wl.points} points, "
        f"rendered in {time.time() - t:.1f}s")
    return wl


def algorithmic_bytes(c, n_points):
    """SURVEY.md §8(d) unique-touch byte model, per kernel, from one frame's counters.
    c = vp_pipeline_counters: cleared freed touched discarded dropped occupied V S K
    fits padded inliers poolv newly groups overflow."""
    cleared, freed, touched, _, dropped, _, V, S, K, F, padded, inl, poolv = c[:13]
    return {
        "k_clear_walk": 12 * n_points + cleared / 8,           # points in, clear marks out
        "k_clear_apply": 2 * C_BITS + 32 * freed,              # clr (+occ) scan, freed cells
        "k_integrate_hash": 12 * n_points + 8 * n_points,
        "k_integrate_fold": 64 * touched + 12 * n_points,      # cell RMW + points
        "k_recenter": 3 * C_BITS + 32 * dropped,
        "k_bitmap_count": C_BITS,
        "k_bitmap_emit": C_BITS + 4 * V,
        "k_normals": 32 * V + 4 * V + 72 * V,                  # cells, list in, estimate out
        "k_ccl_hook": 56 * S,
        "k_ccl_compress": 8 * S,
        "k_ccl_union": 56 * S,                                 # mean+normal+ordinal per voxel
        "k_ccl_flatten": 12 * S,
        "k_ransac_count": 24 * padded,
        "k_extract_count": 24 * padded,
        "k_extract_emit": 24 * padded + 24 * inl,
        "k_refine": 2 * 24 * inl,
        "k_poly_extremes": 24 * inl + 16 * inl,
        "k_poly_keep": 16 * inl,
        "k_poly_hull": 64 * poolv,
    }


C_BITS = 0  # set from the grid size (cells / 8)


def hbm_peak(peaks):
    """HBM copy bandwidth (GB/s) from the driver-written MEASURED_PEAKS.json:
    the burst figure (the top kernel is timed alone, one launch at a time in
    the event profile), else any HBM figure, else the B200_PROFILING fallback."""
    flat = {}

    def walk(d, pre=""):
        for k, v in d.items():
            if isinstance(v, dict):
                walk(v, pre + k + ".")
            elif isinstance(v, (int, float)) and not isinstance(v, bool):
                flat[(pre + k).lower()] = float(v)
    if isinstance(peaks, dict):
        walk(peaks)
    hbm = {k: v for k, v in flat.items() if ("hbm" in k or "dram" in k or "copy" in k) and v > 100}
    for pick in ("burst", ""):
        for k, v in sorted(hbm.items()):
            if pick in k:
                return v, f"MEASURED_PEAKS.json {k}"
    return 6650.0, "fallback 6650 (B200_PROFILING.md)"


# ------------------------------------------------------------------- ours
def run_ours(args, rank, world, dist):
    import numpy as np
    import torch

    from paper_2510_01592_b200 import native

    global C_BITS
    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    wl = load_workload(args.workload)
    nx, ny, nz = wl.extent
    C_BITS = nx * ny * nz // 8
    frames = wl.frames
    nf = len(frames)
    npts = [len(f.points) for f in frames]
    params = native.default_params(seed=wl.seed)
    pl = native.Pipeline(wl.resolution, wl.extent, frames[0].translation, params, device=dev)
    L = native.lib()
    L.vp_pipeline_stream.restype = C.c_void_p
    stream = torch.cuda.ExternalStream(L.vp_pipeline_stream(pl.h))
    start = np.ascontiguousarray(frames[0].translation, np.float64)

    def reset():
        native.check(L.vp_pipeline_reset(pl.h, start.ctypes.data_as(C.POINTER(C.c_double))))

    dev_pts = [torch.from_numpy(f.points).to(f"cuda:{dev}").contiguous() for f in frames]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")
    torch.cuda.synchronize()

    # the whole 30-frame stream is one vp_pipeline_run call (run_frames):
    # consecutive frames overlap on the device; per-frame outputs are identical
    # to the frame-by-frame API (tests/test_gpu_parity.py)
    nfr = len(frames)
    R_all = np.ascontiguousarray(np.stack([f.rotation.reshape(9) for f in frames]), np.float64)
    t_all = np.ascontiguousarray(np.stack([f.translation for f in frames]), np.float64)
    n_all = np.asarray(npts, np.uint64)
    dev_ptrs = (C.c_void_p * nfr)(*[d.data_ptr() for d in dev_pts])
    host_pts = [torch.from_numpy(f.points).pin_memory() for f in frames]
    host_ptrs = (C.c_void_p * nfr)(*[h.data_ptr() for h in host_pts])

    def device_step():
        pl.run_ptrs(dev_ptrs, n_all, R_all, t_all, device_ptrs=True, want_polygons=False)

    # clocks are sampled from the start of the warm-up to the end of the timed
    # loops (the timed region alone is ~0.1 s, a handful of samples)
    clk = ClockSampler(dev).__enter__()
    # warm-up
    for _ in range(args.warmup):
        reset()
        device_step()
    torch.cuda.synchronize()

    # timed: device-resident inputs
    launches0 = native.kernel_launch_count()
    times = []
    if True:
        for _ in range(args.steps):
            reset()
            flush.fill_(1.0)  # > L2: evict the previous step's working set
            torch.cuda.synchronize()
            if dist:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            device_step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    launches = native.kernel_launch_count() - launches0
    counters = np.zeros(16, np.uint64)
    L.vp_pipeline_counters(pl.h, counters.ctypes.data_as(C.POINTER(C.c_uint64)))
    step_ms = sum(times) / len(times)
    if dist:
        t = torch.tensor([sum(times)], device=f"cuda:{dev}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    else:
        total_ms = sum(times)
    value = world * nf * args.steps / (total_ms / 1e3)

    # e2e through the public C ABI (vp_pipeline_run_frames): pinned host
    # points (H2D inside the call), every frame's polygons handed to the host
    # (run_frames' per-frame polygons; packed on the device into mapped host
    # memory) plus the final frame's (PipelineResult::polygons)
    e2e_times = []
    d2h_bytes = 0
    ex = native.RunOutputs()
    pf = (C.POINTER(native.Polygons) * nfr)()
    ex.per_frame = C.cast(pf, C.POINTER(C.POINTER(native.Polygons)))
    for s in range(max(1, args.steps)):
        reset()
        flush.fill_(1.0)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        # the C ABI call returns with every frame's polygons in host memory;
        # the Python dict conversion after e1 is wrapper work
        raw = C.POINTER(native.Polygons)()
        native.check(L.vp_pipeline_run_frames(pl.h, C.c_size_t(nfr), host_ptrs, n_all.ctypes.data_as(
            C.POINTER(C.c_uint64)), R_all.ctypes.data_as(C.POINTER(C.c_double)),
            t_all.ctypes.data_as(C.POINTER(C.c_double)), C.c_int(0), C.byref(raw), C.byref(ex)))
        e1.record(stream)
        e1.synchronize()
        native.polygons_to_py(raw)
        per = [native.polygons_to_py(pf[k]) for k in range(nfr)]
        e2e_times.append(e0.elapsed_time(e1) / 1e3)
        d2h_bytes = sum(8 * (4 + 12 * len(ps) + 5 * sum(len(p["v3d"]) for p in ps)) for ps in per)
    e2e_total = sum(e2e_times)
    if dist:
        t = torch.tensor([e2e_total], device=f"cuda:{dev}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = world * nf * len(e2e_times) / e2e_total
    # per-frame latency (SURVEY §8(d) unit of work): one frame in flight, as a
    # robot streaming at sensor rate sees it -- vp_pipeline_frame from pinned
    # host points (H2D start) to the frame's polygons in host memory, CUDA
    # events on the library stream; median of frames 2..F of a pass from an
    # empty map
    lat, lat_py = [], []
    L.vp_pipeline_latency_ms.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
    lat_ms = C.c_double()
    for rep in range(2):
        reset()
        torch.cuda.synchronize()
        for k, f in enumerate(frames):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            polys, _ = pl.frame_ptr(host_pts[k].data_ptr(), npts[k], f.rotation, f.translation, want_polygons=True,
                                    want_timing=False)
            e1.record(stream)
            e1.synchronize()
            if rep == 1 and k >= 2:
                native.check(L.vp_pipeline_latency_ms(pl.h, C.byref(lat_ms)))
                lat.append(lat_ms.value)           # library events: H2D start -> polygons in host memory
                lat_py.append(e0.elapsed_time(e1))  # the same seen from Python (plus ctypes + numpy conversion)
    clk.__exit__(None, None, None)

    # per-kernel profile of one step (serialised launches; shares only)
    L.vp_profile_read.restype = C.c_int
    reset()
    L.vp_profile_enable(1)
    per_frame_counters = []
    for f, d in zip(frames, dev_pts):
        pl.frame_device(d.data_ptr(), len(f.points), f.rotation, f.translation)
        cc = np.zeros(16, np.uint64)
        L.vp_pipeline_counters(pl.h, cc.ctypes.data_as(C.POINTER(C.c_uint64)))
        per_frame_counters.append(cc.astype(np.float64))
    names = (C.c_char_p * 128)()
    ms = (C.c_double * 128)()
    calls = (C.c_uint64 * 128)()
    nk = L.vp_profile_read(names, ms, calls, 128)
    L.vp_profile_enable(0)
    prof = {names[i].decode(): (ms[i], calls[i]) for i in range(nk)}
    prof_total = sum(v[0] for v in prof.values())
    top = max(prof, key=lambda k: prof[k][0])
    # algorithmic bytes of the top kernel, summed over the step's frames
    alg = sum(algorithmic_bytes(c, n).get(top, 0.0) for c, n in zip(per_frame_counters, npts))
    top_ms, top_calls = prof[top]
    per_launch_bytes = alg / top_calls
    per_launch_s = top_ms / top_calls / 1e3
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak, peak_source = hbm_peak(peaks)
    achieved = per_launch_bytes / per_launch_s / 1e9
    traffic, limiter, winst, atomics = None, None, None, None
    try:  # DRAM bytes, pipe utilisation, instructions, atomics of the same kernel (committed ncu --set full)
        nt = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = nt["dram_bytes_per_launch"].get(top)
        limiter = nt.get("utilisation_pct", {}).get(top)
        winst = nt.get("warp_inst_per_launch", {}).get(top)
        atomics = nt.get("atomics_per_launch", {}).get(top)
    except Exception:
        pass
    # issue roofline of the same kernel: its warp instructions per launch
    # (ncu) / the live launch duration, against 148 SMs x 4 schedulers x 1
    # warp instruction per cycle at the sampled SM clock
    sm_hz = (clk.summary().get("sm_mhz") or 1965.0) * 1e6
    issue = None
    if winst:
        peak_i = 148 * 4 * sm_hz
        issue = {"warp_inst_per_launch": winst, "achieved_ginst_s": round(winst / per_launch_s / 1e9, 1),
                 "peak_ginst_s": round(peak_i / 1e9, 1), "frac": round(winst / per_launch_s / peak_i, 4)}
    # DDA cell steps of the step's frames, estimated as the L1 cell distance
    # sensor -> end point (k_dda_keys' length model; the window clip ignored)
    dda_steps = 0.0
    for f in frames:
        w = f.points.astype(np.float64) @ np.asarray(f.rotation, np.float64).reshape(3, 3).T
        dda_steps += float(np.nansum(np.abs(w) / wl.resolution))
    # whole-step algorithmic bytes (the survey's frame formula)
    step_bytes = 0.0
    for c, n in zip(per_frame_counters, npts):
        cleared, freed, touched, _, dropped, _, V, S, K, F, padded, inl, poolv = c[:13]
        step_bytes += (12 * n + 64 * touched + 32 * freed + C_BITS + 72 * V + 56 * S + 24 * padded
                       + 48 * inl + 64 * poolv)
    out = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "Hz",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4),
        "ms_per_frame": round(step_ms / nf, 4),
        "points_per_s": round(world * sum(npts) * args.steps / (total_ms / 1e3), 1),
        "hbm_gbs_step": round(step_bytes / (step_ms / 1e3) / 1e9, 2),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (library frame source = reference render_frame, byte-identical)",
        "config": c2_config(nf, sum(npts), world),
        "gpu_launches": int(launches),
        "latency_ms_p50": round(statistics.median(lat), 4),
        "latency_ms_p90": round(sorted(lat)[int(0.9 * (len(lat) - 1))], 4),
        "latency_ms_p50_python": round(statistics.median(lat_py), 4),
        "latency": "one frame in flight (vp_pipeline_frame): pinned host points -> polygons on the host, "
                   "library CUDA events (vp_pipeline_latency_ms: before the points H2D -> polygons assembled in "
                   "host memory), frames 2..29 of a pass from an empty map; latency_ms_p50_python adds the "
                   "ctypes call and numpy conversion",
        "e2e": {"value": round(e2e_value, 3), "unit": "Hz",
                "h2d_bytes_per_step": int(12 * sum(npts)), "d2h_bytes_per_step": int(d2h_bytes)},
        "roofline": {"bound": "hbm", "kernel": top, "achieved": round(achieved, 2), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 5), "traffic": traffic,
                     "alg_bytes_per_launch": round(per_launch_bytes), "us_per_launch": round(per_launch_s * 1e6, 2),
                     "share_of_step": round(top_ms / prof_total, 4), "peak_source": peak_source,
                     "utilisation_pct_ncu": limiter, "issue": issue, "atomics_ncu": atomics,
                     # secondary rate of the DDA: cell steps per second
                     "dda_steps_per_launch_est": round(dda_steps / len(frames)) if top == "k_clear_walk" else None,
                     "dda_gsteps_per_s": (round(dda_steps / len(frames) / per_launch_s / 1e9, 1)
                                          if top == "k_clear_walk" else None)},
        "kernels": {k: {"ms_per_step": round(v[0], 4), "calls": int(v[1])}
                    for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args.cpu_frames)
    if rank == 0 and world == 1 and not args.no_configs:
        # the other BASELINE configs on this GPU (secondary lines; C1 is the
        # reference's 0.05 m CPU case, C5 the multi-GPU map as one slab)
        out["configs"] = {}
        for name in ("c1", "c3", "c4"):
            try:
                out["configs"][name] = measure_stream(name, 5, 3, dev, not args.no_cpu_baseline)
            except Exception as e:  # report, do not lose the headline line
                out["configs"][name] = {"error": repr(e)[:200]}
        try:
            a5 = argparse.Namespace(**vars(args))
            a5.steps, a5.warmup = 6, 3
            r5 = run_slabs(a5, 0, 1, None)
            out["configs"]["c5"] = {k: r5[k] for k in ("value", "ms_per_frame", "points_per_s", "e2e", "config")}
        except Exception as e:
            out["configs"]["c5"] = {"error": repr(e)[:200]}
    return out


# ------------------------------------------- other BASELINE configs (N=1)
def measure_stream(name, steps, warmup, dev, with_cpu=True):
    """Frames/s and points/s of one BASELINE config on one GPU: the stream from
    an empty map per step (device-resident inputs; L2 flushed between steps),
    plus the same through the C ABI with pinned host inputs (e2e), and
    oracle/_ref on the host cores over a bounded prefix of the same frames."""
    import numpy as np
    import torch

    from paper_2510_01592_b200 import native
    wl = load_workload(name)
    frames = wl.frames
    nf = len(frames)
    npts = [len(f.points) for f in frames]
    pl = native.Pipeline(wl.resolution, wl.extent, frames[0].translation, native.default_params(seed=wl.seed),
                         device=dev)
    L = native.lib()
    L.vp_pipeline_stream.restype = C.c_void_p
    stream = torch.cuda.ExternalStream(L.vp_pipeline_stream(pl.h))
    start = np.ascontiguousarray(frames[0].translation, np.float64)
    R_all = np.ascontiguousarray(np.stack([f.rotation.reshape(9) for f in frames]), np.float64)
    t_all = np.ascontiguousarray(np.stack([f.translation for f in frames]), np.float64)
    n_all = np.asarray(npts, np.uint64)
    dev_pts = [torch.from_numpy(f.points).to(f"cuda:{dev}").contiguous() for f in frames]
    host_pts = [torch.from_numpy(f.points).pin_memory() for f in frames]
    dev_ptrs = (C.c_void_p * nf)(*[d.data_ptr() for d in dev_pts])
    host_ptrs = (C.c_void_p * nf)(*[h.data_ptr() for h in host_pts])
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")

    def timed(ptrs, device_ptrs, k):
        out = []
        for _ in range(k):
            native.check(L.vp_pipeline_reset(pl.h, start.ctypes.data_as(C.POINTER(C.c_double))))
            flush.fill_(1.0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pl.run_ptrs(ptrs, n_all, R_all, t_all, device_ptrs=device_ptrs, want_polygons=not device_ptrs)
            e1.record(stream)
            e1.synchronize()
            out.append(e0.elapsed_time(e1))
        return out

    timed(dev_ptrs, True, warmup)
    t = timed(dev_ptrs, True, steps)
    te = timed(host_ptrs, False, steps)
    pl.close()
    ms = sum(t) / len(t)
    r = {"workload": name, "frames_per_step": nf, "points_per_frame": round(sum(npts) / nf),
         "resolution_m": wl.resolution, "extent": list(wl.extent), "value_hz": round(nf / (ms / 1e3), 2),
         "ms_per_frame": round(ms / nf, 4), "points_per_s": round(sum(npts) / (ms / 1e3), 1),
         "e2e_hz": round(nf / (sum(te) / len(te) / 1e3), 2), "steps": steps, "warmup": warmup}
    if with_cpu:
        try:
            r["cpu_baseline"] = cpu_baseline_stream(wl)
        except Exception as e:  # the reference library is optional on the box
            r["cpu_baseline"] = {"error": repr(e)[:200]}
    return r


def cpu_baseline_stream(wl, budget_s=8.0):
    """oracle/_ref on the host cores (all threads) over the first frames of a
    secondary config's stream from an empty map, stopping once `budget_s` of
    reference time is spent (the same frames the B200 line runs)."""
    import numpy as np

    from paper_2510_01592_b200.native import default_params  # a ctypes struct: loads no library
    L, kind = ref_lib()
    cores = os.cpu_count()
    L.ref_set_threads(cores)
    p = default_params(seed=wl.seed)
    ext = np.asarray(wl.extent, np.int32)
    c = np.ascontiguousarray(wl.frames[0].translation, np.float64)
    s = L.ref_session_create(C.c_double(wl.resolution), ext.ctypes.data_as(C.POINTER(C.c_int32)),
                             c.ctypes.data_as(C.POINTER(C.c_double)), C.byref(p))
    total, n = 0.0, 0
    for f in wl.frames:
        total += _ref_step(L, s, f)
        n += 1
        if total / 1e3 >= budget_s:
            break
    L.ref_session_destroy(C.c_void_p(s))
    return {"value": round(n / (total / 1e3), 4), "unit": "Hz", "cores": cores, "kind": kind,
            "sample": f"first {n} of {len(wl.frames)} frames from an empty map ({total / 1e3:.1f} s)"}


# ------------------------------------------------------ C5: spatial slabs
def run_slabs(args, rank, world, dist):
    """C5 (BASELINE configs[4]): one 2000x2000x300 window at 0.01 m split into
    x-slabs, one per rank; every frame is broadcast from rank 0
    over NCCL, halo planes are exchanged with the neighbours, the steppable
    lists are gathered on rank 0, which segments. A step = one frame update of
    the whole map (strong scaling: the same map and frames for every N)."""
    import numpy as np
    import torch

    from paper_2510_01592_b200 import native, scenes, slabs

    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    W, K = args.warmup, args.steps
    nf = W + K                          # warm-up (map pre-population) + timed frames
    poses = scenes.c5_poses(nf)
    frames = None
    if rank == 0:
        t0 = time.time()
        frames = scenes.c5_workload(nf).frames
        log(f"[bench] c5: {nf} frames, {sum(len(f.points) for f in frames)} points, "
            f"rendered in {time.time() - t0:.1f}s")
    ext = scenes.C5_EXTENT
    lo, hi = slabs.split_x(ext[0], world)[rank]
    slab = slabs.Slab(0.01, ext, scenes.C5_CENTER, lo, hi, device=dev)
    # the timed frames run the library-orchestrated vp_slab_frame over the
    # library's NCCL communicator; the profiled frame below uses the Python
    # model of the same protocol (its phase counters feed the roofline)
    comm = slabs.DistComm(dist, dev) if dist else slabs.LocalComm(1)
    ncomm = slabs.nccl_comm(dist, dev) if dist else None
    params = native.default_params(seed=2025)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")
    empty = torch.empty(0, dtype=torch.float32, device=f"cuda:{dev}")
    dev_pts = [torch.from_numpy(f.points).to(f"cuda:{dev}") for f in frames] if rank == 0 else None
    host_pts = [torch.from_numpy(f.points).pin_memory() for f in frames] if rank == 0 else None
    npts = [len(f.points) for f in frames] if rank == 0 else [0] * nf
    if dist:  # every rank passes n to vp_slab_frame
        nt = torch.tensor(npts, dtype=torch.int64, device=f"cuda:{dev}")
        dist.broadcast(nt, 0)
        npts = [int(v) for v in nt.cpu().tolist()]

    def rot(i):
        return poses[i][:9].reshape(3, 3), poses[i][9:12]

    def step(i, pts):
        R, t = rot(i)
        if ncomm is None:
            return slabs.frame_local([slab], pts, R, t, params)
        return slabs.frame(slab, ncomm, pts if rank == 0 else None, npts[i], R, t, params)

    for i in range(W):
        step(i, dev_pts[i] if rank == 0 else empty)
    torch.cuda.synchronize()

    def timed(first, inputs):
        times, polys = [], None
        for i in range(first, first + K):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            if dist:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            polys = step(i, inputs(i))
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        total = sum(times)
        if dist:
            tt = torch.tensor([total], device=f"cuda:{dev}", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            total = float(tt.item())
        return total, polys

    launches0 = native.kernel_launch_count()
    with ClockSampler(dev) as clk:
        total_ms, _ = timed(W, lambda i: dev_pts[i] if rank == 0 else empty)
    launches = native.kernel_launch_count() - launches0
    # e2e: the same frames again (the robot revisits), pinned host points ->
    # H2D on rank 0 inside the region -> broadcast -> ... -> polygons on host
    e2e_ms, polys = timed(W, lambda i: host_pts[i].to(f"cuda:{dev}", non_blocking=True)
                          if rank == 0 else empty)

    # one profiled frame (serialised launches): kernel shares + counters
    L = native.lib()
    L.vp_profile_read.restype = C.c_int
    L.vp_profile_enable(1)
    i = W + K - 1
    R, t = rot(i)
    stages = {}
    slabs.slab_frame([slab], comm, dev_pts[i] if rank == 0 else empty, R, t, params, stages=stages)
    c_map = stages["c_map"].astype(np.float64)
    c_step = stages["c_step"].astype(np.float64)
    c_seg = stages["c_seg"].astype(np.float64)
    names = (C.c_char_p * 128)()
    ms = (C.c_double * 128)()
    calls = (C.c_uint64 * 128)()
    nk = L.vp_profile_read(names, ms, calls, 128)
    L.vp_profile_enable(0)
    prof = {names[j].decode(): (ms[j], calls[j]) for j in range(nk)}
    if ncomm is not None:
        slabs.nccl_comm_destroy(ncomm)
    if rank != 0:
        slab.close()
        return None
    n = float(len(frames[i].points))
    cleared, freed, touched = c_map[0], c_map[1], c_map[2]
    V, S_ = c_step[6], c_step[7]
    padded, inl, poolv = c_seg[10], c_seg[11], c_seg[12]
    own_bits = (hi - lo) * ext[1] * ext[2] / 8
    alg = {"k_clear_walk": 12 * n + cleared / 8, "k_clear_apply": 2 * own_bits + 32 * freed,
           "k_integrate_fold": 64 * touched + 12 * n, "k_integrate_hash": 20 * n,
           "k_bitmap_count": own_bits, "k_bitmap_emit": own_bits + 4 * V, "k_normals": 108 * V,
           "k_ccl_hook": 56 * S_, "k_ccl_union": 56 * S_, "k_ccl_compress": 8 * S_, "k_ccl_flatten": 12 * S_,
           "k_map_fill": 16 * S_, "k_ransac_count": 24 * padded, "k_extract_count": 24 * padded,
           "k_refine": 48 * inl, "k_poly_hull": 64 * poolv}
    prof_total = sum(v[0] for v in prof.values())
    top = max((k for k in prof if k in alg), key=lambda k: prof[k][0])
    top_ms, top_calls = prof[top]
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak, peak_source = hbm_peak(peaks)
    achieved = alg[top] / top_calls / (top_ms / top_calls / 1e3) / 1e9
    frame_bytes = 12 * n + 64 * touched + 32 * freed + own_bits + 72 * V + 56 * S_ + 24 * padded + 48 * inl + 64 * poolv
    timed_pts = sum(npts[W:W + K])
    slab.close()
    return {
        "metric": METRIC,
        "value": round(K / (total_ms / 1e3), 3),
        "unit": "Hz",
        "n_gpus": world,
        "steps": K,
        "warmup": W,
        "ms_per_step": round(total_ms / K, 4),
        "ms_per_frame": round(total_ms / K, 4),
        "points_per_s": round(timed_pts / (total_ms / 1e3), 1),
        "hbm_gbs_rank0_frame": round(frame_bytes / (total_ms / K / 1e3) / 1e9, 2),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (library frame source = reference render_frame, sphere LiDAR 1M rays)",
        "config": {"workload": "C5: 20x20x3 m two-level map (floor, mezzanine, 2 stairs, 10 tables), "
                               "2000x2000x300 at 0.01 m, lawnmower sphere-LiDAR frames",
                   "slabs": [list(r) for r in slabs.split_x(ext[0], world)], "timed_frames": f"{W}..{W + K - 1}",
                   "e2e_frames": f"{W}..{W + K - 1} again (revisit)", "points_per_frame": round(timed_pts / K),
                   "l2": "flushed (256 MiB write) between steps; window 38.4 GB >> L2",
                   "parallelism": f"x-slabs x{world}: one vp_slab_frame per rank and frame (halo planes, "
                                  "halo steppable lists, boundary-label merge, cluster gather to the owner, "
                                  "polygon gather; library NCCL communicator)"
                   if world > 1 else "single slab (vp_slab_frame_local)"},
        "gpu_launches": int(launches),
        "e2e": {"value": round(K / (e2e_ms / 1e3), 3), "unit": "Hz",
                "h2d_bytes_per_step": int(12 * timed_pts / K),
                "d2h_bytes_per_step": int(sum(40 + 8 + 40 * len(p["v3d"]) for p in polys or []))},
        "roofline": {"bound": "hbm", "kernel": top, "rank": 0, "achieved": round(achieved, 2), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 5), "traffic": None,
                     "alg_bytes_per_launch": round(alg[top] / top_calls),
                     "us_per_launch": round(top_ms / top_calls * 1e3, 2),
                     "share_of_step": round(top_ms / prof_total, 4),
                     "peak_source": peak_source},
        "kernels_rank0": {k: {"ms_per_frame": round(v[0], 4), "calls": int(v[1])}
                          for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])},
        "clocks": clk.summary(),
        "cpu_baseline": {"value": None, "unit": "Hz", "cores": os.cpu_count(), "kind": "reference",
                         "sample": "not run for C5 (38.4 GB window; the C2 line carries the CPU baseline)"},
    }


# ------------------------------------------------------- reference (CPU)
def ref_lib():
    path = os.path.join(ROOT, "oracle", "_ref", "libvoxplane_ref.so")
    kind = "reference"
    if not os.path.exists(path):
        raise FileNotFoundError(path)
    L = C.CDLL(path)
    L.ref_session_create.restype = C.c_void_p
    dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int)
    L.ref_stock_scene.argtypes = [C.c_int, dp, ip, dp, ip]
    L.ref_default_trajectory.argtypes = [C.c_int, C.c_int, C.c_double, dp]
    L.ref_render.argtypes = [dp, C.c_int, dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                             C.POINTER(C.c_float), C.c_int, C.c_double, C.c_double, C.c_double, dp, C.c_int,
                             C.c_uint64, C.c_char_p]
    return L, kind


def ref_workload_c2(L):
    """The C2 stream built and rendered by the reference itself (oracle/_ref:
    build_scene Stair5 + the six stepping-stone boxes, default_trajectory,
    render_frame, write_frames_binary), read back as VXPF -- the reference arm
    never loads this repository's library. Byte-identical to the B200 arm's
    frames (tests/test_oracle.py::test_reference_arm_frames_match)."""
    import tempfile

    import numpy as np

    from paper_2510_01592_b200.frames import read_frames
    from paper_2510_01592_b200.scenes import stepping_stone_boxes
    dp = C.POINTER(C.c_double)
    boxes, rects = np.zeros(6 * 64), np.zeros(14 * 64)
    nb, nr = C.c_int(), C.c_int()
    L.ref_stock_scene(0, boxes.ctypes.data_as(dp), C.byref(nb), rects.ctypes.data_as(dp), C.byref(nr))
    for i, (lo, hi) in enumerate(stepping_stone_boxes()):
        boxes[6 * (nb.value + i):6 * (nb.value + i + 1)] = (*lo, *hi)
    nbox = nb.value + len(stepping_stone_boxes())
    poses = np.zeros((32, 12))
    nf = L.ref_default_trajectory(0, 30, 30.0, poses.ctypes.data_as(dp))
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "c2.vxpf")
        rc = L.ref_render(boxes.ctypes.data_as(dp), nbox, rects.ctypes.data_as(dp), nr.value, 0, 640, 480,
                          87.0, 58.0, None, 0, 30.0, 6.0, 0.003, poses.ctypes.data_as(dp), nf, 2025,
                          path.encode())
        if rc != 0:
            raise RuntimeError("ref_render failed")
        return read_frames(path)


def _ref_step(L, s, f):
    import numpy as np
    ms = C.c_double()
    npoly = C.c_uint64()
    pts = np.ascontiguousarray(f.points)
    R = np.ascontiguousarray(f.rotation, np.float64).reshape(9)
    t = np.ascontiguousarray(f.translation, np.float64)
    rc = L.ref_session_step(C.c_void_p(s), pts.ctypes.data_as(C.POINTER(C.c_float)), C.c_uint64(len(pts)),
                            R.ctypes.data_as(C.POINTER(C.c_double)), t.ctypes.data_as(C.POINTER(C.c_double)),
                            C.byref(ms), C.byref(npoly))
    if rc != 0:
        raise RuntimeError("ref_session_step failed")
    return ms.value


def _ref_session(L, frames):
    import numpy as np

    from paper_2510_01592_b200.native import default_params  # a ctypes struct: loads no library
    p = default_params(seed=2025)
    ext = np.asarray((500, 500, 500), np.int32)
    c = np.ascontiguousarray(frames[0].translation, np.float64)
    return L.ref_session_create(C.c_double(0.01), ext.ctypes.data_as(C.POINTER(C.c_int32)),
                                c.ctypes.data_as(C.POINTER(C.c_double)), C.byref(p)), p


def cpu_baseline(nframes):
    """oracle/_ref (unmodified reference sources) on the host cores: the first
    `nframes` frames of the C2 stream from an empty map, all host threads."""
    L, kind = ref_lib()
    cores = os.cpu_count()
    L.ref_set_threads(cores)
    frames = ref_workload_c2(L)
    s, _ = _ref_session(L, frames)
    total = sum(_ref_step(L, s, f) for f in frames[:nframes])
    L.ref_session_destroy(C.c_void_p(s))
    return {"value": round(nframes / (total / 1e3), 4), "unit": "Hz", "cores": cores, "kind": kind,
            "cpu_model": cpu_model(),
            "sample": f"first {nframes} frames of the C2 stream from an empty 500^3 map "
                      f"({total / 1e3:.1f} s, run_frames body, VOXPLANE threads={cores})"}


def run_reference(args):
    """The reference's CPU implementation (oracle/_ref) on the same workload,
    config and step as the B200 arm: one pass over the 30-frame C2 stream
    from an empty map, split into `steps` consecutive groups of frames (one
    step = one group; more steps than frames: one frame per step, the map
    emptied at each wrap). Warm-up: `warmup` frames on a separate session."""
    L, kind = ref_lib()
    cores = os.cpu_count()
    L.ref_set_threads(cores)
    t0 = time.time()
    frames = ref_workload_c2(L)
    nf = len(frames)
    npts = sum(len(f.points) for f in frames)
    log(f"[bench] reference arm: C2 rendered by oracle/_ref in {time.time() - t0:.1f}s ({nf} frames)")
    w, _ = _ref_session(L, frames)
    for i in range(args.warmup):
        _ref_step(L, w, frames[i % nf])
    L.ref_session_destroy(C.c_void_p(w))
    K = max(1, args.steps)
    if K <= nf:
        bounds = [round(j * nf / K) for j in range(K + 1)]
        groups = [list(range(bounds[j], bounds[j + 1])) for j in range(K)]
    else:
        groups = [[j % nf] for j in range(K)]
    s, _ = _ref_session(L, frames)
    times, done = [], 0
    for g in groups:
        ms = 0.0
        for i in g:
            if i == 0 and done:  # next pass: a fresh (empty) map, untimed
                L.ref_session_destroy(C.c_void_p(s))
                s, _ = _ref_session(L, frames)
            ms += _ref_step(L, s, frames[i])
            done += 1
        times.append(ms)
    L.ref_session_destroy(C.c_void_p(s))
    total = sum(times) / 1e3
    value = done / total
    world = int(os.environ.get("WORLD_SIZE", "1"))
    sample = (f"frames 0..{nf - 1} of C2 from an empty 500^3 map (one pass) in {K} steps"
              if K <= nf else f"{K} frames of C2 (passes from an empty map), one per step")
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "Hz", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * total / K, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (same frames as the B200 arm, rendered by the reference)",
        "config": c2_config(nf, npts, world),
        "cpu_baseline": {"value": round(value, 4), "unit": "Hz", "cores": cores, "kind": kind,
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "Hz", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def run_reference_c5(args):
    """The reference's CPU implementation (oracle/_ref) on C5, the workload of
    the N > 1 line: the reference renders the C5 frames itself (ref_render:
    the same scene, sphere-LiDAR pattern, lawnmower poses and seed), runs a
    fixed 2000 x 2000 x 300 window (38.4 GB of cells in host RAM) with all
    host threads, one warm-up frame (map pre-population), then times up to two
    frames (a C5 frame takes tens of seconds on the host)."""
    import tempfile

    import numpy as np

    from paper_2510_01592_b200.frames import read_frames
    from paper_2510_01592_b200.native import default_params  # a ctypes struct: loads no library
    from paper_2510_01592_b200.scenes import C5_CENTER, C5_EXTENT, c5_poses, c5_scene, spherical_pattern
    L, kind = ref_lib()
    cores = os.cpu_count()
    L.ref_set_threads(cores)
    W, K = min(max(args.warmup, 0), 1), min(max(args.steps, 1), 2)
    nf = W + K
    sc = c5_scene()
    boxes = np.asarray([(*lo, *hi) for lo, hi in sc.boxes], np.float64).reshape(-1)
    rects = np.asarray([(*np.asarray(R, np.float64).reshape(9), *t, hu, hv) for R, t, hu, hv in sc.rects],
                       np.float64).reshape(-1)
    pat = np.ascontiguousarray(spherical_pattern(1_000_000), np.float32)
    poses = np.ascontiguousarray(c5_poses(nf), np.float64)
    dp = C.POINTER(C.c_double)
    t0 = time.time()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "c5.vxpf")
        rc = L.ref_render(boxes.ctypes.data_as(dp), len(sc.boxes), rects.ctypes.data_as(dp), len(sc.rects), 1, 0, 0,
                          0.0, 0.0, pat.ctypes.data_as(C.POINTER(C.c_float)), len(pat), 10.0, 10.0, 0.003,
                          poses.ctypes.data_as(dp), nf, 2025, path.encode())
        if rc != 0:
            raise RuntimeError("ref_render failed")
        frames = read_frames(path)
    log(f"[bench] reference arm: C5 rendered by oracle/_ref in {time.time() - t0:.1f}s ({nf} frames)")
    p = default_params(seed=2025)
    ext = np.asarray(C5_EXTENT, np.int32)
    c = np.asarray(C5_CENTER, np.float64)
    L.ref_session_create.restype = C.c_void_p
    sess = L.ref_session_create(C.c_double(0.01), ext.ctypes.data_as(C.POINTER(C.c_int32)),
                                c.ctypes.data_as(dp), C.byref(p))
    L.ref_session_set_fixed(C.c_void_p(sess), C.c_int(1))
    for i in range(W):
        _ref_step(L, sess, frames[i])
    times = [_ref_step(L, sess, frames[W + i]) for i in range(K)]
    L.ref_session_destroy(C.c_void_p(sess))
    total = sum(times) / 1e3
    value = K / total
    world = int(os.environ.get("WORLD_SIZE", "1"))
    npts = sum(len(f.points) for f in frames[W:])
    sample = f"{W} warm-up + {K} timed C5 frames (fixed 2000x2000x300 window), one frame per step"
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": "Hz", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(1e3 * total / K, 3), "ms_per_frame": round(1e3 * total / K, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (same scene, pattern, poses and seed as the B200 arm, rendered by the reference)",
        "config": {"workload": "C5: 20x20x3 m two-level map (floor, mezzanine, 2 stairs, 10 tables), "
                               "2000x2000x300 at 0.01 m, lawnmower sphere-LiDAR frames",
                   "points_per_frame": round(npts / K), "parallelism": "host threads"},
        "cpu_baseline": {"value": round(value, 5), "unit": "Hz", "cores": cores, "kind": kind,
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": round(value, 5), "unit": "Hz", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, help="c2 (default at N = 1) or c5 (default at N > 1)")
    ap.add_argument("--cpu-frames", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the secondary C1/C3/C4/C5 lines")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.workload is None:
        args.workload = "c5" if world > 1 else "c2"
    if args.impl == "reference":
        if rank != 0:
            return 0
        try:
            out = run_reference_c5(args) if args.workload == "c5" else run_reference(args)
        except FileNotFoundError as e:
            out = {"impl": "reference", "unavailable": f"reference build missing: {e}"}
        print(json.dumps(out))
        return 0
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        tdist.init_process_group("nccl")
        dist = tdist
    out = (run_slabs if args.workload == "c5" else run_ours)(args, rank, world, dist)
    if rank == 0:
        print(json.dumps(out))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
