"""GPU tier: the C++ drop-in API (include/voxplane/*.hpp, reference names)
replays the reference's tiny_config stream; both the Pipeline path and the
per-stage path must write the reference's golden polygon file byte for byte."""
import os
import subprocess

import pytest

from conftest import ROOT
from workloads import GOLDEN, golden_text

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "tests", "cpp", "_build", "drop_in_replay")


def test_cpp_drop_in_reproduces_golden(tmp_path):
    assert os.path.exists(BIN), "run __graft_entry__.build() first"
    r = subprocess.run([BIN, os.path.join(GOLDEN, "tiny_frames.bin"), str(tmp_path), "77", "140"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    gold = golden_text("pipe_t1")
    assert (tmp_path / "polygons_pipeline.txt").read_text() == gold
    assert (tmp_path / "polygons_stages.txt").read_text() == gold


API_BIN = os.path.join(ROOT, "tests", "cpp", "_build", "drop_in_api")


def read_records(path):
    import struct
    data = open(path, "rb").read()
    out, o = {}, 0
    while o < len(data):
        (tl,) = struct.unpack_from("<I", data, o)
        tag = data[o + 4:o + 4 + tl].decode()
        (nb,) = struct.unpack_from("<Q", data, o + 4 + tl)
        out[tag] = data[o + 12 + tl:o + 12 + tl + nb]
        o += 12 + tl + nb
    return out


def test_cpp_api_names_vs_reference(tmp_path):
    """Every other §8(b) name through the C++ facade (tests/cpp/drop_in_api.cpp)
    against the compiled reference (oracle/_ref): CounterRng streams, Jacobi,
    hull_filter / monotone_chain / convex_hull, label_components on explicit
    adjacency lists -- all bit-exact; replay_pipeline -> run_frames with a
    truth file writes the reference's pipe_replay polygons and IoU report byte
    for byte; the height-map baseline through run_frames writes pipe_baseline."""
    import ctypes as C

    import numpy as np

    from cpu_oracles import CpuSession
    assert os.path.exists(API_BIN), "run __graft_entry__.build() first"
    if not CpuSession.available("ref"):
        pytest.skip("oracle/_ref not built")
    L = CpuSession.load("ref")
    rec_path = tmp_path / "records.bin"
    r = subprocess.run([API_BIN, str(rec_path), os.path.join(GOLDEN, "tiny_frames.bin"),
                        os.path.join(GOLDEN, "pipe_replay.truth_in.txt"), os.path.join(GOLDEN, "baseline_frames.bin"),
                        str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    R = read_records(rec_path)
    u64, f64, u32, i32 = np.uint64, np.float64, np.uint32, np.int32

    def ptr(a, t):
        return a.ctypes.data_as(C.POINTER(t))

    # CounterRng
    n = 257
    raw, uni, bel, nrm = np.zeros(n, u64), np.zeros(n), np.zeros(n, u32), np.zeros(n)
    L.ref_rng(C.c_uint64(2025), C.c_uint64(7), C.c_uint64(3), C.c_uint64(n), C.c_uint32(1000003),
              ptr(raw, C.c_uint64), ptr(uni, C.c_double), ptr(bel, C.c_uint32), ptr(nrm, C.c_double))
    assert R["rng_raw"] == raw.tobytes() and R["rng_uniform"] == uni.tobytes()
    assert R["rng_below"] == bel.tobytes() and R["rng_normal"] == nrm.tobytes()
    # jacobi_eigen_sym3
    A = np.frombuffer(R["jac_a"], f64).reshape(-1, 9)
    vals, vecs = np.frombuffer(R["jac_vals"], f64).reshape(-1, 3), np.frombuffer(R["jac_vecs"], f64).reshape(-1, 9)
    for i in range(len(A)):
        a = np.ascontiguousarray(A[i])
        v, w = np.zeros(3), np.zeros(9)
        L.ref_jacobi(ptr(a, C.c_double), ptr(v, C.c_double), ptr(w, C.c_double))
        assert v.tobytes() == vals[i].tobytes() and w.tobytes() == vecs[i].tobytes(), f"jacobi {i}"
    # hulls
    nsets = 0
    for tag, blob in R.items():
        if not tag.startswith("hull_pts_"):
            continue
        nsets += 1
        sid = tag[len("hull_pts_"):]
        dirs = int(sid.split("_")[1])
        pts = np.frombuffer(blob, f64).copy()
        m = len(pts) // 2
        for op, key in ((0, "hull_filter_"), (2, "hull_convex_"), (1, "hull_chain_")):
            if key + sid not in R:
                continue
            out = np.zeros(max(2 * m, 2))
            k = C.c_uint64()
            L.ref_hull(C.c_int(op), ptr(pts, C.c_double), C.c_uint64(m), C.c_int(dirs), ptr(out, C.c_double),
                       C.byref(k))
            assert R[key + sid] == out[:2 * k.value].tobytes(), f"{key}{sid}"
    assert nsets == 12 * 3 * 4
    # label_components on explicit adjacency lists
    for gi in range(6):
        rows = np.frombuffer(R[f"cc_rows_{gi}"], u64).copy()
        cols = np.frombuffer(R[f"cc_cols_{gi}"], i32).copy()
        lab = np.zeros(len(rows) - 1, i32)
        L.ref_label_adjacency(C.c_uint64(len(lab)), ptr(rows, C.c_uint64), ptr(cols if len(cols) else np.zeros(1, i32),
                                                                                C.c_int32), ptr(lab, C.c_int32))
        assert R[f"cc_labels_{gi}"] == lab.tobytes(), f"graph {gi}"
    # quantize_pose: the f32 round trip
    q = np.frombuffer(R["quant_t"], f64)
    assert q.tolist() == [float(np.float32(0.1)), float(np.float32(1.0 / 3.0)), float(np.float32(-2.0 / 7.0))]
    # run_frames through replay_pipeline (pipe_replay: polygons + IoU report)
    rp = tmp_path / "replay"
    assert (rp / "polygons_final.txt").read_text() == golden_text("pipe_t1")
    assert (rp / "polygons_reread.txt").read_text() == golden_text("pipe_t1")
    assert (rp / "iou_report.txt").read_text() == open(os.path.join(GOLDEN, "pipe_t1.iou_report.txt")).read()
    nf = int(np.frombuffer(R["replay_frames"], u64)[0])
    assert (rp / f"polygons_{nf - 1:04d}.txt").read_text() == golden_text("pipe_t1")
    assert all((rp / f"polygons_{k:04d}.txt").exists() for k in range(nf))
    csv = (rp / "timing.csv").read_text().splitlines()
    assert csv[0].startswith("frame,points,voxels,clusters") and len(csv) == nf + 2 and csv[-1].startswith("mean,")
    assert (rp / "labels_final.txt").exists()
    tm = np.frombuffer(R["replay_timing"], f64).reshape(nf, 4)
    assert np.all(tm[:, 0] > 0) and np.all(tm[:, 3] > 0)
    # the baseline path (pipe_baseline)
    assert (tmp_path / "baseline" / "polygons_final.txt").read_text() == golden_text("pipe_baseline")
