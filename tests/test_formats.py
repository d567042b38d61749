"""Frame and polygon formats on the library path:
VXPF streams read into pinned memory (frame_io.cpp:91-116) and written back
(frame_io.cpp:74-89), the %.9g polygon writer (polygon_io.cpp:30-47).

CPU tier: host-only entry points against the Python reader and the golden
files, error cases of test_frame_io.cpp:91-106. GPU tier: replaying the
reference's tiny_config stream from the pinned stream reproduces the golden
polygon file byte for byte."""
import ctypes as C

import numpy as np
import pytest

from paper_2510_01592_b200 import native
from paper_2510_01592_b200.frames import read_frames
from workloads import GOLDEN, golden_text

TINY = f"{GOLDEN}/tiny_frames.bin"


def test_stream_matches_python_reader():
    s = native.Stream(TINY)
    ref = read_frames(TINY)
    assert len(s) == len(ref) == 6
    for i, f in enumerate(ref):
        pts, R, t = s.frame(i)
        assert pts.tobytes() == f.points.tobytes()
        assert R.tobytes() == np.ascontiguousarray(f.rotation).tobytes() and t.tobytes() == f.translation.tobytes()


def test_write_frames_round_trip_bytes(tmp_path):
    out = tmp_path / "copy.bin"
    native.write_frames_binary(out, read_frames(TINY))
    assert out.read_bytes() == open(TINY, "rb").read()


@pytest.mark.parametrize("mutate,msg", [(lambda b: b[:-5], "truncated"), (lambda b: b"VXPX" + b[4:], "bad magic"),
                                         (lambda b: b[:4] + b"\x02\x00\x00\x00" + b[8:], "unsupported version"),
                                         (lambda b: b[:8 + 30], "truncated")])
def test_stream_errors(tmp_path, mutate, msg):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(mutate(open(TINY, "rb").read()))
    with pytest.raises(native.InvalidArgument, match=msg):
        native.Stream(bad)
    with pytest.raises(native.InvalidArgument, match="cannot open"):
        native.Stream(tmp_path / "missing.bin")


def parse_golden(text):
    """polygon_io.cpp:52-104 read_polygons, enough for the writer test."""
    polys, cur, it = [], None, iter(text.splitlines())
    for line in it:
        if not line or line.startswith("#"):
            continue
        kw, *rest = line.split()
        if kw == "polygon":
            cur = {}
            polys.append(cur)
        elif kw == "normal":
            cur["normal"] = [float(v) for v in rest]
        elif kw == "offset":
            cur["offset"] = float(rest[0])
        elif kw == "vertices":
            cur["v3d"] = [[float(v) for v in next(it).split()] for _ in range(int(rest[0]))]
        elif kw == "area":
            cur["area"] = float(rest[0])
        elif kw == "label":
            cur["label"] = int(rest[0])
        elif kw == "inliers":
            cur["inliers"] = int(rest[0])
    return polys


@pytest.mark.parametrize("run", ["pipe_t1", "pipe_stair", "pipe_smallobs", "pipe_rosette"])
def test_polygon_writer_reproduces_golden(tmp_path, run):
    gold = golden_text(run)
    polys = parse_golden(gold)
    arr = (native.Polygon * max(len(polys), 1))()
    keep = []
    for q, p in zip(arr, polys):
        v = np.ascontiguousarray(p["v3d"], np.float64).reshape(-1, 3)
        keep.append(v)
        q.plane.normal[:] = p["normal"]
        q.plane.offset, q.plane.inlier_count, q.plane.cluster_label = p["offset"], p["inliers"], p["label"]
        q.nverts, q.area = len(v), p["area"]
        q.v3d = v.ctypes.data_as(C.POINTER(C.c_double))
    out = native.Polygons(len(polys), arr)
    native.write_polygons(tmp_path / "p.txt", C.byref(out))
    assert (tmp_path / "p.txt").read_text() == gold


@pytest.mark.gpu
def test_replay_pinned_stream_reproduces_golden(tmp_path):
    # replay_pipeline (pipeline.cpp:291-302) on test_pipeline.cpp:15-26's tiny_config
    s = native.Stream(TINY)
    pts0, R0, t0 = s.frame(0)
    pl = native.Pipeline(0.01, (140, 140, 140), t0, native.default_params(seed=77, refine_exact=True))
    out = s.replay(pl)
    native.write_polygons(tmp_path / "polygons_final.txt", out)
    native.lib().vp_polygons_free(out)
    assert (tmp_path / "polygons_final.txt").read_text() == golden_text("pipe_t1")
