"""Parser for the per-frame stage trace (include/voxplane_trace.h).

The same byte format is produced by the B200 library
(`vp_pipeline_frame_trace`), the C oracle and the compiled reference, so the
parity tests compare every stage of pipeline.cpp:199-213 / :43-85 field by
field.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Trace:
    frame: int = 0
    cleared: int = 0
    freed: int = 0
    touched: int = 0
    discarded: int = 0
    recentered: int = 0
    shift: tuple = (0, 0, 0)
    dropped: int = 0
    origin: tuple = (0.0, 0.0, 0.0)
    occupied_count: int = 0
    occ_idx: np.ndarray = field(default_factory=lambda: np.zeros((0, 3), np.int32))
    occ_mean: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    occ_count: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    occ_status: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    normal: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    ncount: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    valid: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    st_idx: np.ndarray = field(default_factory=lambda: np.zeros((0, 3), np.int32))
    st_mean: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    st_normal: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    labels: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    clusters: list = field(default_factory=list)  # [(label, size)]
    skipped: int = 0
    unfit: int = 0
    fits: list = field(default_factory=list)  # dict(normal, offset, inliers_count, label, inliers)
    refined: list = field(default_factory=list)  # (normal, offset)
    polygons: list = field(default_factory=list)  # dict(normal, offset, inlier_count, label, v2d, v3d, area)


class _Reader:
    def __init__(self, buf: bytes):
        self.b = memoryview(buf)
        self.o = 0

    def take(self, fmt):
        v = struct.unpack_from("<" + fmt, self.b, self.o)
        self.o += struct.calcsize("<" + fmt)
        return v if len(v) > 1 else v[0]

    def arr(self, dtype, count, shape=None):
        dt = np.dtype(dtype).newbyteorder("<")
        n = dt.itemsize * count
        a = np.frombuffer(self.b[self.o:self.o + n], dtype=dt).copy()
        self.o += n
        return a.reshape(shape) if shape else a


def parse_trace(buf: bytes) -> Trace:
    r = _Reader(buf)
    if bytes(r.b[0:4]) != b"VPTR":
        raise ValueError("bad trace magic")
    r.o = 4
    ver = r.take("I")
    if ver != 1:
        raise ValueError(f"trace version {ver}")
    t = Trace()
    t.frame = r.take("I")
    t.cleared, t.freed, t.touched, t.discarded = r.take("4Q")
    t.recentered = r.take("B")
    t.shift = tuple(r.take("3i"))
    t.dropped = r.take("Q")
    t.origin = tuple(r.take("3d"))
    t.occupied_count = r.take("Q")
    V = r.take("Q")
    t.occ_idx = r.arr(np.int32, 3 * V, (V, 3))
    t.occ_mean = r.arr(np.float64, 3 * V, (V, 3))
    t.occ_count = r.arr(np.uint32, V)
    t.occ_status = r.arr(np.uint8, V)
    t.normal = r.arr(np.float64, 3 * V, (V, 3))
    t.ncount = r.arr(np.int32, V)
    t.valid = r.arr(np.uint8, V)
    S = r.take("Q")
    t.st_idx = r.arr(np.int32, 3 * S, (S, 3))
    t.st_mean = r.arr(np.float64, 3 * S, (S, 3))
    t.st_normal = r.arr(np.float64, 3 * S, (S, 3))
    t.labels = r.arr(np.int32, S)
    K = r.take("Q")
    t.clusters = [(r.take("i"), r.take("Q")) for _ in range(K)]
    t.skipped, t.unfit = r.take("2Q")
    F = r.take("Q")
    for _ in range(F):
        n = r.arr(np.float64, 3)
        off = r.take("d")
        cnt, lab = r.take("2i")
        M = r.take("Q")
        inl = r.arr(np.float64, 3 * M, (M, 3))
        t.fits.append(dict(normal=n, offset=off, inlier_count=cnt, label=lab, inliers=inl))
    for _ in range(F):
        n = r.arr(np.float64, 3)
        t.refined.append((n, r.take("d")))
    P = r.take("Q")
    for _ in range(P):
        n = r.arr(np.float64, 3)
        off = r.take("d")
        cnt, lab = r.take("2i")
        nv = r.take("Q")
        v2 = r.arr(np.float64, 2 * nv, (nv, 2))
        v3 = r.arr(np.float64, 3 * nv, (nv, 3))
        area = r.take("d")
        t.polygons.append(dict(normal=n, offset=off, inlier_count=cnt, label=lab, v2d=v2,
                               v3d=v3, area=area))
    if r.o != len(buf):
        raise ValueError(f"trailing bytes in trace: {len(buf) - r.o}")
    return t


def format_polygons(polys) -> str:
    """write_polygons (polygon_io.cpp:30-47) byte format, %.9g."""
    f = lambda v: "%.9g" % v  # noqa: E731
    out = ["# voxplane polygons v1\n"]
    for p in polys:
        n = p["normal"]
        out.append("polygon\n")
        out.append(f"normal {f(n[0])} {f(n[1])} {f(n[2])}\n")
        out.append(f"offset {f(p['offset'])}\n")
        out.append(f"vertices {len(p['v3d'])}\n")
        for v in p["v3d"]:
            out.append(f"{f(v[0])} {f(v[1])} {f(v[2])}\n")
        out.append(f"area {f(p['area'])}\n")
        out.append(f"label {p['label']}\n")
        out.append(f"inliers {p['inlier_count']}\n")
    return "".join(out)
