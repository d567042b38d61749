"""VXPF frame stream I/O (frame_io.hpp:10-23, frame_io.cpp:110-152).

Little-endian: magic "VXPF", u32 version = 1, then per frame u32 point_count,
12 x f32 pose [R|t] row-major, point_count x 3 f32 sensor-frame xyz.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np


@dataclass
class Frame:
    points: np.ndarray      # (n, 3) float32, sensor frame
    rotation: np.ndarray    # (3, 3) float64 (already f32-quantised)
    translation: np.ndarray  # (3,) float64

    @property
    def R9(self):
        return np.ascontiguousarray(self.rotation, dtype=np.float64).reshape(9)


def read_frames(path: str) -> list[Frame]:
    data = open(path, "rb").read()
    if data[:4] != b"VXPF":
        raise ValueError(f"frame stream: bad magic in {path}")
    (ver,) = struct.unpack_from("<I", data, 4)
    if ver != 1:
        raise ValueError("frame stream: unsupported version")
    o = 8
    frames = []
    while o < len(data):
        if o + 52 > len(data):
            raise ValueError("frame stream: truncated file")
        (n,) = struct.unpack_from("<I", data, o)
        pose = np.frombuffer(data, dtype="<f4", count=12, offset=o + 4).astype(np.float64).reshape(3, 4)
        o += 52
        if o + 12 * n > len(data):
            raise ValueError("frame stream: truncated file")
        pts = np.frombuffer(data, dtype="<f4", count=3 * n, offset=o).reshape(n, 3).copy()
        o += 12 * n
        frames.append(Frame(pts, pose[:, :3].copy(), pose[:, 3].copy()))
    return frames


def write_frames(path: str, frames: list[Frame]) -> None:
    with open(path, "wb") as f:
        f.write(b"VXPF" + struct.pack("<I", 1))
        for fr in frames:
            pts = np.ascontiguousarray(fr.points, dtype="<f4")
            f.write(struct.pack("<I", len(pts)))
            pose = np.concatenate([fr.rotation, fr.translation.reshape(3, 1)], axis=1)
            f.write(pose.astype("<f4").tobytes())
            f.write(pts.tobytes())
