"""Synthetic workloads built from the reference's scene
primitives and rendered by the library's frame source (include/voxplane_scene.h).

Stock scenes / trajectories follow scene_sim.cpp:43-114 and
pipeline.cpp:89-155; C2-C5 compose extra `Box`/`Rect` primitives the way the
survey specifies (the reference only ships Stair5 / SingleStage / Overhang /
SmallObstacle).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import native
from .frames import Frame

STAIR5, SINGLE_STAGE, OVERHANG, SMALL_OBSTACLE = 0, 1, 2, 3


class Box(C.Structure):
    _fields_ = [("min", C.c_double * 3), ("max", C.c_double * 3)]


class Rect(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3), ("half_u", C.c_double),
                ("half_v", C.c_double)]


class Sensor(C.Structure):
    _fields_ = [("kind", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("hfov_deg", C.c_double), ("vfov_deg", C.c_double),
                ("pattern", C.POINTER(C.c_float)), ("npattern", C.c_uint64),
                ("rate_hz", C.c_double), ("max_range", C.c_double), ("noise_sigma", C.c_double)]


@dataclass
class Scene:
    boxes: list = field(default_factory=list)   # (min3, max3)
    rects: list = field(default_factory=list)   # (R 3x3, t3, half_u, half_v)

    def ctypes(self):
        nb, nr = max(len(self.boxes), 1), max(len(self.rects), 1)
        B = (Box * nb)()
        R = (Rect * nr)()
        for i, (lo, hi) in enumerate(self.boxes):
            B[i].min[:] = tuple(float(v) for v in lo)
            B[i].max[:] = tuple(float(v) for v in hi)
        for i, (rot, t, hu, hv) in enumerate(self.rects):
            R[i].R[:] = tuple(float(v) for v in np.asarray(rot, float).reshape(9))
            R[i].t[:] = tuple(float(v) for v in t)
            R[i].half_u, R[i].half_v = hu, hv
        return B, len(self.boxes), R, len(self.rects)


@dataclass
class SensorSpec:
    kind: int = 0            # 0 pinhole, 1 ray pattern
    width: int = 320
    height: int = 240
    hfov_deg: float = 87.0
    vfov_deg: float = 58.0
    pattern: np.ndarray | None = None
    rate_hz: float = 20.0
    max_range: float = 4.0
    noise_sigma: float = 0.003


def _L():
    return native.lib()


def stock_scene(kind: int) -> Scene:
    B = (Box * 16)()
    R = (Rect * 16)()
    nb, nr = C.c_size_t(), C.c_size_t()
    native.check(_L().vp_stock_scene(C.c_int(kind), B, C.byref(nb), R, C.byref(nr)))
    s = Scene()
    for i in range(nb.value):
        s.boxes.append((tuple(B[i].min), tuple(B[i].max)))
    for i in range(nr.value):
        s.rects.append((np.array(R[i].R[:]).reshape(3, 3), tuple(R[i].t), R[i].half_u, R[i].half_v))
    return s


def default_trajectory(kind: int, frames: int, rate_hz: float) -> np.ndarray:
    poses = np.zeros((max(frames, 1) + 2, 12))
    n = _L().vp_default_trajectory(C.c_int(kind), C.c_int(frames), C.c_double(rate_hz),
                                   poses.ctypes.data_as(C.POINTER(C.c_double)))
    return poses[:n]


def straight_trajectory(frames, rate, start, end, pitch0, pitch1) -> np.ndarray:
    spec = np.zeros(21)
    spec[0], spec[1] = frames / rate, rate
    spec[2:5], spec[5:8] = start, end
    spec[8], spec[9] = pitch0, pitch1
    spec[13], spec[14], spec[16], spec[17], spec[18] = 0.5, 0.5, 1.0, 0.17, 0.29
    poses = np.zeros((frames + 2, 12))
    n = _L().vp_scripted_trajectory(C.c_int(0), spec.ctypes.data_as(C.POINTER(C.c_double)),
                                    poses.ctypes.data_as(C.POINTER(C.c_double)), C.c_int(frames + 2))
    return poses[:n]


def spherical_pattern(n: int) -> np.ndarray:
    out = np.zeros((n, 3), np.float32)
    _L().vp_spherical_pattern(C.c_int(n), out.ctypes.data_as(C.POINTER(C.c_float)))
    return out


def rosette_pattern(n: int, cone_deg=70.0, freq_ratio=7.96) -> np.ndarray:
    out = np.zeros((n, 3), np.float32)
    _L().vp_rosette_pattern(C.c_int(n), C.c_double(cone_deg), C.c_double(freq_ratio),
                            out.ctypes.data_as(C.POINTER(C.c_float)))
    return out


def render(scene: Scene, sensor: SensorSpec, poses: np.ndarray, seed: int, threads: int = 0,
           first_index: int = 0) -> list[Frame]:
    """render_frame (scene_sim.cpp:186-236) for each pose, frame index = position."""
    B, nb, R, nr = scene.ctypes()
    s = Sensor()
    s.kind, s.width, s.height = sensor.kind, sensor.width, sensor.height
    s.hfov_deg, s.vfov_deg = sensor.hfov_deg, sensor.vfov_deg
    pat = None
    if sensor.pattern is not None:
        pat = np.ascontiguousarray(sensor.pattern, np.float32)
        s.pattern = pat.ctypes.data_as(C.POINTER(C.c_float))
        s.npattern = len(pat)
    s.rate_hz, s.max_range, s.noise_sigma = sensor.rate_hz, sensor.max_range, sensor.noise_sigma
    out = []
    for fi, pose in enumerate(poses):
        Rm = np.ascontiguousarray(pose[:9], np.float64)
        t = np.ascontiguousarray(pose[9:12], np.float64)
        pts = C.POINTER(C.c_float)()
        n = C.c_uint64()
        qR = np.zeros(9)
        qt = np.zeros(3)
        native.check(_L().vp_render_frame(B, C.c_size_t(nb), R, C.c_size_t(nr), C.byref(s),
                                          Rm.ctypes.data_as(C.POINTER(C.c_double)),
                                          t.ctypes.data_as(C.POINTER(C.c_double)), C.c_uint64(seed),
                                          C.c_uint64(fi + first_index), C.c_int(threads), C.byref(pts), C.byref(n),
                                          qR.ctypes.data_as(C.POINTER(C.c_double)),
                                          qt.ctypes.data_as(C.POINTER(C.c_double))))
        arr = np.ctypeslib.as_array(pts, (n.value, 3)).copy() if n.value else np.zeros((0, 3), np.float32)
        _L().vp_free(pts)
        out.append(Frame(arr, qR.reshape(3, 3), qt))
    return out


def horizontal_rect(center, hx, hy):
    return (np.eye(3), tuple(center), hx, hy)


# ----------------------------------------------------------------------------
# Workloads
# ----------------------------------------------------------------------------
@dataclass
class Workload:
    name: str
    frames: list
    resolution: float
    extent: tuple
    seed: int

    @property
    def points(self):
        return sum(len(f.points) for f in self.frames)


def tiny_frames():
    """test_pipeline.cpp:15-26 tiny_config: SmallObstacle, 96x72, 6 frames, seed 77."""
    sensor = SensorSpec(width=96, height=72)
    return render(stock_scene(SMALL_OBSTACLE), sensor, default_trajectory(SMALL_OBSTACLE, 6, 20.0), 77)


def stair_frames(frames=25):
    """test_pipeline.cpp:77-88: Stair5, 240x180, 25 frames, seed 5, 200^3."""
    sensor = SensorSpec(width=240, height=180)
    return render(stock_scene(STAIR5), sensor, default_trajectory(STAIR5, frames, 20.0), 5)


def lidar_stair_frames(frames=6, rays=200_000, seed=11):
    """Stair5 seen by a spherical ray pattern along the Stair5 trajectory:
    incoherent rays (the brick-mask walk) for tests."""
    sensor = SensorSpec(kind=1, pattern=spherical_pattern(rays), max_range=4.0)
    return render(stock_scene(STAIR5), sensor, default_trajectory(STAIR5, frames, 20.0), seed)


def stepping_stone_boxes():
    """The six 0.3 x 0.3 m stepping stones (0.05-0.15 m) C2 adds on the Stair5 approach floor."""
    heights = [0.05, 0.08, 0.10, 0.12, 0.15, 0.06]
    out = []
    k = 0
    for cx in (-1.05, -0.72, -0.39):
        for cy in (-0.3, 0.3):
            h = heights[k]
            k += 1
            out.append(((cx - 0.15, cy - 0.15, 0.0), (cx + 0.15, cy + 0.15, h)))
    return out


def stepping_stones():
    """C2 scene: Stair5 plus six 0.3 x 0.3 m stepping stones (0.05-0.15 m) on the approach floor."""
    s = stock_scene(STAIR5)
    s.boxes.extend(stepping_stone_boxes())
    return s


@dataclass
class WorkloadSpec:
    """Scene, sensor, poses and grid of a workload before rendering."""
    name: str
    scene: Scene
    sensor: SensorSpec
    poses: np.ndarray
    seed: int
    resolution: float
    extent: tuple
    first_index: int = 0


def workload_spec(name: str, frames: int | None = None) -> WorkloadSpec:
    """SURVEY.md §8(d) configs C1-C5."""
    if name == "c1":  # Stair5, one 640x480 frame, 0.05 m, 100^3
        sensor = SensorSpec(width=640, height=480, max_range=6.0, rate_hz=30.0)
        poses = default_trajectory(STAIR5, 30, 30.0)[:1]
        return WorkloadSpec(name, stock_scene(STAIR5), sensor, poses, 2025, 0.05, (100, 100, 100))
    if name == "c2":  # Stair5 + stepping stones, 30 frames, 640x480, 0.01 m, 500^3
        n = frames or 30
        sensor = SensorSpec(width=640, height=480, max_range=6.0, rate_hz=30.0)
        poses = default_trajectory(STAIR5, n, 30.0)
        return WorkloadSpec(name, stepping_stones(), sensor, poses, 2025, 0.01, (500, 500, 500))
    if name == "c3":  # open-tread stairs + overhanging table, 0.01 m, 500^3
        n = frames or 30
        s = Scene()
        s.rects.append(horizontal_rect((0.3, 0.0, 0.0), 1.5, 1.5))
        for k in range(5):
            s.rects.append(horizontal_rect((0.145 + 0.29 * k, 0.0, 0.17 * (k + 1)), 0.12, 0.6))
        s.rects.append(horizontal_rect((-0.8, 0.0, 0.75), 0.6, 0.4))
        sensor = SensorSpec(width=640, height=480, max_range=6.0, rate_hz=30.0)
        poses = straight_trajectory(n, 30.0, (-1.7, 0.0, 0.45), (0.1, 0.0, 0.45), -35.0, 10.0)
        return WorkloadSpec(name, s, sensor, poses, 2025, 0.01, (500, 500, 500))
    if name == "c4":  # ~1M-point sphere LiDAR in Stair5 + 20x20 m floor
        n = frames or 30
        s = stock_scene(STAIR5)
        s.rects.append(horizontal_rect((0.0, 0.0, -0.001), 10.0, 10.0))
        sensor = SensorSpec(kind=1, pattern=spherical_pattern(2_000_000), max_range=10.0, rate_hz=30.0)
        poses = default_trajectory(STAIR5, n, 30.0)
        return WorkloadSpec(name, s, sensor, poses, 2025, 0.01, (500, 500, 500))
    if name == "c5":
        n = frames or 6
        sensor = SensorSpec(kind=1, pattern=spherical_pattern(1_000_000), max_range=10.0, rate_hz=10.0)
        return WorkloadSpec(name, c5_scene(), sensor, c5_poses(n), 2025, 0.01, C5_EXTENT)
    raise ValueError(name)


def workload(name: str, frames: int | None = None) -> Workload:
    """SURVEY.md §8(d) configs C1-C4 (C5 is the multi-GPU map), rendered on the host."""
    if name == "c5":
        return c5_workload(frames or 6)
    w = workload_spec(name, frames)
    return Workload(name, render(w.scene, w.sensor, w.poses, w.seed), w.resolution, w.extent, w.seed)


class DeviceFrameSource:
    """render_frame on the GPU (vp_frame_source_*): frames stay in HBM."""

    def __init__(self, scene: Scene, sensor: SensorSpec, seed: int, device: int = 0):
        B, nb, R, nr = scene.ctypes()
        s = Sensor()
        s.kind, s.width, s.height = sensor.kind, sensor.width, sensor.height
        s.hfov_deg, s.vfov_deg = sensor.hfov_deg, sensor.vfov_deg
        self._pat = None
        if sensor.pattern is not None:
            self._pat = np.ascontiguousarray(sensor.pattern, np.float32)
            s.pattern = self._pat.ctypes.data_as(C.POINTER(C.c_float))
            s.npattern = len(self._pat)
        s.rate_hz, s.max_range, s.noise_sigma = sensor.rate_hz, sensor.max_range, sensor.noise_sigma
        self.h = C.c_void_p()
        self.device = device
        native.check(_L().vp_frame_source_create(B, C.c_size_t(nb), R, C.c_size_t(nr), C.byref(s),
                                                 C.c_uint64(seed), C.c_int(device), C.byref(self.h)))

    def render_ptr(self, pose, index):
        """(device pointer, n, R 3x3, t) of frame `index` at pose (12 doubles R|t)."""
        Rm = np.ascontiguousarray(pose[:9], np.float64)
        t = np.ascontiguousarray(pose[9:12], np.float64)
        ptr = C.c_void_p()
        n = C.c_uint64()
        qR, qt = np.zeros(9), np.zeros(3)
        native.check(_L().vp_frame_source_render(self.h, Rm.ctypes.data_as(C.POINTER(C.c_double)),
                                                 t.ctypes.data_as(C.POINTER(C.c_double)), C.c_uint64(index),
                                                 C.byref(ptr), C.byref(n),
                                                 qR.ctypes.data_as(C.POINTER(C.c_double)),
                                                 qt.ctypes.data_as(C.POINTER(C.c_double))))
        return ptr.value or 0, n.value, qR.reshape(3, 3), qt

    def render(self, pose, index):
        """Frame with its points copied to the host (tests)."""
        import torch

        from .slabs import _dev_bytes
        ptr, n, R, t = self.render_ptr(pose, index)
        pts = _dev_bytes(ptr, 12 * n, self.device).view(torch.float32).view(-1, 3).cpu().numpy().copy()
        return Frame(pts, R, t)

    def close(self):
        if self.h:
            _L().vp_frame_source_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def c5_scene() -> Scene:
    """C5: 20 x 20 m floor, 20 x 10 m mezzanine at 1.5 m, two 9-step box stairs
    up to it, ten 1.2 x 0.8 m tables at 0.75 m."""
    s = Scene()
    s.rects.append(horizontal_rect((0.0, 0.0, 0.0), 10.0, 10.0))
    s.rects.append(horizontal_rect((0.0, 5.0, 1.5), 10.0, 5.0))
    rise, run, width = 1.5 / 9.0, 0.3, 1.2
    for x0 in (-6.0, 5.0):
        y0 = -9 * run
        for k in range(9):
            s.boxes.append(((x0, y0 + k * run, 0.0), (x0 + width, y0 + (k + 1) * run, (k + 1) * rise)))
    for i in range(5):
        for j in range(2):
            s.rects.append(horizontal_rect((-8.0 + 3.5 * i, -6.0 + 4.0 * j, 0.75), 0.6, 0.4))
    return s


C5_EXTENT = (2000, 2000, 300)
C5_CENTER = (0.0, 0.0, 1.45)


def c5_workload(frames: int, rays: int = 1_000_000, first: int = 0) -> Workload:
    """Sphere LiDAR (1M rays, 10 m) along a lawnmower path at 0.6 m over the
    C5 scene; fixed 2000 x 2000 x 300 window at 0.01 m. Frame indices
    first .. first + frames - 1 of the path."""
    poses = c5_poses(first + frames)[first:]
    sensor = SensorSpec(kind=1, pattern=spherical_pattern(rays), max_range=10.0, rate_hz=10.0)
    out = render(c5_scene(), sensor, poses, 2025, first_index=first)
    return Workload("c5", out, 0.01, C5_EXTENT, 2025)


def c5_poses(frames: int) -> np.ndarray:
    """Lawnmower path: lanes of 4 poses along x, 3 m apart in y."""
    poses = []
    for k in range(frames):
        lane = k // 4
        u = (k % 4) / 3.0
        x = -7.0 + 14.0 * (u if lane % 2 == 0 else 1.0 - u)
        y = -7.0 + 3.0 * lane
        R = np.eye(3)
        poses.append(np.concatenate([R.reshape(9), [x, y, 0.6]]))
    return np.array(poses)
