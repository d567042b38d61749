"""ctypes bindings for the CPU checkers (TEST INFRASTRUCTURE).

* liboracle.so  — oracle/voxplane_oracle.c, the C restatement (always built)
* libvoxplane_ref.so — oracle/_ref, the unmodified reference sources compiled
  by oracle/Makefile (present when it was built in the dev container; the
  .so travels to the GPU box with the snapshot)
Both expose the same session ABI producing voxplane_trace.h traces.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2510_01592_b200.native import PipelineParams, default_params  # noqa: F401
from paper_2510_01592_b200.trace import parse_trace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libvoxplane_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


def _ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class CpuSession:
    """One run_frames session on a CPU checker (prefix 'oracle' or 'ref')."""

    _libs: dict = {}

    def __init__(self, which: str, res: float, extent, center, params):
        self.lib = self.load(which)
        self.prefix = "oracle" if which == "oracle" else "ref"
        ext = np.asarray(extent, np.int32)
        c = np.asarray(center, np.float64)
        fn = getattr(self.lib, f"{self.prefix}_session_create")
        fn.restype = C.c_void_p
        self.h = fn(C.c_double(res), _ptr(ext, C.c_int32), _ptr(c, C.c_double), C.byref(params))
        if not self.h:
            raise ValueError("session create failed")
        self.ncells = int(np.prod(ext))

    @classmethod
    def load(cls, which):
        if which not in cls._libs:
            path = ORACLE_SO if which == "oracle" else REF_SO
            lib = C.CDLL(path)
            cls._libs[which] = lib
        return cls._libs[which]

    @staticmethod
    def available(which):
        return os.path.exists(ORACLE_SO if which == "oracle" else REF_SO)

    def frame_raw(self, pts, R, t) -> bytes:
        pts = np.ascontiguousarray(pts, np.float32)
        R = np.ascontiguousarray(R, np.float64).reshape(9)
        t = np.ascontiguousarray(t, np.float64).reshape(3)
        buf = C.POINTER(C.c_uint8)()
        n = C.c_uint64()
        fn = getattr(self.lib, f"{self.prefix}_session_frame")
        rc = fn(C.c_void_p(self.h), _ptr(pts, C.c_float), C.c_uint64(len(pts)), _ptr(R, C.c_double),
                _ptr(t, C.c_double), C.byref(buf), C.byref(n))
        if rc != 0:
            raise ValueError(f"{self.prefix} frame failed rc={rc}")
        data = C.string_at(buf, n.value)
        getattr(self.lib, f"{self.prefix}_free")(buf)
        return data

    def frame(self, pts, R, t):
        return parse_trace(self.frame_raw(pts, R, t))

    def set_fixed(self, fixed=True):
        """Fixed window: no recenter (the C5 map / slab path)."""
        getattr(self.lib, f"{self.prefix}_session_set_fixed")(C.c_void_p(self.h), C.c_int(1 if fixed else 0))

    def cells(self):
        sums = np.zeros((self.ncells, 3))
        cnt = np.zeros(self.ncells, np.uint32)
        st = np.zeros(self.ncells, np.uint8)
        getattr(self.lib, f"{self.prefix}_session_cells")(
            C.c_void_p(self.h), _ptr(sums, C.c_double), _ptr(cnt, C.c_uint32), _ptr(st, C.c_uint8))
        return sums, cnt, st

    def close(self):
        if self.h:
            getattr(self.lib, f"{self.prefix}_session_destroy")(C.c_void_p(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
