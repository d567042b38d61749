"""Cluster-parallel ablation (pipeline.cpp:304-381, the paper's Fig. 9).

CPU tier: the library's synthetic-cluster generator equals a restatement of
the reference's (rng.hpp:13-64 CounterRng, pipeline.cpp:330-347) in plain
Python -- host code, no device needed.
GPU tier: fit_planes gives bitwise-identical fits in both RansacExecution
modes and equals the CPU oracle on the ablation clusters; run_ablation times
both modes and writes the reference's CSV format."""
import ctypes as C
import math

import numpy as np
import pytest

from paper_2510_01592_b200 import native

M64 = (1 << 64) - 1


class PyCounterRng:
    """rng.hpp:13-64 in Python integers / floats (same libm for log/sin/cos)."""

    def __init__(self, seed, k1=0, k2=0):
        self.s = self.mix((seed + 0x9e3779b97f4a7c15) & M64)
        self.s = self.mix(self.s ^ self.mix((k1 + 0xbf58476d1ce4e5b9) & M64))
        self.s = self.mix(self.s ^ self.mix((k2 + 0x94d049bb133111eb) & M64))
        self.cached = None

    @staticmethod
    def mix(z):
        z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & M64
        z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & M64
        return z ^ (z >> 31)

    def next(self):
        self.s = (self.s + 0x9e3779b97f4a7c15) & M64
        return self.mix(self.s)

    def uniform(self, lo=0.0, hi=1.0):
        u = float(self.next() >> 11) * 2.0 ** -53
        return lo + (hi - lo) * u if (lo, hi) != (0.0, 1.0) else u

    def below(self, n):
        return (self.next() * n) >> 64

    def normal(self):
        if self.cached is not None:
            v, self.cached = self.cached, None
            return v
        u1 = self.uniform()
        while u1 <= 0.0:
            u1 = self.uniform()
        u2 = self.uniform()
        r = math.sqrt(-2.0 * math.log(u1))
        a = 6.283185307179586476925286766559 * u2
        self.cached = r * math.sin(a)
        return r * math.cos(a)


def ref_clusters(cfg, trial, count):
    """pipeline.cpp:330-347."""
    tr = PyCounterRng(cfg.seed, count, trial)
    m = cfg.points_min + tr.below(cfg.points_max - cfg.points_min + 1)
    out = np.zeros((count, m, 3))
    for c in range(count):
        rng = PyCounterRng(cfg.seed ^ 0x5eed, (trial << 8) | c, 7)
        z0 = rng.uniform(0.0, 0.5)
        for i in range(m):
            x = rng.uniform(-0.5, 0.5)
            y = rng.uniform(-0.5, 0.5)
            out[c, i] = (x, y, z0 + 0.004 * rng.normal())
    return out


@pytest.mark.parametrize("trial,count", [(0, 1), (3, 4), (7, 2)])
def test_ablation_generator_matches_reference(trial, count):
    cfg = native.ablation_config(points_min=200, points_max=400, seed=1234)
    got = native.ablation_clusters(cfg, trial, count)
    exp = ref_clusters(cfg, trial, count)
    assert got.shape == exp.shape and got.tobytes() == exp.tobytes()


def fits_of(clusters, execution):
    count, m, _ = clusters.shape
    labels = np.arange(count, dtype=np.int32)
    offs = np.arange(count + 1, dtype=np.uint64) * m
    rp = native.default_params(seed=1234).ransac
    rp.execution = execution
    return native.fit_planes(labels, offs, clusters.reshape(-1, 3), rp)


@pytest.mark.gpu
def test_execution_modes_bitwise_and_oracle():
    # test_plane_fit.cpp:80-102: bitwise determinism across execution modes
    from test_gpu_api import oracle_fit
    cfg = native.ablation_config(points_min=1500, points_max=2500, seed=1234)
    cl = native.ablation_clusters(cfg, 1, 5)
    (a, sa), (b, sb) = fits_of(cl, 0), fits_of(cl, 1)
    assert sa == sb and len(a) == len(b) == 5
    for x, y in zip(a, b):
        assert (x["label"], x["inlier_count"]) == (y["label"], y["inlier_count"])
        assert x["normal"].tobytes() == y["normal"].tobytes() and x["offset"] == y["offset"]
        assert x["inliers"].tobytes() == y["inliers"].tobytes()
    count, m, _ = cl.shape
    rp = native.default_params(seed=1234).ransac
    exp, _ = oracle_fit(np.arange(count, dtype=np.int32), np.arange(count + 1, dtype=np.uint64) * m,
                        cl.reshape(-1, 3), rp)
    for x, y in zip(a, exp):
        assert x["normal"].tobytes() == y["normal"].tobytes() and x["inliers"].tobytes() == y["inliers"].tobytes()


@pytest.mark.gpu
def test_run_ablation_rows_and_csv(tmp_path):
    cfg = native.ablation_config(counts=(1, 4, 16), trials=6, points_min=3000, points_max=5000)
    path = tmp_path / "ablation.csv"
    rows = native.run_ablation(cfg, str(path))
    assert [r["clusters"] for r in rows] == [1, 4, 16] and all(r["trials"] == 6 for r in rows)
    assert all(r["parallel_ms"] > 0 and r["serial_ms"] > 0 for r in rows)
    # serial launches one kernel sequence per cluster: it cannot be faster at 16 clusters
    assert rows[-1]["serial_ms"] > rows[-1]["parallel_ms"]
    lines = path.read_text().splitlines()
    assert lines[0] == "clusters,trials,parallel_ms,serial_ms,ratio,parallel_median_ms,serial_median_ms"
    assert len(lines) == 4 and lines[1].startswith("1,6,")
