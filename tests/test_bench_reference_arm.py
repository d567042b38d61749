"""The reference arm of bench.py (`--impl reference`) times the unmodified
reference (oracle/_ref) on frames the reference renders itself: it must not
map this repository's CUDA library (CPU tier)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "libvoxplane_ref.so")


@pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref not built (no /root/reference here)")
def test_reference_arm_loads_only_the_reference():
    code = ("import bench\n"
            "L, kind = bench.ref_lib()\n"
            "frames = bench.ref_workload_c2(L)\n"
            "assert kind == 'reference' and len(frames) == 30\n"
            "maps = {l.split()[-1] for l in open('/proc/self/maps') if l.rstrip().endswith('.so')}\n"
            "mine = [m for m in maps if 'voxplane' in m or 'oracle' in m]\n"
            "print(sorted(mine))\n"
            "assert all(m.endswith('oracle/_ref/libvoxplane_ref.so') for m in mine), mine\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "libvoxplane_ref.so" in r.stdout
