"""GPU tier: real slabs in separate processes.

Two ranks run tools/slab_procs.py under torch.distributed.run on the one GPU
of the box: each owns a slab grid and calls the library's vp_slab_frame once
per frame over a gloo-backed communicator table (TorchCommOps; NCCL refuses
two ranks on one device, the exchanges are otherwise the same collectives).
Rank 0's polygons must equal the single grid's."""
import os
import socket
import subprocess
import sys

import pytest

from test_gpu_slabs import CENTER, EXTENT, RES, one_grid  # noqa: F401
from paper_2510_01592_b200 import native, scenes
from paper_2510_01592_b200.trace import format_polygons

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,lidar", [(2, False), (3, True)])
def test_slab_processes_equal_one_grid(tmp_path, world, lidar):
    out = tmp_path / "polys.txt"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.join(ROOT, "tools", "slab_procs.py"),
           "--comm", "gloo", "--frames", "5", "--out", str(out)] + (["--lidar"] if lidar else [])
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    frames = scenes.lidar_stair_frames(5) if lidar else scenes.stair_frames(5)
    _, ref = one_grid(frames, native.default_params(seed=5, refine_exact=True))
    assert len(ref) >= 3
    assert out.read_text() == format_polygons(ref)
