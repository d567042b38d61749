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
