"""Regenerate the committed golden fixtures (run in the dev container, where
/root/reference and oracle/_ref exist; the GPU box only reads the outputs).

* tiny_frames.bin  — the reference's own emitted VXPF stream for its
  test_pipeline.cpp tiny_config (run_pipeline with output.emit_frames), via
  oracle/_ref (ref_run_named("live")).
* baseline_frames.bin — the stream of the reference's baseline (height-map)
  run, test_pipeline.cpp:183-192, emitted by oracle/_ref ("baseline").
* pipe_*.polygons_final.txt, pipe_*.iou_report.txt — the reference's golden outputs copied verbatim
  from /root/reference/proj/test_scratch (left there by its own ctest run).
"""
import ctypes as C
import os
import shutil
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
SCRATCH = "/root/reference/proj/test_scratch"


def main():
    ref = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libvoxplane_ref.so"))
    with tempfile.TemporaryDirectory() as d:
        assert ref.ref_run_named(b"live", d.encode()) == 0
        shutil.copy(os.path.join(d, "frames.bin"), os.path.join(HERE, "tiny_frames.bin"))
    with tempfile.TemporaryDirectory() as d:  # the baseline (height-map) run's 4-frame stream
        assert ref.ref_run_named(b"baseline", d.encode()) == 0
        shutil.copy(os.path.join(d, "frames.bin"), os.path.join(HERE, "baseline_frames.bin"))
        with open(os.path.join(d, "polygons_final.txt")) as a, \
                open(os.path.join(SCRATCH, "pipe_baseline", "polygons_final.txt")) as b:
            assert a.read() == b.read(), "reference baseline run does not reproduce its golden"
    for run in ("pipe_t1", "pipe_stair", "pipe_smallobs", "pipe_rosette", "pipe_baseline"):
        dst = os.path.join(HERE, f"{run}.polygons_final.txt")
        shutil.copyfile(os.path.join(SCRATCH, run, "polygons_final.txt"), dst)
        shutil.copyfile(os.path.join(SCRATCH, run, "iou_report.txt"), os.path.join(HERE, f"{run}.iou_report.txt"))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    sys.exit(main())
