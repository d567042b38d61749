"""One slab per process through the library's vp_slab_frame.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        --master-port P tools/slab_procs.py [--comm gloo|nccl] [--frames F] [--out FILE]

--comm gloo: TorchCommOps over a gloo group (device buffers staged through the
host), so several processes may share one GPU (NCCL refuses duplicate
devices); --comm nccl: the library's NCCL communicator, one GPU per rank.
The window is tests/test_gpu_slabs.py's 300 x 200 x 150 stair window; rank 0
writes the final polygons (write_polygons format) to --out."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2510_01592_b200 import native, scenes, slabs  # noqa: E402
from paper_2510_01592_b200.trace import format_polygons  # noqa: E402

RES, EXTENT, CENTER = 0.01, (300, 200, 150), (0.0, 0.0, 0.5)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--comm", default="gloo", choices=["gloo", "nccl"])
    ap.add_argument("--frames", type=int, default=6)
    ap.add_argument("--lidar", action="store_true")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    dist.init_process_group(a.comm)
    rank, world = dist.get_rank(), dist.get_world_size()
    device = int(os.environ.get("LOCAL_RANK", "0")) if a.comm == "nccl" else 0
    torch.cuda.set_device(device)
    lo, hi = slabs.split_x(EXTENT[0], world)[rank]
    slab = slabs.Slab(RES, EXTENT, CENTER, lo, hi, device=device)
    comm = slabs.nccl_comm(dist, device) if a.comm == "nccl" else slabs.TorchCommOps(dist, device)
    params = native.default_params(seed=5, refine_exact=True)
    frames = scenes.lidar_stair_frames(a.frames) if a.lidar else scenes.stair_frames(a.frames)
    polys = None
    for f in frames:
        polys = slabs.frame(slab, comm, f.points if rank == 0 else None, len(f.points), f.rotation, f.translation,
                            params)
    if rank == 0 and a.out:
        with open(a.out, "w") as fh:
            fh.write(format_polygons(polys))
    if a.comm == "nccl":
        slabs.nccl_comm_destroy(comm)
    slab.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
