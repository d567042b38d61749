"""Pinned H2D bandwidth of frame-sized copies (C2: 3.3 MB of float32 points
per frame): one stream vs several streams (copy engines) in flight."""
import torch

mb, frames = 3.3, 30
n = int(mb * 1e6 / 4)
h = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(frames)]
d = [torch.empty(n, device="cuda") for _ in range(frames)]
for ns in (1, 2, 3, 4, 1):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in streams:
            s.wait_event(e0)
        for k in range(frames):
            with torch.cuda.stream(streams[k % ns]):
                d[k].copy_(h[k], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{ns} stream(s): {frames} x {mb} MB in {ms:.2f} ms = {frames * mb / ms:.1f} GB/s, {ms / frames * 1e3:.0f} us/frame")
