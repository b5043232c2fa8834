"""ds_run_host chunk-size sweep on the HD 4:2:0 stream (pinned host buffers)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1103_4881_b200 as ds

n = 300
d = ds.Downscaler(1920, 1080, 3)
x = ds.generate_frames(n, d.in_frame_bytes, seed=1)
hin = torch.empty((n, d.in_frame_bytes), dtype=torch.uint8, pin_memory=True)
hin.copy_(x)
hout = torch.empty((n, d.out_frame_bytes), dtype=torch.uint8, pin_memory=True)
for chunk in (2, 5, 10, 20, 40, 75, 150):
    d.set_host_chunk(chunk)
    d.run_host(hin, hout)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        d.run_host(hin, hout)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"chunk={chunk:4d} frames ({chunk * d.in_frame_bytes / 2**20:7.1f} MiB): {n / ms * 1e3:9.0f} frames/s, "
          f"H2D {n * d.in_frame_bytes * 8 / 9 / ms / 1e6:6.1f} GB/s")
