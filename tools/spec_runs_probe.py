"""K-N1s launch length vs run length (halo spec): is the drop on long launches
(1200 HD / 1000 4K frames) the unit plan?  Times one launch per (frames,
ds_set_run_bands) pair; 0 = the automatic plan (~4 units per CTA slot)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1103_4881_b200 as ds


def timed(fn, steps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


h, v = bench.HALO_SPEC
W, H = int(os.environ.get("W", 1920)), int(os.environ.get("H", 1080))
d = ds.Downscaler(W, H, 3, spec=ds.make_spec(h=h, v=v))
d.set_kernel(ds.DS_KERNEL_FUSED_GENERAL)
L = ds.lib()
for n in (300, 1200):
    x = ds.generate_frames(n, d.in_frame_bytes, seed=1)
    y = d.alloc_out(n)
    row = []
    for rb in (0, 1, 2, 3, 5, 10, 40):
        d.set_run_bands(rb)
        ms = timed(lambda: d(x, y), steps=10)
        row.append(f"rb{rb}:{ms:.3f}ms/{n * (d.in_frame_bytes + d.out_frame_bytes) / ms / 1e6:.0f}GB/s/u{L.ds_units(d.handle, n, ds.DS_KERNEL_FUSED_GENERAL)}")
    print(n, " ".join(row), flush=True)
    del x, y
    torch.cuda.empty_cache()
