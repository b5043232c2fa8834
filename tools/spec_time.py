#!/usr/bin/env python
"""Time K-N1g on the halo spec (300 HD 4:2:0 frames), both variants, for
same-call A/B of library builds (tools/gpu_lib_ab.sh).  Prints one line."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1103_4881_b200 as ds


def timed(fn, steps=20):
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
# SPEC_TIME_CFGS="WxHxCHxCHROMA:N,...": other geometries, compiled variant only
cfgs = os.environ.get("SPEC_TIME_CFGS")
if cfgs:
    out = []
    for c in cfgs.split(","):
        g, n = c.split(":")
        W, H, ch, chroma = (int(t) for t in g.split("x"))
        n = int(n)
        d = ds.Downscaler(W, H, ch, chroma=chroma, spec=ds.make_spec(h=h, v=v, chroma=chroma))
        d.set_kernel(ds.DS_KERNEL_FUSED_GENERAL)
        x = ds.generate_frames(n, d.in_frame_bytes, seed=1)
        y = d.alloc_out(n)
        ms = timed(lambda: d(x, y))
        out.append(f"{g}:{n}={ms:.4f}ms({n * (d.in_frame_bytes + d.out_frame_bytes) / ms / 1e6:.0f}GB/s,v{d.last_variant()})")
        del x, y, d
        torch.cuda.empty_cache()
    print(" ".join(out), flush=True)
    sys.exit(0)
W, H, n = 1920, 1080, 300
h, v = bench.HALO_SPEC
d = ds.Downscaler(W, H, 3, spec=ds.make_spec(h=h, v=v))
x = ds.generate_frames(n, d.in_frame_bytes, seed=1)
y = d.alloc_out(n)
out = []
for var, name in ((ds.DS_GENERAL_COMPILED, "compiled"), (ds.DS_GENERAL_RUNTIME, "runtime")):
    try:
        d.set_general_variant(var)
    except ds.DSError:
        continue
    ms = timed(lambda: d(x, y))
    out.append(f"{name}={ms:.4f}ms({n * (d.in_frame_bytes + d.out_frame_bytes) / ms / 1e6:.0f}GB/s)")
print(" ".join(out), flush=True)
