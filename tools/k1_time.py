#!/usr/bin/env python
"""Time K-N1 (SPEC taps) on BASELINE-shaped streams for same-call A/B of
library builds (tools/gpu_lib_ab.sh TOOL=tools/k1_time.py): per-call CUDA
events over 50 launches; prints ms and required-byte GB/s per config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1103_4881_b200 as ds

CFG = {"hd420": (1920, 1080, 1, 300), "hd444": (1920, 1080, 0, 300), "4k420": (3840, 2160, 1, 300),
       "cif420": (352, 288, 1, 2000), "qcif420": (176, 144, 1, 2000), "cif420_300": (352, 288, 1, 300),
       "hd420_1200": (1920, 1080, 1, 1200), "hd420_3000": (1920, 1080, 1, 3000), "4k420_1000": (3840, 2160, 1, 1000),
       "sd420": (720, 576, 1, 2000)}
out = []
only = sys.argv[1].split(",") if len(sys.argv) > 1 else list(CFG)
for name, (W, H, chroma, n) in CFG.items():
    if name not in only:
        continue
    d = ds.Downscaler(W, H, 3, chroma=chroma)
    x = ds.generate_frames(n, d.in_frame_bytes, seed=1)
    y = d.alloc_out(n)
    for _ in range(5):
        d(x, y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        d(x, y)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 50
    req = n * (d.in_frame_bytes * 8 // 9 + d.out_frame_bytes)
    out.append(f"{name}={ms:.4f}ms({req / ms / 1e6:.0f}GB/s)")
    del x, y
    torch.cuda.empty_cache()
print(" ".join(out), flush=True)
