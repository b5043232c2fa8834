#!/usr/bin/env python
"""K-N1 on small frames (QCIF, CIF): band size x CTAs per SM x ring depth
sweep, per-call events over 100 launches; best first."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1103_4881_b200 as ds


def timed(d, x, y, reps=100):
    for _ in range(5):
        d(x, y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        d(x, y)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for W, H, n in ((176, 144, 2000), (352, 288, 2000), (352, 288, 300)):
    d = ds.Downscaler(W, H, 3)
    x = ds.generate_frames(n, d.in_frame_bytes, seed=1)
    y = d.alloc_out(n)
    req = n * (d.in_frame_bytes * 8 // 9 + d.out_frame_bytes)
    res = []
    for band in (0, 8192, 16384, 24576, 49152, 65536):
        d.set_band_bytes(band)
        for ctas in (0, 1, 2, 3, 4, 6):
            for stages in (2, 3, 4):
                try:
                    d.set_tuning(stages, ctas)
                except ds.DSError:
                    continue
                ms = timed(d, x, y)
                res.append((ms, band, ctas, stages, d.launch_shape(n)))
    res.sort()
    d.set_band_bytes(0)
    base = timed(d, x, y)
    print(f"{W}x{H} n={n}: default {base:.4f} ms ({req / base / 1e6:.0f} GB/s); best:")
    for ms, band, ctas, stages, shape in res[:6]:
        print(f"   {ms:.4f} ms ({req / ms / 1e6:.0f} GB/s) band={band} ctas={ctas} stages={stages} grid/block/smem={shape}")
