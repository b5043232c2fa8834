#!/usr/bin/env python
"""K-N1g on wide frames (halo spec of tools/general_perf.py): HD vs 4K vs 8K
4:2:0, which kernel AUTO picks and the in+out GB/s."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch

import paper_1103_4881_b200 as ds
from general_perf import HALO_H, HALO_V, timed

torch.cuda.set_device(0)
spec = ds.make_spec(h=HALO_H, v=HALO_V)
res = {}
for W, H, n in ((1920, 1080, 300), (3840, 2160, 100), (7680, 4320, 24)):
    H = H // 18 * 18
    d = ds.Downscaler(W, H, 3, spec=spec)
    x = ds.generate_frames(n, d.in_frame_bytes, seed=1)
    y = d.alloc_out(n)
    ms = timed(lambda: d(x, y), 10)
    res[f"{W}x{H}"] = {"frames": n, "kernel": ds.KERNEL_NAMES[d.last_kernel()], "ms": ms,
                       "gbs_in_out": n * (d.in_frame_bytes + d.out_frame_bytes) / ms / 1e6,
                       "k1g_eligible": d.plan.fused_general_eligible,
                       "k1g_bands": list(d.plan.general_band_reps)}
print(json.dumps(res, indent=1))
