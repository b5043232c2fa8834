"""K-N1g on planes the TMA cannot copy: the halo spec on 4K / HD 4:2:0 from an
input pointer 1 byte into its allocation (rows staged by the producer warp),
against the aligned pointer (TMA).  Prints ms per call and in+out GB/s."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch

import paper_1103_4881_b200 as ds
from general_perf import HALO_H, HALO_V

res = {}
for (W, H, n) in ((1920, 1080, 300), (3840, 2160, 100)):
    d = ds.Downscaler(W, H, 3, spec=ds.make_spec(h=HALO_H, v=HALO_V))
    buf = ds.generate_frames(1, n * d.in_frame_bytes + 64, seed=1).view(-1)
    y = d.alloc_out(n)
    for off in (0, 1):
        x = buf[off:off + n * d.in_frame_bytes].view(n, d.in_frame_bytes)
        for _ in range(3):
            d(x, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            d(x, y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        res[f"{W}x{H} off={off}"] = {"ms": ms, "gbs": n * (d.in_frame_bytes + d.out_frame_bytes) / ms / 1e6,
                                     "kernel": ds.KERNEL_NAMES.get(d.last_kernel())}
print(json.dumps(res, indent=1))
