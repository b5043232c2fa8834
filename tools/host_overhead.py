#!/usr/bin/env python
"""Host cost of one un-captured call for configs[1] (one HD frame): the
Downscaler facade vs a direct C-ABI ds_run vs a bare torch kernel launch."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1103_4881_b200 as ds

torch.cuda.set_device(0)
d = ds.Downscaler(1920, 1080, 3)
x = ds.generate_frames(1, d.in_frame_bytes, seed=1)
y = d.alloc_out(1)
L = ds.lib()
h, xp, yp = d.handle, x.data_ptr(), y.data_ptr()
sp = torch.cuda.current_stream().cuda_stream


def per_call_us(fn, n=5000):
    for _ in range(200):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / n * 1e6


res = {
    "facade_us": per_call_us(lambda: d(x, y)),
    "c_abi_ds_run_us": per_call_us(lambda: L.ds_run(h, xp, 1, yp, sp)),
    "torch_fill_launch_us": per_call_us(lambda: y.fill_(0)),
}
print(json.dumps(res))
