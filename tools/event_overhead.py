#!/usr/bin/env python
"""How much do per-launch CUDA event records cost the whole-region rate?
300 HD 4:2:0 frames per ds_run, K back-to-back launches timed (a) with two
events around the whole region, (b) with an event pair around every launch."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1103_4881_b200 as ds

torch.cuda.set_device(0)
d = ds.Downscaler(1920, 1080, 3)
x = ds.generate_frames(300, d.in_frame_bytes, seed=1)
y = d.alloc_out(300)
K = 300
for _ in range(5):
    d(x, y)
torch.cuda.synchronize()
res = {}
for rep in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        d(x, y)
    b.record()
    torch.cuda.synchronize()
    res.setdefault("two_events_ms_per_launch", []).append(a.elapsed_time(b) / K)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * K)]
    for k in range(K):
        evs[2 * k].record()
        d(x, y)
        evs[2 * k + 1].record()
    torch.cuda.synchronize()
    res.setdefault("per_launch_events_ms_per_launch", []).append(evs[0].elapsed_time(evs[-1]) / K)
    res.setdefault("per_launch_mean_ms", []).append(
        sum(evs[2 * k].elapsed_time(evs[2 * k + 1]) for k in range(K)) / K)
print(json.dumps(res))
