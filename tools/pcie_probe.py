#!/usr/bin/env python
"""Raw PCIe ceilings for the e2e path: pinned H2D alone, D2H alone, and both
concurrently on two streams (CUDA events), 1 GiB / 160 MiB transfers."""
import json
import torch

torch.cuda.set_device(0)
n_in, n_out = 1 << 30, 160 << 20
hin = torch.empty(n_in, dtype=torch.uint8, pin_memory=True)
hout = torch.empty(n_out, dtype=torch.uint8, pin_memory=True)
din = torch.empty(n_in, dtype=torch.uint8, device="cuda")
dout = torch.empty(n_out, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        din.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2):
        hout.copy_(dout, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


res = {
    "h2d_gbs": n_in / timed(lambda: din.copy_(hin, non_blocking=True)) / 1e6,
    "d2h_gbs": n_out / timed(lambda: hout.copy_(dout, non_blocking=True)) / 1e6,
}
t = timed(both)
res["concurrent_ms"] = t
res["concurrent_h2d_gbs_if_h2d_bound"] = n_in / t / 1e6
print(json.dumps(res))
