"""(usage: python tools/k1_mode_probe.py [W H chroma n], chroma 1 = 4:2:0, 0 = 4:4:4)
Is K-N1's one-CTA-per-SM bimodality (0.97 or 1.02 of the copy peak on HD
4:2:0, run to run) tied to where the buffers land?  One process: allocate the
300-frame input/output as bench.py does, time a CUDA graph of 20 ds_run calls
with --stages 4 --ctas 1 and with the default, print both with the buffers'
address bits.  Run it in several processes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1103_4881_b200 as ds

W, H, CH, n = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (1920, 1080, 1, 300)))
d = ds.Downscaler(W, H, 3, chroma=CH)
x = ds.generate_frames(n, d.in_frame_bytes, seed=1)
y = d.alloc_out(n)
res = {"cfg": f"{W}x{H} chroma={CH} n={n}", "in_ptr_mod_2M": x.data_ptr() % (1 << 21), "in_ptr_mod_1G": x.data_ptr() % (1 << 30),
       "out_ptr_mod_2M": y.data_ptr() % (1 << 21), "out_ptr_mod_1G": y.data_ptr() % (1 << 30)}
bytes_req = n * (d.in_frame_bytes * 8 // 9 + d.out_frame_bytes)
arms = [("one_cta", (4, 1)), ("default", None)]
if os.environ.get("PROBE_ORDER") == "default_first":
    arms.reverse()
for name, tune in arms:
    if tune:
        d.set_tuning(*tune)
    else:
        d.set_band_bytes(0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            d(x, y)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                d(x, y)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(5):
            g.replay()
        e1.record(s)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 100
    res[name] = round(bytes_req / ms / 1e6 / 6548.8, 4)
print(json.dumps(res))
