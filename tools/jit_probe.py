"""Run-time compilation probe: compile K-N1s for a spec without a built-in
instance and print the NVRTC log (DS_JIT_VERBOSE=1)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("DS_JIT_VERBOSE", "1")
import torch

import paper_1103_4881_b200 as ds

h = dict(pattern=13, paving=8, origin=3, weights=[[1, 2, 3, 0, 0, 0, 0, 0, 0, 0, 0, 1, 1],
                                                  [0, 0, 0, 2, 2, 2, 0, 0, 0, 0, 0, 0, 2],
                                                  [0, 0, 0, 0, 0, 0, 4, 4, 1, 1, 0, 0, 0]], divisor=8, bias=4)
v = dict(pattern=14, paving=9, origin=-5, weights=[[2, 2, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 4], [0, 0, 4, 4],
                                                   [0, 0, 0, 0, 0, 3, 3, 0, 0, 0, 0, 2], [0, 0, 0, 0, 0, 0, 0, 5, 3]],
         divisor=8, bias=4)
d = ds.Downscaler(1920, 1080, 3, spec=ds.make_spec(h=h, v=v))
d.set_kernel(ds.DS_KERNEL_FUSED_GENERAL)
t0 = time.time()
try:
    d.set_general_variant(ds.DS_GENERAL_COMPILED)
    print("compiled in %.2f s" % (time.time() - t0), d.launch_info(300, ds.DS_KERNEL_FUSED_GENERAL))
except ds.DSError as e:
    print("failed:", e)
