"""K-N1g on the 300-frame HD stream with SPEC taps or the halo spec (profiling target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1103_4881_b200 as ds
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from general_perf import HALO_H, HALO_V
spec = ds.make_spec(h=HALO_H, v=HALO_V) if "halo" in sys.argv else None
d = ds.Downscaler(1920, 1080, 3, spec=spec, kernel=ds.DS_KERNEL_FUSED_GENERAL)
x = ds.generate_frames(300, d.in_frame_bytes, seed=1)
y = d.alloc_out(300)
for _ in range(4):
    d(x, y)
torch.cuda.synchronize()
print("ok", d.last_kernel())
