"""Profiling targets for the non-headline rows (run under ncu, one kernel family each):
   python tools/prof_cases.py tasks   -> K-N3 ds_htask_kernel + ds_vtask_kernel (300 HD 4:2:0)
   python tools/prof_cases.py general -> K-N1g on the halo spec (300 HD 4:2:0)
   python tools/prof_cases.py runtask -> ds_run_task on yhfk over 300 HD luma planes (3-D task: dense path)
   python tools/prof_cases.py runtask_v -> ds_run_task on the V task over 300 HD luma planes (column path)
   python tools/prof_cases.py sd420 -> K-N1 on 300 PAL SD 4:2:0 frames (wide luma + narrow chroma planes)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch

import paper_1103_4881_b200 as ds
from general_perf import HALO_H, HALO_V

what = sys.argv[1]
if what == "tasks":
    d = ds.Downscaler(1920, 1080, 3)
    x = ds.generate_frames(300, d.in_frame_bytes, seed=1)
    mid = torch.empty((300, d.mid_frame_bytes), dtype=torch.uint8, device="cuda")
    y = d.alloc_out(300)
    for _ in range(3):
        d.htask(x, mid)
        d.vtask(mid, y)
elif what == "sd420":
    d = ds.Downscaler(720, 576, 3)
    x = ds.generate_frames(300, d.in_frame_bytes, seed=1)
    y = d.alloc_out(300)
    for _ in range(3):
        d(x, y)
elif what == "general":
    d = ds.Downscaler(1920, 1080, 3, spec=ds.make_spec(h=HALO_H, v=HALO_V))
    x = ds.generate_frames(300, d.in_frame_bytes, seed=1)
    y = d.alloc_out(300)
    for _ in range(3):
        d(x, y)
elif what == "runtask_v":
    # the paper's V task as one 3-D task (the column path)
    n, H, W = 300, 1080, 1920
    Wm, Ho = W // 8 * 3, H // 9 * 4
    mid = ds.generate_frames(n, H * Wm, seed=2).view(n, H, Wm)
    out = torch.empty((n, Ho, Wm), dtype=torch.uint8, device="cuda")
    spec = ds.ds_default_spec()
    vw = [[spec.v.weight[k][i] for i in range(9)] for k in range(4)]
    tin = ds.make_tiler((n, H, Wm), (0, 0, 0), [[1, 0, 0], [0, 9, 0], [0, 0, 1]], [[0], [1], [0]], [9])
    tout = ds.make_tiler((n, Ho, Wm), (0, 0, 0), [[1, 0, 0], [0, 4, 0], [0, 0, 1]], [[0], [1], [0]], [4])
    for _ in range(3):
        ds.run_task(mid, tin, out, tout, [n, H // 9, Wm], ds.make_body(vw, 8, 4, n_in=9))
elif what == "runtask":
    n, H, W = 300, 1080, 1920
    x = ds.generate_frames(n, W * H, seed=1)
    mid = torch.empty((n, H, W // 8 * 3), dtype=torch.uint8, device="cuda")
    spec = ds.ds_default_spec()
    hw = [[spec.h.weight[k][i] for i in range(8)] for k in range(3)]
    tin = ds.make_tiler((n, H, W), (0, 0, 0), [[1, 0, 0], [0, 1, 0], [0, 0, 8]], [[0], [0], [1]], [8])
    tout = ds.make_tiler((n, H, W // 8 * 3), (0, 0, 0), [[1, 0, 0], [0, 1, 0], [0, 0, 3]], [[0], [0], [1]], [3])
    for _ in range(3):
        ds.run_task(x, tin, mid, tout, [n, H, W // 8], ds.make_body(hw, 6, 3, n_in=8))
torch.cuda.synchronize()
print("ok", what)
