"""The README's Python usage example, run as written (documentation check)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1103_4881_b200 as ds

d = ds.Downscaler(1920, 1080, 3)                 # HD 4:2:0, SPEC's downscaler
x = torch.empty((300, d.in_frame_bytes), dtype=torch.uint8, device="cuda")   # planar Y, U, V frames
y = d(x)                                         # (300, d.out_frame_bytes): 720x480 + 2 x 360x240 planes

# host-resident frames: chunked, overlapped H2D -> kernel -> D2H (only live rows cross PCIe)
hin = torch.empty((300, d.in_frame_bytes), dtype=torch.uint8, pin_memory=True)
hout = d.run_host(hin); torch.cuda.synchronize()

# any separable Array-OL stage spec (halos, origins, other ratios, negative taps)
halo = ds.make_spec(h=dict(pattern=13, paving=8, origin=-2, weights=[[1, 3, 5, 3, 1], [0, 0, 0, 1, 3, 5, 3, 1],
                                                                     [0, 0, 0, 0, 0, 0, 1, 3, 5, 3, 1]],
                           divisor=13, bias=6))
y2 = ds.Downscaler(1920, 1080, 3, spec=halo)(x)  # runs K-N1g

# a general Array-OL repetitive task: the paper's yhfk (repetition [288, 44])
plane = torch.empty((288, 352), dtype=torch.uint8, device="cuda")
mid = torch.empty((288, 132), dtype=torch.uint8, device="cuda")
ds.run_task(plane, ds.make_tiler((288, 352), (0, 0), [[1, 0], [0, 8]], [[0], [1]], [8]), mid,
            ds.make_tiler((288, 132), (0, 0), [[1, 0], [0, 3]], [[0], [1]], [3]), [288, 44],
            ds.make_body([[1, 5], [0, 0, 0, 3, 3], [0, 0, 0, 0, 0, 0, 5, 1]], 6, 3, n_in=8))
print("readme snippet ok", y.shape, y2.shape, hout.shape, mid.shape)
