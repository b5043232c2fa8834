"""Small end-to-end exercise of every kernel path for compute-sanitizer runs
(one tool per gpurun call): K-N1 bulk-store path (CIF, HD), K-N1 cooperative
store path (tiny 48x27), K-N2 (forced and halo spec), ds_run_host, ds_generate.
Checks results against the oracle so a silent race also shows up as a diff."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_1103_4881_b200 as ds
import synth

bad = 0
for W, H, ch, n, kern in [(352, 288, 3, 4, None), (1920, 1080, 3, 2, None), (48, 27, 1, 3, None),
                          (352, 288, 3, 2, ds.DS_KERNEL_GENERIC)]:
    d = ds.Downscaler(W, H, ch, kernel=kern or ds.DS_KERNEL_AUTO)
    fr = synth.random_frames(3, 0, n, W, H, ch, 1)
    y = d(torch.from_numpy(fr).cuda())
    torch.cuda.synchronize()
    ok = np.array_equal(y.cpu().numpy(), oracle.execute_frames(fr, W, H, ch, 1))
    bad += not ok
    print(W, H, ch, "kernel", d.last_kernel(), "ok" if ok else "MISMATCH")
d = ds.Downscaler(352, 288, 3)
fr = synth.random_frames(4, 0, 9, 352, 288)
d.set_host_chunk(4)
out = d.run_host(torch.from_numpy(fr).pin_memory())
torch.cuda.synchronize()
ok = np.array_equal(out.numpy(), oracle.execute_frames(fr, 352, 288))
bad += not ok
print("run_host", "ok" if ok else "MISMATCH")
g = ds.generate_frames(2, 1008, seed=5)
torch.cuda.synchronize()
ok = np.array_equal(g.cpu().numpy().ravel(), synth.random_bytes(5, 0, 2016))
bad += not ok
print("generate", "ok" if ok else "MISMATCH")
sys.exit(1 if bad else 0)
