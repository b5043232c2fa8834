"""torchrun worker for tests/test_dist_gpu.py: frame-sharded downscaling
(paper_1103_4881_b200.dist.run_sharded) + the process-group gather to rank 0
(argv[5] == "gather"), or the gather fused into the kernels (argv[5] ==
"fused": run_sharded_fused_gather, every rank writes into rank 0's buffer
through CUDA IPC); rank 0 saves the stream.  The process-group backend is
DS_DIST_BACKEND: "gloo" lets several ranks share one GPU (their kernels never
wait on one another; gloo moves the shards through the host), "nccl" needs
one GPU per rank."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

from paper_1103_4881_b200.dist import run_sharded, run_sharded_fused_gather

total, W, H, out_path = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
mode = sys.argv[5] if len(sys.argv) > 5 else "gather"
backend = os.environ.get("DS_DIST_BACKEND", "nccl")
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local % torch.cuda.device_count())
if backend == "nccl":     # eager NCCL init bound to this rank's GPU
    dist.init_process_group(backend, device_id=torch.device("cuda", local))
else:
    dist.init_process_group(backend)
if mode == "fused":
    full, (lo, hi) = run_sharded_fused_gather(total, W, H, 3, seed=3)
else:
    full, mine, (lo, hi) = run_sharded(total, W, H, 3, seed=3)
torch.cuda.synchronize()
if dist.get_rank() == 0:
    np.save(out_path, full.cpu().numpy())
dist.barrier()
dist.destroy_process_group()
