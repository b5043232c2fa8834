"""Frame-parallel sharding across the GPUs of one box.

Frames carry no state between them ("no inter-frame
state"), so rank r of P owns the contiguous block
[floor(r N / P), floor((r+1) N / P)) and filters it with no communication.
The only collective is the final gather of output shards to rank 0, in rank
(= frame) order, over NCCL (NVLink/NVSwitch) -- never inside the filter.  The
fused variant (run_sharded_fused_gather) has no separate gather at all: rank 0
shares its output buffer through CUDA IPC and every rank's ds_run stores its
frames straight into it over NVLink, so the transfer overlaps the filtering
unit by unit.

Host-side logic only; the per-rank compute is ds_run (Downscaler).  The
gather works with any torch.distributed backend (NCCL on GPUs, gloo in the
CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous frame block of `rank` (balanced to within one frame)."""
    if total < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("bad shard arguments")
    return (total * rank) // world, (total * (rank + 1)) // world


def gather_frames(local: torch.Tensor, total: int, group=None, dst: int = 0, out=None):
    """Gather every rank's (n_r, frame_bytes) shard to `dst` in frame order
    (collective C-1).  `local` may also be already padded to
    (m, frame_bytes), its first n_r rows valid: then nothing is copied.

    One collective that every rank of the group enters: shards differ by at
    most one frame (shard_range), so each rank pads its shard to
    m = ceil(total / world) frames and the group runs ``dist.gather`` of
    equal-sized tensors (NCCL: one grouped send/recv on the group's
    communicator; gloo: the same on the host).  dst then compacts the
    per-rank blocks [r*m, r*m + n_r) to the frame-ordered [lo_r, hi_r) in
    place, moving rows only towards the front, rank by rank.  No plain
    send/recv is mixed with batched P2P, so NCCL's lazily created
    communicators cannot mismatch.

    `out` (dst only, optional): a (world*m, frame_bytes) receive buffer to
    reuse across calls (padded_gather_rows gives its row count).  Returns the
    (total, frame_bytes) tensor on dst (a view of `out` when given), None
    elsewhere; on the host when the group's backend is gloo."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if local.is_cuda and dist.get_backend(group) == "gloo":
        local = local.cpu()              # gloo moves host tensors (tests on one GPU)
    lo, hi = shard_range(total, world, rank)
    n = hi - lo
    m = padded_gather_rows(total, world) // world
    if local.dim() != 2 or local.shape[0] not in (n, m):
        raise ValueError(f"rank {rank}: local must be ({n} or {m}, frame_bytes) for shard [{lo}, {hi})")
    fb = local.shape[1]
    if total == 0:
        return local.new_empty((0, fb)) if rank == dst else None
    if local.shape[0] < m:               # pad to the common shard size
        send = local.new_zeros((m, fb))
        send[:n].copy_(local[:n])
    else:
        send = local.contiguous()
    if rank != dst:
        dist.gather(send, None, dst=dst, group=group)
        return None
    if out is None:
        out = local.new_empty((world * m, fb))
    elif tuple(out.shape) != (world * m, fb) or out.dtype != local.dtype or out.device != local.device:
        raise ValueError("out must be a (padded_gather_rows(total, world), frame_bytes) buffer like local")
    dist.gather(send, [out[r * m:(r + 1) * m] for r in range(world)], dst=dst, group=group)
    for r in range(1, world):            # compact: rows only move towards the front
        a, b = shard_range(total, world, r)
        if b > a and a != r * m:
            src = out[r * m:r * m + (b - a)]
            out[a:b].copy_(src.clone() if b > r * m else src)   # clone when the ranges overlap
    return out[:total]


def padded_gather_rows(total: int, world: int) -> int:
    """Rows of gather_frames' receive buffer: world x ceil(total / world)."""
    return world * (-(-total // world) if total else 0)


def run_sharded(total_frames: int, w: int, h: int, channels: int = 3, chroma: str = "420",
                seed: int = 1, gather: bool = True, spec=None):
    """Each rank generates its frames by GLOBAL frame index on its own GPU,
    downscales them with one ds_run, then (optionally) rank 0 gathers.

    Returns (rank-0 gathered output or None, local output, (lo, hi))."""
    from . import Downscaler, generate_frames

    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    lo, hi = shard_range(total_frames, world, rank)
    d = Downscaler(w, h, channels, chroma=chroma, spec=spec)
    x = generate_frames(hi - lo, d.in_frame_bytes, seed=seed, first_frame=lo)
    y = d(x)
    full = None
    if gather and world > 1:
        full = gather_frames(y, total_frames)
    elif gather:
        full = y
    return full, y, (lo, hi)


def share_rank0_tensor(t, group=None):
    """Rank 0's tensor, mapped into every rank: serialised with the
    multiprocessing pickler torch registers its sharing reductions with (a
    CUDA tensor becomes a CUDA IPC handle; a CPU tensor a shared-memory name
    under the file_system sharing strategy), the bytes broadcast through the
    process group.  Returns the local view (rank 0: t itself)."""
    import pickle
    from multiprocessing.reduction import ForkingPickler

    import torch.multiprocessing  # noqa: F401  (registers torch's reductions)

    rank = dist.get_rank(group)
    obj = [bytes(ForkingPickler.dumps(t)) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    if rank == 0:
        return t
    return pickle.loads(obj[0])


def run_sharded_fused_gather(total_frames: int, w: int, h: int, channels: int = 3, chroma: str = "420",
                             seed: int = 1, spec=None):
    """Frame-sharded downscaling whose gather is fused into the kernels: rank
    0 allocates the whole output; each rank maps it (CUDA IPC) and runs ds_run
    with its slice [lo, hi) of that buffer as the output, so the bulk stores
    of the output bands go to rank 0's HBM over NVLink while the rank is
    still filtering.  Ranks never wait on one another inside the kernel; one
    host barrier after the local synchronize ends the step.

    Returns (rank-0 full output or None, (lo, hi))."""
    from . import Downscaler, generate_frames

    world = dist.get_world_size()
    rank = dist.get_rank()
    lo, hi = shard_range(total_frames, world, rank)
    d = Downscaler(w, h, channels, chroma=chroma, spec=spec)
    x = generate_frames(hi - lo, d.in_frame_bytes, seed=seed, first_frame=lo)
    full = torch.empty((total_frames, d.out_frame_bytes), dtype=torch.uint8, device="cuda") if rank == 0 else None
    full = share_rank0_tensor(full)
    d.enable_peer(full.device.index)        # explicit, once: ds_run has no side effects
    if hi > lo:
        d(x, out=full[lo:hi])
    torch.cuda.synchronize()
    dist.barrier()
    return (full if rank == 0 else None), (lo, hi)
