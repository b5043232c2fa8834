"""Multi-process path on the CPU (gloo, world_size 2 and 3): frame-block
sharding and the gather to rank 0.  Frames are independent
(S:576), so sharded output must equal the unsharded output.  The
per-rank compute here is the CPU oracle (test infrastructure) standing in
for ds_run; the sharding and gather code is the product's
(paper_1103_4881_b200/dist.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1103_4881_b200.dist import gather_frames, shard_range


def test_shard_ranges_partition_the_stream():
    for total in (0, 1, 7, 300, 3000, 1000):
        for world in (1, 2, 3, 4, 8):
            blocks = [shard_range(total, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == total
            for (a, b), (c, d) in zip(blocks, blocks[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
    # 3000 frames over 8 GPUs -> 375 each; 1000 -> 125
    assert shard_range(3000, 8, 3) == (1125, 1500)
    assert shard_range(1000, 8, 7) == (875, 1000)
    with pytest.raises(ValueError):
        shard_range(10, 0, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, W, H, q, padded=False):
    import oracle
    import synth
    from paper_1103_4881_b200.dist import padded_gather_rows

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_range(total, world, rank)
        frames = synth.random_frames(5, lo, hi - lo, W, H)          # by GLOBAL frame index
        fin, fout = oracle.frame_bytes(W, H)
        local = oracle.execute_frames(frames, W, H) if hi > lo else np.zeros((0, fout), np.uint8)
        local = torch.from_numpy(local.copy())
        m = padded_gather_rows(total, world) // world
        if padded:                       # the shard already sits in an (m, fout) buffer
            buf = torch.full((m, fout), 77, dtype=torch.uint8)
            buf[: hi - lo] = local
            local = buf
        out = torch.empty((world * m, fout), dtype=torch.uint8) if rank == 0 else None
        for rep in range(2):             # the receive buffer is reused across calls
            full = gather_frames(local, total, out=out)
            if rank == 0:
                q.put(full.numpy().copy())
            else:
                assert full is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,total,padded", [(2, 7, False), (3, 5, False), (2, 1, False), (3, 11, False),
                                                (4, 2, False), (2, 7, True), (3, 10, True)])
def test_gloo_sharded_equals_unsharded(world, total, padded):
    """One dist.gather of equal padded shards (the NCCL-safe form: every rank
    enters the same collective) reassembles the stream in frame order for
    uneven shards, empty shards and pre-padded shards."""
    import oracle
    import synth

    W, H = 48, 36
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, W, H, q, padded))
             for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = oracle.execute_frames(synth.random_frames(5, 0, total, W, H), W, H)
    for g in got:
        assert g.shape == want.shape
        assert np.array_equal(g, want)


def test_gather_rejects_a_wrong_shard_shape():
    """A local shard that does not match shard_range fails before any
    collective (no rank can hang in a mismatched gather)."""
    ctx = mp.get_context("spawn")
    port = _free_port()
    p = ctx.Process(target=_bad_shard_worker, args=(port,))
    p.start()
    p.join(timeout=120)
    assert p.exitcode == 0


def _bad_shard_worker(port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        with pytest.raises(ValueError):
            gather_frames(torch.zeros((3, 8), dtype=torch.uint8), 5)
        full = gather_frames(torch.ones((5, 8), dtype=torch.uint8), 5)
        assert full.shape == (5, 8) and int(full.sum()) == 40
    finally:
        dist.destroy_process_group()


def _share_worker(rank, world, port, total, q):
    from paper_1103_4881_b200.dist import share_rank0_tensor

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    # CPU storages travel by shared-memory name under the file_system strategy
    # (the default passes file descriptors, which plain pickling cannot carry);
    # CUDA tensors carry a CUDA IPC handle either way
    mp.set_sharing_strategy("file_system")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = torch.zeros((total, 4), dtype=torch.uint8).share_memory_() if rank == 0 else None
        full = share_rank0_tensor(full)                   # every rank maps rank 0's buffer
        lo, hi = shard_range(total, world, rank)
        full[lo:hi] = rank + 1                            # each rank writes its own slice in place
        dist.barrier()
        if rank == 0:
            q.put(full.numpy().copy())
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,total", [(2, 7), (3, 10)])
def test_share_rank0_tensor_writes_land_in_rank0(world, total):
    """The buffer sharing behind the fused gather (dist.share_rank0_tensor):
    writes each rank makes into its slice of the mapped tensor are rank 0's
    data, with no gather.  On the CPU the mapping is shared memory; ds_run
    uses the same reduction for CUDA tensors (CUDA IPC)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_share_worker, args=(world, _free_port(), total, q), nprocs=world, join=True)
    got = q.get()
    want = np.zeros((total, 4), np.uint8)
    for r in range(world):
        lo, hi = shard_range(total, world, r)
        want[lo:hi] = r + 1
    assert np.array_equal(got, want)
