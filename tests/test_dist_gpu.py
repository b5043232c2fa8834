"""Multi-process sharded path on the GPU: torchrun with 2 and 3 ranks on one
GPU (gloo process group), run_sharded + gather, or the gather fused into the
kernels; with two or more GPUs also one rank per GPU over NCCL.  The gathered
stream must equal the single-process output and the oracle (frames are
independent)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth
from conftest import ROOT

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(tmp_path, ranks, total, mode, backend):
    torch = pytest.importorskip("torch")
    import paper_1103_4881_b200 as ds

    W, H = 352, 288
    out = str(tmp_path / "gathered.npy")
    env = dict(os.environ, DS_DIST_BACKEND=backend)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ranks}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "dist_worker.py"), str(total), str(W), str(H), out, mode]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    got = np.load(out)
    d = ds.Downscaler(W, H, 3)
    x = ds.generate_frames(total, d.in_frame_bytes, seed=3)
    single = d(x).cpu().numpy()
    assert np.array_equal(got, single)
    want = oracle.execute_frames(synth.random_frames(3, 0, total, W, H), W, H)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("mode", ["gather", "fused"])
@pytest.mark.parametrize("ranks,total", [(2, 7), (3, 5)])
def test_torchrun_sharded_gather_one_gpu(tmp_path, ranks, total, mode):
    """Frame-sharded runs gathered to rank 0 equal the 1-GPU run and the
    oracle, with several ranks on one GPU over a gloo process group.  mode
    "fused": no separate gather -- every rank's ds_run writes its frames into
    rank 0's buffer mapped through CUDA IPC (on one GPU the ranks share the
    device; the kernels never wait on one another)."""
    _run(tmp_path, ranks, total, mode, "gloo")


@pytest.mark.parametrize("mode", ["gather", "fused"])
def test_torchrun_sharded_gather_nccl(tmp_path, mode):
    """One rank per GPU over NCCL (NVLink / NVSwitch): the padded dist.gather
    and the fused gather through peer stores (ds_enable_peer).  Needs >= 2
    GPUs; uneven shards (total not a multiple of the rank count)."""
    torch = pytest.importorskip("torch")
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs two or more GPUs (NCCL refuses two ranks on one device)")
    ranks = min(n, 4)
    _run(tmp_path, ranks, 2 * ranks + 1, mode, "nccl")


@pytest.mark.parametrize("mode", ["gather", "fused"])
def test_torchrun_sharded_nccl_single_rank(tmp_path, mode):
    """The NCCL plumbing on one GPU: a one-rank NCCL group (eager init bound
    to the device) runs the padded dist.gather and the broadcast of rank 0's
    CUDA IPC handle (fused mode) through NCCL itself -- the code path the
    multi-GPU run takes, minus the peer traffic."""
    _run(tmp_path, 1, 5, mode, "nccl")
