"""Multi-process sharded path on the GPU: torchrun with 2 and 3 ranks on one
GPU (gloo backend), run_sharded + gather; the gathered stream must equal the
single-process output and the oracle (frames are independent)."""
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


@pytest.mark.parametrize("mode", ["nccl", "fused"])
@pytest.mark.parametrize("ranks,total", [(2, 7), (3, 5)])
def test_torchrun_sharded_gather(tmp_path, ranks, total, mode):
    """Frame-sharded runs gathered to rank 0 equal the 1-GPU run and the
    oracle.  mode "fused": no separate gather -- every rank's ds_run writes
    its frames into rank 0's buffer mapped through CUDA IPC (on one GPU the
    ranks share the device; the kernels never wait on one another)."""
    torch = pytest.importorskip("torch")
    import paper_1103_4881_b200 as ds

    W, H = 352, 288
    out = str(tmp_path / "gathered.npy")
    env = dict(os.environ, DS_DIST_BACKEND="gloo")
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
