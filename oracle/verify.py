"""Every-frame verification of a GPU output stream against the CPU oracle --
TEST INFRASTRUCTURE (like the rest of oracle/).

SURVEY 8.d: "Verification is separate from timing.  For C2-C4, every GPU
frame is compared byte for byte against O1/O2.  On large configs this fans
out across all host cores as independent single-threaded oracle processes,
and it is reported only as verification wall time with its core count."
The bar is SPEC.md:646 (acceptance 1: bit-identical output, zero tolerance)
over the whole stream.

Each worker process is single-threaded: it regenerates its frames from the
seeded counter-hash generator by GLOBAL frame index (synth/, the only code
both sides share; no input or expected value comes from the CUDA path),
runs the oracle on them -- O2, SPEC's direct nested loops, for
SPEC's taps, else O1, the tiler executor, with the given stages
-- and compares with the GPU's bytes.  The GPU output array is inherited by
the forked workers (copy-on-write, read only); workers never touch CUDA.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

_JOB = {}


def _init(job):
    _JOB.clear()
    _JOB.update(job)
    try:                                   # undo any 1-core pinning of the parent (cpu_baseline)
        os.sched_setaffinity(0, job["cores"])
    except Exception:
        pass


def _check_range(rng):
    import oracle
    import synth

    a, b = rng
    j = _JOB
    W, H, ch, chroma = j["W"], j["H"], j["channels"], j["chroma"]
    gpu = j["gpu"]
    bad = []
    step = j["batch"]
    buf = None
    for f0 in range(a, b, step):
        m = min(step, b - f0)
        if buf is None or buf.shape[0] != m:
            buf = np.empty((m, j["fin"]), np.uint8)
        fr = synth.random_frames(j["seed"], j["first_frame"] + f0, m, W, H, ch, chroma, out=buf)
        if j["stages"] is None:
            want = oracle.direct_frames(fr, W, H, ch, chroma)                      # O2
        else:
            hs, vs = (oracle.stage_from_dict(d) for d in j["stages"])
            want = oracle.execute_frames(fr, W, H, ch, chroma, hs, vs)             # O1
        got = gpu[f0:f0 + m]
        if not np.array_equal(got, want):
            for k in range(m):
                if not np.array_equal(got[k], want[k]):
                    bad.append(f0 + k)
    return b - a, bad


def verify_stream(gpu_out: np.ndarray, W: int, H: int, channels: int, chroma: int, seed: int,
                  first_frame: int = 0, stages=None, workers: int | None = None,
                  frames: int | None = None) -> dict:
    """Compare gpu_out[k] (host u8 array (n, out_frame_bytes)) with the oracle
    on frame first_frame + k of the seeded stream, for k < frames (default:
    all n).  stages: None for SPEC's taps (O2), else (h, v) oracle Stage
    dicts (O1).  Returns {"frames_checked", "frames_total", "bit_exact",
    "mismatched_frames" (first 16), "oracle", "workers", "wall_s"}."""
    import oracle

    n = gpu_out.shape[0] if frames is None else min(frames, gpu_out.shape[0])
    fin, fout = (oracle.frame_bytes(W, H, channels, chroma) if stages is None else
                 oracle.frame_bytes(W, H, channels, chroma, *(oracle.stage_from_dict(d) for d in stages)))
    if gpu_out.ndim != 2 or gpu_out.shape[1] != fout:
        raise ValueError("gpu_out must be (n, out_frame_bytes)")
    try:
        cores = sorted(os.sched_getaffinity(0))
    except Exception:
        cores = list(range(os.cpu_count() or 1))
    all_cores = set(range(os.cpu_count() or 1))
    workers = max(1, min(workers or len(all_cores), n or 1))
    # ~4 chunks per worker, at least one frame each, so the tail is short
    per = max(1, -(-n // (workers * 4)))
    ranges = [(a, min(n, a + per)) for a in range(0, n, per)]
    job = dict(W=W, H=H, channels=channels, chroma=chroma, seed=seed, first_frame=first_frame,
               stages=None if stages is None else [dict(s) for s in stages], gpu=gpu_out, fin=fin,
               batch=max(1, min(8, (64 << 20) // max(fin, 1))), cores=all_cores)
    t0 = time.perf_counter()
    bad, done = [], 0
    if workers == 1 or n <= 1:
        _init(job)
        for r in ranges:
            c, b = _check_range(r)
            done += c
            bad += b
        try:
            os.sched_setaffinity(0, set(cores))
        except Exception:
            pass
    else:
        ctx = mp.get_context("fork")   # workers inherit gpu_out; they never touch CUDA
        with ctx.Pool(workers, initializer=_init, initargs=(job,)) as pool:
            for c, b in pool.imap_unordered(_check_range, ranges):
                done += c
                bad += b
    bad.sort()
    return {"frames_checked": done, "frames_total": n, "bit_exact": done == n and not bad,
            "mismatched_frames": bad[:16], "n_mismatched": len(bad),
            "oracle": "O2 direct loops (S:547-551)" if stages is None else "O1 tiler executor (S:517-520)",
            "workers": workers, "wall_s": round(time.perf_counter() - t0, 2),
            "seed": seed, "first_frame": first_frame}
