"""The every-frame verifier (oracle/verify.py) on the CPU: it passes the
oracle's own stream, pins every corrupted frame, honours first_frame (global
frame index) and the O1 path for a non-default spec."""
import numpy as np

import oracle
import synth
from oracle.verify import verify_stream


def test_verifier_accepts_exact_and_flags_corruption():
    W, H, n = 352, 288, 23
    fr = synth.random_frames(9, 40, n, W, H)
    out = oracle.execute_frames(fr, W, H)
    r = verify_stream(out, W, H, 3, 1, seed=9, first_frame=40, workers=3)
    assert r["bit_exact"] and r["frames_checked"] == n == r["frames_total"]
    bad = out.copy()
    bad[0, 5] ^= 1
    bad[17, -1] ^= 0x80
    r = verify_stream(bad, W, H, 3, 1, seed=9, first_frame=40, workers=4)
    assert not r["bit_exact"] and r["mismatched_frames"] == [0, 17] and r["frames_checked"] == n
    # wrong global offset: every frame differs
    r = verify_stream(out, W, H, 3, 1, seed=9, first_frame=41, workers=1)
    assert r["n_mismatched"] == n


def test_verifier_o1_with_stages():
    W, H, n = 64, 36, 5
    hs = oracle.make_stage(13, 8, -2, [[1, 3, 5, 3, 1], [0, 0, 0, 1, 3, 5, 3, 1]], 13, 6)
    vs = oracle.make_stage(14, 9, -2, [[1, 2, 4, 2, 1], [0, 0, 1, 2, 4, 2, 1]], 10, 5)
    fr = synth.random_frames(2, 0, n, W, H, 3, 0)
    out = oracle.execute_frames(fr, W, H, 3, 0, hs, vs)
    st = (oracle.stage_to_dict(hs), oracle.stage_to_dict(vs))
    assert verify_stream(out, W, H, 3, 0, seed=2, stages=st, workers=2)["bit_exact"]
    out[3, 0] ^= 1
    assert verify_stream(out, W, H, 3, 0, seed=2, stages=st, workers=2)["mismatched_frames"] == [3]
