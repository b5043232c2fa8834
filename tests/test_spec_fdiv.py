"""The float division of K-N1s (ds_spec.cuh StageInfo::fs / qbyte), checked
exhaustively on the CPU: for every accumulator value a in [amin, amax] of a
stage, the FADD + FFMA sequence

    y = float(2^23 + fs*a - c) - 2^23          (exact)
    G = fmaf(y, fl(1 / (fs*D)), 1.5 * 2^23)     (one rounding, to nearest even)

must leave floor(a / D) in the low byte of G's bit pattern (truncating
division after the round-half-up bias; a >= 0 here, so trunc = floor).  The
FMA is emulated exactly in float64 (y * R is exact there: y < 2^21 and R has a
24-bit mantissa) and rounded once to float32, as the hardware does."""
import numpy as np
import pytest


def _fs(D, B, wpos, wneg, s):
    """StageInfo::fs_for: the same eligibility rules, for one scale s."""
    if D <= 1 or (D & (D - 1)) == 0:
        return 0
    amin, amax = B + 255 * wneg, B + 255 * wpos
    if amin < 0:
        return 0
    c = s * (D - 1) // 2
    if s * amin < c or s * amax >= (1 << 20) or amax // D > 255:
        return 0
    return s


def _check(D, B, wsum):
    s = 1 if D % 2 else 2
    if not _fs(D, B, wsum, 0, s):
        pytest.skip("stage not eligible for the float division")
    c = s * (D - 1) // 2
    a = np.arange(B, B + 255 * wsum + 1, dtype=np.int64)
    want = np.minimum(a // D, 255)
    y = (s * a - c).astype(np.float64)                         # exact in float32 too (< 2^21)
    sD, ymax = s * D, s * (B + 255 * wsum)
    # two-op form: FADD (exact) then FFMA with fl(1 / (fs D))
    R = np.float64(np.float32(1.0) / np.float32(sD))
    G = (y * R + 12582912.0).astype(np.float32)                # single rounding to float32
    low = G.view(np.uint32) & 0xFF
    assert np.array_equal(low, want), (D, B, int(np.argmax(low != want)))
    # one-op form (ymax * fs D < 2^21): FFMA straight on the accumulator's bits
    # 2^23 + y, R = round(2^23 / (fs D)) / 2^23, K = 1.5 * 2^23 - 2^23 R
    if ymax * sD < (1 << 21):
        n = ((1 << 24) // sD + 1) // 2
        F = 8388608.0 + y
        G1 = (F * (n / 8388608.0) + (12582912.0 - n)).astype(np.float32)   # exact product + K, one rounding
        low1 = G1.view(np.uint32) & 0xFF
        assert np.array_equal(low1, want), (D, B, "one-op", int(np.argmax(low1 != want)))


@pytest.mark.parametrize("D,B,wsum", [(13, 6, 13), (10, 5, 10), (6, 3, 6), (3, 1, 3), (5, 2, 5), (7, 3, 7),
                                      (9, 4, 9), (11, 5, 11), (12, 6, 12), (15, 7, 15), (100, 50, 100),
                                      (255, 127, 255), (1000, 500, 1000)])
def test_float_division_exact_over_the_accumulator_range(D, B, wsum):
    _check(D, B, wsum)


def test_halo_and_spec_stages_use_it():
    # bench.py's halo spec (H: D 13, B 6, taps sum 13; V: D 10, B 5, sum 10) and
    # SPEC's hfilter_8to3 (D 6, B 3, sum 6) take the float path; vfilter_9to4
    # (D 8) is a shift
    assert _fs(13, 6, 13, 0, 1) == 1 and _fs(10, 5, 10, 0, 2) == 2 and _fs(6, 3, 6, 0, 2) == 2
    assert _fs(8, 4, 8, 0, 2) == 0
