"""Pins for the CPU oracle (oracle/ds_oracle.c) -- all CPU, `-m "not gpu"`.

Each test pins the oracle to something other than itself: SPEC's worked
examples, values printed in the paper, hand-worked goldens, closed forms
re-derived from SPEC's interpolation positions, invariants, and an exact
rational brute force.  P:n = PAPER.md line n, S:n = SPEC.md line n.
"""
import hashlib
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from conftest import GOLDEN


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def _plane_from_rule(rule):
    W, H = rule["W"], rule["H"]
    y, x = np.mgrid[0:H, 0:W]
    if rule["kind"] == "linear":
        return ((rule["a"] * y + rule["b"] * x) % 256).astype(np.uint8)
    if rule["kind"] == "checkerboard":
        return (((x + y) & 1) * 255).astype(np.uint8)
    raise ValueError(rule)


def _yhfk_in_tiler(W=352, H=288):
    # SURVEY sec. 8 H input tiler: origin 0, paving [[1,0],[0,8]], fitting [[0],[1]], pattern [8]
    return oracle.make_tiler((H, W), (0, 0), [[1, 0], [0, 8]], [[0], [1]], [8])


# ------------------------------------------------------------------ tilers --
class TestTilerSpecExamples:
    def test_element_index_s254(self):
        # S:254 origin (0,0), paving [[1,0],[0,8]], fitting (0,1)^T, array (288,352), r=(0,1), f=(3) -> (0,11)
        assert oracle.element_index(_yhfk_in_tiler(), (0, 1), (3,)) == (0, 11)

    def test_element_index_s255_identity(self):
        # S:255 zero origin, identity paving, zero fitting, r=(5,7), f=(0,0) -> (5,7)
        t = oracle.make_tiler((10, 10), (0, 0), [[1, 0], [0, 1]], [[0, 0], [0, 0]], [1, 1])
        assert oracle.element_index(t, (5, 7), (0, 0)) == (5, 7)

    def test_element_index_s256_wrap(self):
        # S:256 origin (350), paving [(0)], fitting [(1)], array (352), r=(0), f=(5) -> (3)
        t = oracle.make_tiler((352,), (350,), [[0]], [[1]], [8])
        assert oracle.element_index(t, (0,), (5,)) == (3,)

    def test_element_index_negative_modulo(self):
        # S:251 "the mathematical (always non-negative) modulo"
        t = oracle.make_tiler((352,), (-3,), [[0]], [[1]], [8])
        assert oracle.element_index(t, (0,), (1,)) == (350,)

    def test_extract_pattern_s264(self):
        # S:264 yhfk input tiler, r=(0,1), rows valued by column 0..351 -> [8..15]
        arr = np.tile(np.arange(352) % 256, (288, 1)).astype(np.uint8)
        assert list(oracle.extract_pattern(arr, _yhfk_in_tiler(), (0, 1))) == list(range(8, 16))

    def test_extract_pattern_s265_constant(self):
        arr = np.full((288, 352), 42, np.uint8)
        for r in [(0, 0), (17, 43), (287, 5)]:
            assert list(oracle.extract_pattern(arr, _yhfk_in_tiler(), r)) == [42] * 8

    def test_extract_pattern_s266_single(self):
        # S:266 1-element pattern, fitting empty -> [array[origin + paving.r]]
        arr = np.arange(24, dtype=np.uint8).reshape(4, 6)
        t = oracle.make_tiler((4, 6), (1, 2), [[1, 0], [0, 1]], [[], []], [])
        assert list(oracle.extract_pattern(arr, t, (2, 3))) == [arr[3, 5]]

    def test_write_pattern_s274(self):
        # S:274 output tiler paving step 3, r=(0,1), p=[a,b,c] -> columns 3,4,5 of row 0
        arr = np.zeros((4, 12), np.uint8)
        t = oracle.make_tiler((4, 12), (0, 0), [[1, 0], [0, 3]], [[0], [1]], [3])
        oracle.write_pattern(arr, t, (0, 1), [7, 8, 9])
        want = np.zeros((4, 12), np.uint8)
        want[0, 3:6] = [7, 8, 9]
        assert (arr == want).all()

    def test_write_pattern_s276_count(self):
        arr = np.zeros((4, 12), np.uint8)
        t = oracle.make_tiler((4, 12), (0, 0), [[1, 0], [0, 3]], [[0], [1]], [3])
        oracle.write_pattern(arr, t, (2, 2), [1, 2, 3])
        assert int((arr != 0).sum()) == 3

    def test_coverage_s284_exact(self):
        # S:284 downscaler output tiler (132-wide rows, pattern [3], step 3, 44 reps) -> exact
        t = oracle.make_tiler((288, 132), (0, 0), [[1, 0], [0, 3]], [[0], [1]], [3])
        assert oracle.check_coverage(t, (288, 44))[0] == "exact"

    def test_coverage_s285_overlaps(self):
        # S:285 pattern [8], paving step 4, width 352 -> overlaps
        t = oracle.make_tiler((352,), (0,), [[4]], [[1]], [8])
        assert oracle.check_coverage(t, (88,))[0] == "overlaps"

    def test_coverage_s286_gaps(self):
        # S:286 pattern [3], paving step 4, width 12 -> gaps {3,7,11}
        t = oracle.make_tiler((12,), (0,), [[4]], [[1]], [3])
        kind, wit = oracle.check_coverage(t, (3,))
        assert kind == "gaps" and wit == [3, 7, 11]

    def test_yhfk_multiplicity_and_coverage(self):
        # P:110 "The yhfk task has a multiplicity equals to [288,44]"; S:647 tilers exact.
        W, H = 352, 288
        assert (H, W // 8) == (288, 44)
        assert oracle.check_coverage(_yhfk_in_tiler(), (288, 44))[0] == "exact"
        vin = oracle.make_tiler((288, 132), (0, 0), [[9, 0], [0, 1]], [[1], [0]], [9])
        vout = oracle.make_tiler((128, 132), (0, 0), [[4, 0], [0, 1]], [[1], [0]], [4])
        assert oracle.check_coverage(vin, (32, 132))[0] == "exact"
        assert oracle.check_coverage(vout, (32, 132))[0] == "exact"


def _random_tiler(rng):
    if rng.random() < 0.3:
        # a blocked partition (exact by construction), random origin, 2-D
        rep = [int(rng.integers(1, 5)), int(rng.integers(1, 5))]
        pattern = [int(rng.integers(1, 4)), int(rng.integers(1, 4))]
        shape = [rep[0] * pattern[0], rep[1] * pattern[1]]
        origin = [int(rng.integers(-20, 20)), int(rng.integers(-20, 20))]
        paving = [[pattern[0], 0], [0, pattern[1]]]
        fitting = [[1, 0], [0, 1]]
        return oracle.make_tiler(shape, origin, paving, fitting, pattern), shape, pattern, rep
    ndim = int(rng.integers(1, 3))
    nrep = int(rng.integers(1, 3))
    npat = int(rng.integers(0, 3))
    shape = [int(rng.integers(1, 24)) for _ in range(ndim)]
    origin = [int(rng.integers(-30, 30)) for _ in range(ndim)]
    paving = [[int(rng.integers(-5, 6)) for _ in range(nrep)] for _ in range(ndim)]
    fitting = [[int(rng.integers(-3, 4)) for _ in range(npat)] for _ in range(ndim)]
    pattern = [int(rng.integers(1, 5)) for _ in range(npat)]
    rep = [int(rng.integers(1, 6)) for _ in range(nrep)]
    return oracle.make_tiler(shape, origin, paving, fitting, pattern), shape, pattern, rep


def test_random_tilers_properties():
    """S:650 / S:289-292: bounds, linearity, coverage vs an independent
    set-based counter, write-then-extract identity when exact."""
    rng = np.random.default_rng(1234)
    n_exact = 0
    for _ in range(400):
        t, shape, pattern, rep = _random_tiler(rng)
        pats = list(np.ndindex(*pattern)) if pattern else [()]
        reps = list(np.ndindex(*rep))
        counter = {}
        for r in reps:
            for f in pats:
                idx = oracle.element_index(t, r, f)
                assert all(0 <= i < s for i, s in zip(idx, shape))
                counter[idx] = counter.get(idx, 0) + 1
                # linearity: e(r,f) - e(0,f) == paving.r (mod shape)
                base = oracle.element_index(t, tuple(0 for _ in r), f)
                for d in range(len(shape)):
                    pr = sum(t.paving[d][j] * r[j] for j in range(len(r)))
                    assert (idx[d] - base[d] - pr) % shape[d] == 0
        total = int(np.prod(shape))
        if any(c > 1 for c in counter.values()):
            want = "overlaps"
        elif len(counter) < total:
            want = "gaps"
        else:
            want = "exact"
        kind, _ = oracle.check_coverage(t, rep)
        assert kind == want
        if kind == "exact":
            n_exact += 1
            arr = np.zeros(shape, np.uint8)
            written = {}
            for r in reps:
                p = rng.integers(0, 256, size=len(pats)).astype(np.uint8)
                oracle.write_pattern(arr, t, r, p)
                written[r] = p
            for r in reps:
                assert (oracle.extract_pattern(arr, t, r) == written[r]).all()
    assert n_exact > 5


# ------------------------------------------------------------- filters --
def test_hfilter_spec_examples():
    assert list(oracle.hfilter_8to3([100] * 8)) == [100, 100, 100]
    assert oracle.hfilter_8to3([0, 6, 0, 0, 0, 0, 0, 0])[0] == 5
    assert list(oracle.hfilter_8to3([255] * 8)) == [255, 255, 255]


def test_vfilter_spec_examples():
    assert list(oracle.vfilter_9to4([100] * 9)) == [100] * 4
    assert oracle.vfilter_9to4([8, 0, 0, 0, 0, 0, 0, 0, 0])[0] == 3
    assert list(oracle.vfilter_9to4([0] * 9)) == [0] * 4


def _interp_taps(P, Q, D):
    """Taps re-derived from SPEC's sample positions s_k = (k+1/2)P/Q - 1/2
    (S:530): linear interpolation between floor(s_k) and +1, scaled
    by the fixed-point denominator D."""
    taps = []
    for k in range(Q):
        s = Fraction(2 * k + 1, 2) * Fraction(P, Q) - Fraction(1, 2)
        i0 = s.numerator // s.denominator
        fr = s - i0
        w0, w1 = (1 - fr) * D, fr * D
        assert w0.denominator == 1 and w1.denominator == 1
        row = [0] * P
        row[i0] += int(w0)
        if i0 + 1 < P:
            row[i0 + 1] += int(w1)
        taps.append(row)
    return taps


def test_taps_follow_from_interpolation_positions():
    h, v = oracle.default_stages()
    hd, vd = oracle.stage_to_dict(h), oracle.stage_to_dict(v)
    assert hd["weights"] == _interp_taps(8, 3, 6) and hd["divisor"] == 6 and hd["bias"] == 3
    assert vd["weights"] == _interp_taps(9, 4, 8) and vd["divisor"] == 8 and vd["bias"] == 4
    # and the literal SPEC functions have those taps (probe with impulses of 255)
    for i in range(8):
        e = [0] * 8
        e[i] = 48
        got = oracle.hfilter_8to3(e)
        for k in range(3):
            assert got[k] == (hd["weights"][k][i] * 48 + 3) // 6
    for i in range(9):
        e = [0] * 9
        e[i] = 64
        got = oracle.vfilter_9to4(e)
        for k in range(4):
            assert got[k] == (vd["weights"][k][i] * 64 + 4) // 8


def test_filters_exhaustive_round_half_up():
    """Every phase, all 65,536 (a, b) tap pairs: the oracle output equals
    round-half-up of the exact interpolated value, and
    lies in [min(a,b), max(a,b)]; constants are preserved."""
    htaps, vtaps = _interp_taps(8, 3, 6), _interp_taps(9, 4, 8)
    a = np.repeat(np.arange(256), 256)
    b = np.tile(np.arange(256), 256)
    for k, row in enumerate(htaps):
        i0 = next(i for i, w in enumerate(row) if w)
        pats = np.zeros((65536, 8), np.uint8)
        pats[:, i0], pats[:, i0 + 1] = a, b
        got = np.array([oracle.hfilter_8to3(p)[k] for p in pats])
        w0, w1 = row[i0], row[i0 + 1]
        exact = np.floor((w0 * a + w1 * b) / 6 + 0.5)  # exact in binary: denominators 6 -> check via ints too
        want = (2 * (w0 * a + w1 * b) + 6) // 12       # floor(x/6 + 1/2) in integers
        assert (got == want).all() and (got == exact).all()
        assert ((got >= np.minimum(a, b)) & (got <= np.maximum(a, b))).all()
    for k, row in enumerate(vtaps):
        i0 = next(i for i, w in enumerate(row) if w)
        pats = np.zeros((65536, 9), np.uint8)
        pats[:, i0], pats[:, i0 + 1] = a, b
        got = np.array([oracle.vfilter_9to4(p)[k] for p in pats])
        w0, w1 = row[i0], row[i0 + 1]
        want = (2 * (w0 * a + w1 * b) + 8) // 16
        assert (got == want).all()
        assert ((got >= np.minimum(a, b)) & (got <= np.maximum(a, b))).all()


def test_stage_table_equals_literal_functions():
    h, v = oracle.default_stages()
    rng = np.random.default_rng(5)
    for _ in range(2000):
        p8 = rng.integers(0, 256, 8).astype(np.uint8)
        p9 = rng.integers(0, 256, 9).astype(np.uint8)
        assert (oracle.stage_apply(h, p8) == oracle.hfilter_8to3(p8)).all()
        assert (oracle.stage_apply(v, p9) == oracle.vfilter_9to4(p9)).all()


# ------------------------------------------------------------- geometry --
def test_printed_geometry():
    # 352x288 -> 132x128; S:554 176x144 -> 66x64
    assert oracle.out_plane_dims(352, 288, 3, 1) == [(132, 128), (66, 64), (66, 64)]
    fr = synth.random_frames(0, 0, 1, 352, 288)
    out = oracle.execute_frames(fr, 352, 288)
    assert out.shape == (1, 132 * 128 + 2 * 66 * 64)
    y = oracle.execute_plane(fr[0, : 352 * 288].reshape(288, 352))
    assert y.shape == (128, 132)


def test_hd_geometry_closed_form():
    # W_out = 3W/8, H_out = 4H/9
    fin, fout = oracle.frame_bytes(1920, 1080, 3, 1)
    assert (fin, fout) == (3110400, 518400)
    assert oracle.frame_bytes(1920, 1080, 3, 0) == (6220800, 1036800)
    assert oracle.frame_bytes(3840, 2160, 3, 1) == (12441600, 2073600)
    assert oracle.frame_bytes(48, 27, 1, 0) == (1296, 216)


def test_non_divisible_is_error():
    # S:551 non-divisible shape -> error
    with pytest.raises(oracle.OracleError):
        oracle.direct_plane(np.zeros((27, 50), np.uint8))
    with pytest.raises(oracle.OracleError):
        oracle.execute_plane(np.zeros((28, 48), np.uint8))


# ------------------------------------------------------ goldens (tests/golden) --
@pytest.mark.parametrize("name", ["ramp_9x8.json", "checkerboard_9x8.json", "linear_16x18.json"])
def test_golden_planes(name):
    g = _golden(name)
    plane = _plane_from_rule(g["input_rule"])
    want = np.array(g["output"], np.uint8)
    assert (oracle.execute_plane(plane) == want).all()
    assert (oracle.direct_plane(plane) == want).all()


def test_golden_48x27_checksum():
    g = _golden("linear_48x27.json")
    plane = _plane_from_rule(g["input_rule"])
    out = oracle.execute_plane(plane)
    assert list(out.shape) == g["out_shape"]
    assert int(out.astype(np.int64).sum()) == g["byte_sum"]
    assert hashlib.sha256(out.tobytes()).hexdigest().startswith(g["sha256_prefix"])
    assert list(out[0]) == [g["row0_start"] + g["row0_step"] * i for i in range(18)]


def test_golden_rounding_order():
    g = _golden("rounding_order_counterexample.json")
    plane = np.zeros((9, 8), np.uint8)
    for r, c, val in g["tile_9x8_nonzero"]:
        plane[r, c] = val
    out = oracle.execute_plane(plane)
    assert out[0, 0] == g["expected_out00_two_stage"]
    # one rounding of the exact composition would give the other value
    exact = (3 * Fraction(1 * 0 + 5 * 3, 6) + 5 * Fraction(1 * 3 + 5 * 0, 6)) / 8
    assert int(exact + Fraction(1, 2)) == g["single_rounding_out00"] != out[0, 0]


# ----------------------------------------------------- O1 == O2 == O3 --
def test_o1_o2_o3_agree_cif_random():
    """100 random seeded CIF 4:2:0 frames, tiler executor == direct oracle,
    bit-exact; O3 closed form on every pixel of the first frames."""
    W, H = 352, 288
    frames = np.concatenate([synth.random_frames(s, 0, 1, W, H) for s in range(100)])
    o1 = oracle.execute_frames(frames, W, H)
    o2 = oracle.direct_frames(frames, W, H)
    assert (o1 == o2).all()
    for f in range(2):
        ins = oracle.split_planes(frames[f], W, H)
        outs = oracle.split_planes(o1[f], W, H, out=True)
        for pin, pout in zip(ins, outs):
            ho, wo = pout.shape
            o3 = np.array([[oracle.pixel(pin, R, Cc) for Cc in range(wo)] for R in range(ho)],
                          np.uint8)
            assert (o3 == pout).all()


def test_order_independence():
    # S:569 reverse repetition order gives identical output
    rng = np.random.default_rng(3)
    plane = rng.integers(0, 256, (36, 64)).astype(np.uint8)
    h, v = oracle.default_stages()
    assert (oracle.execute_plane(plane, h, v, 0) == oracle.execute_plane(plane, h, v, 1)).all()


def test_constants_and_fixed_points():
    # S:523, S:555, S:570 constants preserved; 0 and 255 are fixed points
    for c in (0, 1, 100, 254, 255):
        fr = synth.constant_frames(c, 1, 176, 144)
        assert (oracle.execute_frames(fr, 176, 144) == c).all()


def test_output_within_tap_range():
    # S:571 each output within [min, max] of its input pixels' footprint
    rng = np.random.default_rng(9)
    plane = rng.integers(0, 256, (18, 16)).astype(np.uint8)
    out = oracle.execute_plane(plane)
    for R in range(out.shape[0]):
        for Cc in range(out.shape[1]):
            g, p = R // 4, Cc // 3
            foot = plane[9 * g: 9 * g + 9, 8 * p: 8 * p + 8]
            assert foot.min() <= out[R, Cc] <= foot.max()


def test_dead_taps():
    """Tap liveness: an impulse of 255 at (row, col) of a 9x8
    tile changes the output iff row != 4 and col not in {2, 5}."""
    for r in range(9):
        for c in range(8):
            plane = np.zeros((9, 8), np.uint8)
            plane[r, c] = 255
            live = bool(oracle.execute_plane(plane).any())
            assert live == (r != 4 and c not in (2, 5)), (r, c)
    plane = np.zeros((9, 8), np.uint8)
    plane[0, 0] = 8
    assert not oracle.execute_plane(plane).any()
    plane[0, 0] = 9
    assert oracle.execute_plane(plane)[0, 0] == 1


def _brute_force_exact(plane):
    """Independent exact-rational model: mid = round-half-up of the linear
    interpolation at s_k, u8; out = same on mid columns."""
    H, W = plane.shape

    def interp(vals, s):
        i0 = s.numerator // s.denominator
        fr = s - i0
        x = (1 - fr) * int(vals[i0]) + fr * (int(vals[i0 + 1]) if fr else 0)
        return int(x + Fraction(1, 2))

    mid = np.zeros((H, W // 8 * 3), np.int64)
    for y in range(H):
        for p in range(W // 8):
            pk = plane[y, 8 * p: 8 * p + 8]
            for k in range(3):
                mid[y, 3 * p + k] = interp(pk, Fraction(2 * k + 1, 2) * Fraction(8, 3) - Fraction(1, 2))
    out = np.zeros((H // 9 * 4, W // 8 * 3), np.uint8)
    for c in range(mid.shape[1]):
        for g in range(H // 9):
            pk = mid[9 * g: 9 * g + 9, c]
            for k in range(4):
                out[4 * g + k, c] = interp(pk, Fraction(2 * k + 1, 2) * Fraction(9, 4) - Fraction(1, 2))
    return out


def test_brute_force_exact_rational_tiny():
    plane = synth.random_frames(7, 0, 1, 48, 27, 1)[0].reshape(27, 48)
    assert (oracle.execute_plane(plane) == _brute_force_exact(plane)).all()


# ------------------------------------------------ general stages (halo) --
def _halo_stages():
    # P > S on both axes: halos of 5 columns and 5 rows
    h = oracle.make_stage(13, 8, 0, [[1, 2, 3, 0, 0, 0, 0, 0, 0, 0, 0, 1, 1],
                                     [0, 0, 0, 2, 2, 2, 0, 0, 0, 0, 0, 0, 2],
                                     [0, 0, 0, 0, 0, 0, 4, 4, 1, 1, 0, 0, 0]], 8, 4)
    v = oracle.make_stage(14, 9, 0, [[2, 2, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 4],
                                     [0, 0, 4, 4, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0],
                                     [0, 0, 0, 0, 0, 3, 3, 0, 0, 0, 0, 2, 0, 0],
                                     [0, 0, 0, 0, 0, 0, 0, 5, 3, 0, 0, 0, 0, 0]], 8, 4)
    return h, v


def test_origin_is_a_toroidal_roll():
    """S:251 modulo rule: origin (o_h, o_v) equals the origin-0 result on the
    input rolled by (-o_v, -o_h)."""
    rng = np.random.default_rng(11)
    plane = rng.integers(0, 256, (36, 48)).astype(np.uint8)
    h, v = _halo_stages()
    base = oracle.execute_plane(plane, h, v)
    for oh, ov in [(3, 0), (0, 5), (-7, 2), (13, 31)]:
        d_h, d_v = oracle.stage_to_dict(h), oracle.stage_to_dict(v)
        d_h["origin"], d_v["origin"] = oh, ov
        h2, v2 = oracle.stage_from_dict(d_h), oracle.stage_from_dict(d_v)
        got = oracle.execute_plane(plane, h2, v2)
        want = oracle.execute_plane(np.roll(plane, (-ov, -oh), axis=(0, 1)), h, v)
        assert (got == want).all()
    assert base.shape == (16, 18)


def _stage_matrix(d, n_in):
    """Linear map of one stage with divisor 1, bias 0 as a dense matrix
    (rows = outputs over all repetitions, cols = input positions mod n)."""
    reps = n_in // d["paving"]
    Q = len(d["weights"])
    A = np.zeros((Q * reps, n_in), np.int64)
    for r in range(reps):
        for k in range(Q):
            for i, w in enumerate(d["weights"][k]):
                A[Q * r + k, (d["origin"] + d["paving"] * r + i) % n_in] += w
    return A


def test_halo_stages_equal_matrix_form():
    """With divisor 1 and bias 0 and no clamping, the two tasks are linear
    maps, so Out = A_v . In . A_h^T (a matmul, library routine)."""
    h, v = _halo_stages()
    dh, dv = oracle.stage_to_dict(h), oracle.stage_to_dict(v)
    for d in (dh, dv):
        d["divisor"], d["bias"] = 1, 0
    dh["origin"], dv["origin"] = 5, -4
    # keep all sums <= 255: input values tiny, weights sum small
    dh["weights"] = [[1 if w else 0 for w in row] for row in dh["weights"]]
    dv["weights"] = [[1 if w else 0 for w in row] for row in dv["weights"]]
    rng = np.random.default_rng(2)
    plane = rng.integers(0, 6, (27, 40)).astype(np.uint8)
    got = oracle.execute_plane(plane, oracle.stage_from_dict(dh), oracle.stage_from_dict(dv))
    Ah, Av = _stage_matrix(dh, 40), _stage_matrix(dv, 27)
    want = Av @ plane.astype(np.int64) @ Ah.T
    assert want.max() <= 255
    assert (got == want).all()


def test_negative_weights_truncate_and_clamp():
    # truncating division toward zero then clamp 0..255 ("clamped")
    s = oracle.make_stage(2, 2, 0, [[-1, 1], [3, 0]], 2, 0)
    assert list(oracle.stage_apply(s, [5, 2])) == [0, 7]      # (-3)/2 -> -1 -> 0 ; 15/2 -> 7
    assert list(oracle.stage_apply(s, [0, 255])) == [127, 0]
    s2 = oracle.make_stage(1, 1, 0, [[4]], 1, 0)
    assert list(oracle.stage_apply(s2, [200])) == [255]


def test_mid_array_is_the_h_task_output():
    """The exposed intermediate equals SPEC's literal hfilter_8to3 on
    every consecutive 8-pixel packet of every row (O2's first loop)."""
    rng = np.random.default_rng(21)
    plane = rng.integers(0, 256, (18, 64)).astype(np.uint8)
    mid, out = oracle.execute_plane_mid(plane)
    want = np.array([[v for p in range(8) for v in oracle.hfilter_8to3(row[8 * p: 8 * p + 8])]
                     for row in plane], np.uint8)
    assert (mid == want).all()
    assert (out == oracle.execute_plane(plane)).all()


# ------------------------------------------------- general tasks (row f4) --
def _identity_body(n):
    return oracle.make_stage(n, n, 0, [[1 if i == k else 0 for i in range(n)] for k in range(n)], 1, 0)


def test_run_task_identity_model():
    # S:525 "identity model (pass-through body, identity tilers) -> output equals input"
    rng = np.random.default_rng(4)
    a = rng.integers(0, 256, (6, 10)).astype(np.uint8)
    t = oracle.make_tiler((6, 10), (0, 0), [[1, 0], [0, 1]], [[], []], [])
    out = oracle.run_task(a, t, (6, 10), t, (6, 10), _identity_body(1))
    assert (out == a).all()


def test_run_task_transpose_and_blocks_match_numpy():
    """Tilers that realise np.transpose and a 2x3-block regrouping (library
    routines), with a 2x3 pattern and a pass-through body."""
    rng = np.random.default_rng(5)
    a = rng.integers(0, 256, (4, 6)).astype(np.uint8)
    # transpose: out[c][r] = in[r][c]; rep (r, c); in paving identity, out paving swapped
    tin = oracle.make_tiler((4, 6), (0, 0), [[1, 0], [0, 1]], [[], []], [])
    tout = oracle.make_tiler((6, 4), (0, 0), [[0, 1], [1, 0]], [[], []], [])
    assert (oracle.run_task(a, tin, (6, 4), tout, (4, 6), _identity_body(1)) == a.T).all()
    # blocks: rep (bi, bj) over (2, 2); pattern 2x3 from in; written as row bi*2+bj of a (4, 6) array
    tin = oracle.make_tiler((4, 6), (0, 0), [[2, 0], [0, 3]], [[1, 0], [0, 1]], [2, 3])
    tout = oracle.make_tiler((4, 6), (0, 0), [[2, 1], [0, 0]], [[0], [1]], [6])
    got = oracle.run_task(a, tin, (4, 6), tout, (2, 2), _identity_body(6))
    want = a.reshape(2, 2, 2, 3).transpose(0, 2, 1, 3).reshape(4, 6)
    assert (got == want).all()


def test_run_task_reproduces_the_downscaler_h_task():
    """The downscaler's yhfk task through the general executor equals
    the Mid array of O1 and SPEC's literal hfilter_8to3."""
    plane = synth.random_frames(2, 0, 1, 352, 288, 1)[0].reshape(288, 352)
    h, v = oracle.default_stages()
    tin = oracle.make_tiler((288, 352), (0, 0), [[1, 0], [0, 8]], [[0], [1]], [8])
    tout = oracle.make_tiler((288, 132), (0, 0), [[1, 0], [0, 3]], [[0], [1]], [3])
    mid = oracle.run_task(plane, tin, (288, 132), tout, (288, 44), h)
    assert (mid == oracle.execute_plane_mid(plane)[0]).all()
    assert (mid[5, 6:9] == oracle.hfilter_8to3(plane[5, 16:24])).all()
