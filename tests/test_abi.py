"""Boundary tests that need no GPU: libds.so loads, exports every symbol
include/ds.h declares, and its host-only logic (validation, geometry,
K-N1 band planning) is right.  Compute calls are in test_parity_gpu.py."""
import os
import re
import subprocess

import pytest

import paper_1103_4881_b200 as ds
from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "ds.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"DS_API\s+[\w\s\*]+?\b(ds_\w+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for must in ("ds_create", "ds_run", "ds_destroy"):
        assert must in names


def test_library_exports_every_declared_symbol():
    L = ds.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    out = subprocess.check_output(["nm", "-D", "--defined-only", ds.lib_path()], text=True)
    exported = set(re.findall(r"\bT (ds_\w+)", out))
    assert set(declared_functions()) <= exported
    # the binding wraps exactly the header's calls
    assert sorted(n for n, _, _ in ds.SIGNATURES) == declared_functions()


def test_library_is_sm100a():
    out = subprocess.check_output(["cuobjdump", "--list-elf", ds.lib_path()], text=True)
    assert "sm_100a" in out


def test_strerror_and_no_error_yet():
    for code in (0, -1, -2, -3, -4, -5, 7):
        assert isinstance(ds.ds_strerror(code), str) and ds.ds_strerror(code)


def test_default_spec_is_spec_taps():
    s = ds.ds_default_spec()
    h, v = ds.stage_to_dict(s.h), ds.stage_to_dict(s.v)
    # compared with the literal values printed in SPEC
    assert h == dict(pattern=8, paving=8, origin=0, divisor=6, bias=3,
                     weights=[[1, 5, 0, 0, 0, 0, 0, 0], [0, 0, 0, 3, 3, 0, 0, 0],
                              [0, 0, 0, 0, 0, 0, 5, 1]])
    assert v == dict(pattern=9, paving=9, origin=0, divisor=8, bias=4,
                     weights=[[3, 5, 0, 0, 0, 0, 0, 0, 0], [0, 0, 1, 7, 0, 0, 0, 0, 0],
                              [0, 0, 0, 0, 0, 7, 1, 0, 0], [0, 0, 0, 0, 0, 0, 0, 5, 3]])
    assert s.chroma == ds.DS_CHROMA_420


@pytest.mark.parametrize("W,H,ch,chroma,fin,fout", [
    (1920, 1080, 3, 1, 3110400, 518400),
    (1920, 1080, 3, 0, 6220800, 1036800),
    (3840, 2160, 3, 1, 12441600, 2073600),
    (352, 288, 3, 1, 152064, 25344),
    (48, 27, 1, 1, 1296, 216),
])
def test_plan_geometry(W, H, ch, chroma, fin, fout):
    spec = ds.ds_default_spec()
    spec.chroma = chroma
    p = ds.ds_plan(W, H, ch, spec)
    assert (p.in_frame_bytes, p.out_frame_bytes) == (fin, fout)
    for q in range(ch):
        assert p.out_w[q] == 3 * p.in_w[q] // 8 and p.out_h[q] == 4 * p.in_h[q] // 9


def test_plan_cif_matches_paper():
    p = ds.ds_plan(352, 288, 3)
    assert (p.out_w[0], p.out_h[0]) == (132, 128)
    assert (p.out_w[1], p.out_h[1]) == (66, 64)
    assert p.fused_eligible == 1


def test_plan_hd_bands_equal_bytes():
    p = ds.ds_plan(1920, 1080, 3)
    assert p.fused_eligible == 1
    # 32 KiB band target: luma 2 groups, chroma 4 groups -> 30,720 B staged each
    assert list(p.band_groups) == [2, 4, 4]
    assert p.units_per_frame == 60 + 15 + 15
    assert p.unit_in_bytes_max == 8 * 2 * 1920
    assert p.unit_out_bytes_max == 4 * 2 * 720


def test_plan_tiny_is_fused_eligible_but_unaligned_out():
    p = ds.ds_plan(48, 27, 1)
    assert p.fused_eligible == 1 and p.out_frame_bytes == 216


@pytest.mark.parametrize("W,H,ch", [(50, 27, 1), (48, 28, 1), (352, 289, 3), (1920, 1081, 3),
                                    (0, 27, 1), (48, -9, 1), (360, 288, 3)])
def test_plan_rejects_non_divisible(W, H, ch):
    # S:551 non-divisible shape -> error; 4:2:0 needs W % 16 == 0, H % 18 == 0
    with pytest.raises(ds.DSError) as e:
        ds.ds_plan(W, H, ch)
    assert e.value.code == ds.DS_ESHAPE


def test_plan_rejects_bad_channels_and_specs():
    with pytest.raises(ds.DSError) as e:
        ds.ds_plan(48, 27, 2)
    assert e.value.code == ds.DS_EUNSUPPORTED
    for bad in (dict(pattern=17), dict(divisor=0), dict(outputs=9)):
        s = ds.ds_default_spec()
        for k, v in bad.items():
            setattr(s.h, k, v)
        with pytest.raises(ds.DSError) as e:
            ds.ds_plan(48, 27, 1, s)
        assert e.value.code == ds.DS_EUNSUPPORTED
    s = ds.ds_default_spec()
    s.h.weight[0][12] = 1          # tap beyond the pattern
    with pytest.raises(ds.DSError):
        ds.ds_plan(48, 27, 1, s)


def test_plan_generic_spec_not_fused():
    h = dict(pattern=13, paving=8, origin=2, weights=[[1, 2, 3], [0, 0, 0, 4, 4], [1] * 13],
             divisor=8, bias=4)
    p = ds.ds_plan(48, 27, 1, ds.make_spec(h=h))
    assert p.fused_eligible == 0 and p.out_w[0] == 18
    # K-N1g takes it: bands of k V repetitions stage Sv (k-1) + Pv rows
    assert p.fused_general_eligible == 1
    k = p.general_band_reps[0]
    assert 3 % k == 0 and p.general_units_per_frame == 3 // k
    assert p.general_stage_bytes_max == (9 * (k - 1) + 9) * (48 + 32)   # row pitch: 48 + 32-byte wrap pad


def test_plan_narrow_rows():
    # W % 16 == 8 planes (PAL SD / QCIF 4:2:0 chroma: 360 / 88 B rows) stay on K-N1:
    # whole bands are bulk-copied from a 16-aligned superset (needs 16-aligned frames)
    p = ds.ds_plan(720, 576, 3)
    assert p.fused_eligible == 1 and list(p.band_groups) == [4, 8, 8]
    assert p.unit_in_bytes_max == 9 * 8 * 360 + 16          # 9 rows per group + alignment slack
    assert ds.ds_plan(176, 144, 3).fused_eligible == 1        # QCIF
    # frames that are not 16-byte multiples: K-N1g stages the rows itself
    p = ds.ds_plan(40, 45, 1)                                 # 1,800-byte frames
    assert p.fused_eligible == 0 and p.fused_general_eligible == 1


def test_create_validates_before_touching_cuda():
    with pytest.raises(ds.DSError) as e:
        ds.ds_create(50, 27, 1)
    assert e.value.code == ds.DS_ESHAPE
    assert ds.ds_last_error() == ds.DS_ESHAPE


def test_null_handle_calls():
    L = ds.lib()
    assert L.ds_run(None, None, 0, None, None) == ds.DS_EINVAL
    assert L.ds_in_frame_bytes(None) == -1
    assert L.ds_set_kernel(None, 0) == ds.DS_EINVAL
    assert L.ds_enable_peer(None, 0) == ds.DS_EINVAL
    L.ds_destroy(None)                                    # NULL-safe
    assert L.ds_generate(None, 0, 1, 0, None) == ds.DS_OK   # n = 0 no-op
    assert L.ds_generate(None, 16, 1, 0, None) == ds.DS_EINVAL


def test_schedule_byte_model_matches_spec_and_paper():
    """S:375 / S:385: naive 12 transfers per frame, optimised 6; S:365 byte
    sizes.  The byte reductions 27.3% (H2D) and 69.2% (D2H) are the
    deterministic counterpart of P:148's "about 30% and 70% faster transfer
    times in host to device and device to host"."""
    naive = ds.ds_schedule_plan(352, 288, 3, ds.DS_SCHED_NAIVE)
    opt = ds.ds_schedule_plan(352, 288, 3, ds.DS_SCHED_OPTIMIZED)
    assert naive["h2d_count"] + naive["d2h_count"] == 12 and naive["launches"] == 6
    assert opt["h2d_count"] == 3 and opt["d2h_count"] == 3 and opt["launches"] == 6
    # Y input array 352x288 = 101,376 B; Mid = 288x132 + 2 * 144x66
    assert (naive["h2d_bytes"], naive["d2h_bytes"]) == (152064 + 57024, 57024 + 25344)
    assert (opt["h2d_bytes"], opt["d2h_bytes"]) == (152064, 25344)
    h2d_cut = 1 - opt["h2d_bytes"] / naive["h2d_bytes"]
    d2h_cut = 1 - opt["d2h_bytes"] / naive["d2h_bytes"]
    assert abs(h2d_cut - 0.273) < 0.001 and abs(d2h_cut - 0.692) < 0.001
    assert abs(h2d_cut - 0.30) < 0.05 and abs(d2h_cut - 0.70) < 0.05     # P:148 "about"
    fused = ds.ds_schedule_plan(352, 288, 3, ds.DS_SCHED_FUSED)
    assert fused["h2d_count"] == fused["d2h_count"] == fused["launches"] == 1
    # the reductions depend only on the 8->3 / 9->4 geometry, not on the taps
    hd = ds.ds_schedule_plan(1920, 1080, 3, ds.DS_SCHED_NAIVE)
    assert 1 - 3110400 / hd["h2d_bytes"] == pytest.approx(h2d_cut, abs=1e-3)
    with pytest.raises(ds.DSError):
        ds.ds_schedule_plan(352, 288, 3, 9)


def test_plan_wide_planes_and_smem_limit():
    # 7680-wide (8K) luma: one group stages 61,440 B; a 2-deep ring + 3 output
    # slots fits 227 KB -> K-N1 with 1 group per band
    p = ds.ds_plan(7680, 4320, 1)
    assert p.fused_eligible == 1 and p.band_groups[0] == 1
    # 11520-wide: 92,160 B per group -> 2 x 92,160 + 3 x 17,280 > 227 KB -> not K-N1;
    # K-N1g takes it in column strips (1440 H repetitions -> strips of a multiple of 16)
    p = ds.ds_plan(11520, 2160, 1)
    assert p.fused_eligible == 0 and p.fused_general_eligible == 1
    assert p.general_strips[0] > 1 and p.general_stage_bytes_max <= 40 * 1024


def test_plan_general_column_strips():
    """K-N1g column strips: planes whose k = 1 band exceeds the
    stage target are split; narrow planes keep whole rows; the stage knob
    re-plans (ds_set_general_stage_bytes, exercised in test_parity_gpu)."""
    h = dict(pattern=13, paving=8, origin=-2, weights=[[1, 3, 5, 3, 1]], divisor=13, bias=6)
    v = dict(pattern=14, paving=9, origin=-2, weights=[[1, 2, 4, 2, 1]], divisor=10, bias=5)
    spec = ds.make_spec(h=h, v=v)
    hd = ds.ds_plan(1920, 1080, 3, spec)
    assert hd.fused_general_eligible == 1 and list(hd.general_strips) == [1, 1, 1]
    p8k = ds.ds_plan(7680, 4320, 3, spec)                  # was K-N2-only before strips
    assert p8k.fused_general_eligible == 1
    assert p8k.general_strips[0] > 1 and p8k.general_stage_bytes_max <= 28 * 1024
    p4k = ds.ds_plan(3840, 2160, 3, spec)
    assert p4k.general_strips[0] > 1 and p4k.general_stage_bytes_max <= 28 * 1024
    assert ds.ds_plan(352, 288, 3, spec).general_strips[0] == 1


def test_plan_invariants_random():
    """Host planners (K-N1 bands, K-N1g bands / strips) on random valid
    geometries and specs: exact band tiling of every plane, unit counts,
    staging within shared memory, strips only for wide planes."""
    import numpy as np
    rng = np.random.default_rng(7)
    checked = 0
    for _ in range(300):
        ch = int(rng.choice([1, 3]))
        chroma = int(rng.integers(0, 2))
        h = None if rng.random() < 0.3 else dict(
            pattern=int(rng.integers(1, 17)), paving=int(rng.choice([2, 4, 8, 16])), origin=int(rng.integers(-9, 9)),
            weights=[[1, 2, 1]], divisor=4, bias=2)
        v = None if rng.random() < 0.3 else dict(
            pattern=int(rng.integers(1, 17)), paving=int(rng.choice([3, 6, 9, 12])), origin=int(rng.integers(-9, 9)),
            weights=[[1, 2, 1]], divisor=4, bias=2)
        sh = 8 if h is None else h["paving"]
        sv = 9 if v is None else v["paving"]
        mw = sh * (2 if ch == 3 and chroma else 1)
        mh = sv * (2 if ch == 3 and chroma else 1)
        W = mw * int(rng.integers(1, max(2, 8000 // mw)))
        H = mh * int(rng.integers(1, max(2, 2200 // mh)))
        spec = ds.make_spec(h=h, v=v, chroma=chroma)
        try:
            p = ds.ds_plan(W, H, ch, spec)
        except ds.DSError:
            continue
        n = p.n_planes
        if p.fused_eligible:
            units = 0
            for q in range(n):
                k = p.band_groups[q]
                assert k >= 1 and (p.in_h[q] // 9) % k == 0
                units += p.in_h[q] // (9 * k)
            assert units == p.units_per_frame
            assert p.unit_in_bytes_max <= 227 * 1024
        if p.fused_general_eligible:
            units = 0
            for q in range(n):
                k, s = p.general_band_reps[q], p.general_strips[q]
                G = p.in_h[q] // sv
                assert k >= 1 and G % k == 0 and s >= 1
                units += s * (G // k)
                if s > 1:                                   # strips only when a whole-row band is too big
                    pv = 9 if v is None else v["pattern"]
                    target = 28 * 1024 if pv > sv else 40 * 1024
                    assert pv * ((p.in_w[q] + 15) // 16 * 16 + 32) > target
            assert units == p.general_units_per_frame
            assert p.general_stage_bytes_max <= 227 * 1024
        checked += 1
    assert checked >= 150
