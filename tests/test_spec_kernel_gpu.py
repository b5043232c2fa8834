"""K-N1s (ds_spec.cuh): the K-N1g fused band kernel with the filter spec
compiled in.  Byte-for-byte against the CPU oracle (O1 with the spec's
stages, halos wrap toroidally) and against the runtime-tap
K-N1g on the same inputs: the bench's halo spec and SPEC's downscaler on the
paper's and BASELINE's geometries, column strips, ragged chunk tails, every
unit processed once, every output byte written, rows and input pointers
aligned to 8 or 4 bytes only or not at all (funnel-shifted words), and the
fallbacks (planes without a common window phase, or a run-time compiled spec
from a less aligned pointer, run the runtime-tap kernel)."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
ds = pytest.importorskip("paper_1103_4881_b200")

pytestmark = pytest.mark.gpu

GENERAL = ds.DS_KERNEL_FUSED_GENERAL

# bench.py HALO_SPEC (kept literally: the built-in K-N1s instance matches it)
HALO = (
    dict(pattern=13, paving=8, origin=-2, weights=[[1, 3, 5, 3, 1], [0, 0, 0, 1, 3, 5, 3, 1],
                                                    [0, 0, 0, 0, 0, 0, 1, 3, 5, 3, 1]],
         divisor=13, bias=6),
    dict(pattern=14, paving=9, origin=-2, weights=[[1, 2, 4, 2, 1], [0, 0, 1, 2, 4, 2, 1],
                                                    [0, 0, 0, 0, 0, 1, 2, 4, 2, 1],
                                                    [0, 0, 0, 0, 0, 0, 0, 0, 1, 2, 4, 2, 1]],
         divisor=10, bias=5),
)


def _stage(d):
    return oracle.make_stage(d["pattern"], d["paving"], d["origin"], d["weights"], d["divisor"], d["bias"])


def _want(fr, W, H, ch, chroma, spec):
    if spec is None:
        return oracle.execute_frames(fr, W, H, ch, chroma)
    return oracle.execute_frames(fr, W, H, ch, chroma, _stage(spec[0]), _stage(spec[1]))


def _handle(W, H, ch, chroma, spec):
    s = None if spec is None else ds.make_spec(h=spec[0], v=spec[1], chroma=chroma)
    d = ds.Downscaler(W, H, ch, chroma=chroma, spec=s)
    d.set_kernel(GENERAL)
    return d


def _same(got, want, what):
    if not np.array_equal(got, want):
        bad = np.argwhere(got != want)
        raise AssertionError(f"{what}: {len(bad)} bytes differ, first at {bad[:4].tolist()}")


@pytest.mark.parametrize("spec", ["halo", "spec"])
@pytest.mark.parametrize("W,H,ch,chroma,n", [(1920, 1080, 3, 1, 5), (1920, 1080, 3, 0, 3), (352, 288, 3, 1, 7),
                                             (3840, 2160, 3, 1, 2), (128, 72, 1, 1, 9), (704, 576, 3, 1, 3),
                                             (1024, 144, 3, 0, 4)])
def test_compiled_spec_matches_oracle_and_runtime_taps(spec, W, H, ch, chroma, n):
    sp = HALO if spec == "halo" else None
    d = _handle(W, H, ch, chroma, sp)
    d.set_general_variant(ds.DS_GENERAL_COMPILED)
    fr = synth.random_frames(77, 3, n, W, H, ch, chroma)
    x = torch.from_numpy(fr).cuda()
    y = d(x)
    torch.cuda.synchronize()
    assert d.last_kernel() == GENERAL and d.last_variant() == 2
    want = _want(fr, W, H, ch, chroma, sp)
    _same(y.cpu().numpy(), want, f"K-N1s {spec} {W}x{H}")
    d.set_general_variant(ds.DS_GENERAL_RUNTIME)
    y2 = d(x)
    torch.cuda.synchronize()
    assert d.last_variant() == 1
    _same(y2.cpu().numpy(), want, f"K-N1g runtime taps {spec} {W}x{H}")


def test_compiled_spec_plans_strips_and_ragged_chunks():
    """4K luma needs column strips; 720-wide CIF-like planes (W/8 = 90 H
    repetitions, not a multiple of 4) end rows in partial chunks; both
    exact."""
    for W, H in ((3840, 2160), (720, 288), (208, 144)):
        d = _handle(W, H, 3, 0, HALO)
        info = d.launch_info(2, GENERAL)
        assert info["variant"] == 2
        fr = synth.random_frames(5, 0, 2, W, H, 3, 0)
        y = d(torch.from_numpy(fr).cuda())
        torch.cuda.synchronize()
        assert d.last_variant() == 2
        _same(y.cpu().numpy(), _want(fr, W, H, 3, 0, HALO), f"{W}x{H}")


def test_auto_picks_compiled_variant_and_falls_back():
    W, H, n = 352, 288, 4
    d = _handle(W, H, 3, 1, HALO)
    fr = synth.random_frames(8, 0, n, W, H)
    want = _want(fr, W, H, 3, 1, HALO)
    x = torch.from_numpy(fr).cuda()
    y = d(x)
    torch.cuda.synchronize()
    assert d.last_variant() == 2
    _same(y.cpu().numpy(), want, "auto")
    # output rows at every alignment: K-N1s stores words, half-words or bytes by alignment
    for off in (1, 2, 3):
        buf = torch.zeros(n * d.out_frame_bytes + 8, dtype=torch.uint8, device="cuda")
        yo = buf[off:off + n * d.out_frame_bytes].view(n, -1)
        d(x, yo)
        torch.cuda.synchronize()
        assert d.last_variant() == 2
        _same(yo.cpu().numpy(), want, f"output offset {off}")
    # input pointer 4- or 8-byte aligned: K-N1s with 4- / 8-byte loads; not
    # 4-byte aligned: K-N1s funnel-shifts each window word out of two aligned words
    xb = torch.zeros(n * d.in_frame_bytes + 16, dtype=torch.uint8, device="cuda")
    for off, variant in ((4, 2), (8, 2), (12, 2), (1, 2), (2, 2), (7, 2)):
        xi = xb[off:off + n * d.in_frame_bytes]
        xi.copy_(x.view(-1))
        y3 = d(xi.view(n, -1))
        torch.cuda.synchronize()
        assert d.last_variant() == variant, off
        _same(y3.cpu().numpy(), want, f"input offset {off}")


def test_compiled_variant_rejected_where_it_cannot_run():
    # 48-byte chroma rows (96x72 4:2:0) are shorter than K-N1s's 64-byte minimum
    d = _handle(96, 72, 3, 1, HALO)
    with pytest.raises(ds.DSError):
        d.set_general_variant(ds.DS_GENERAL_COMPILED)
    fr = synth.random_frames(2, 0, 2, 96, 72)
    y = d(torch.from_numpy(fr).cuda())
    torch.cuda.synchronize()
    assert d.last_variant() == 1
    _same(y.cpu().numpy(), _want(fr, 96, 72, 3, 1, HALO), "96x72 halo runtime taps")


@pytest.mark.parametrize("spec", ["halo", "spec"])
@pytest.mark.parametrize("W,H,ch,chroma,n", [(176, 144, 3, 1, 6), (352, 288, 3, 1, 4), (64, 90, 1, 1, 5),
                                             (88, 72, 1, 1, 7), (200, 36, 1, 1, 4)])
def test_compiled_spec_several_rows_per_warp(spec, W, H, ch, chroma, n):
    """Rows of at most 16 chunks (64 H repetitions) are taken 2, 4 or 8 to a
    warp (QCIF chroma: 3 chunks, 8 rows per warp); a warp's last pass may run
    past the band's rows on its later row lanes.  Exact, every unit once."""
    sp = HALO if spec == "halo" else None
    d = _handle(W, H, ch, chroma, sp)
    d.set_general_variant(ds.DS_GENERAL_COMPILED)
    fr = synth.random_frames(41, 5, n, W, H, ch, chroma)
    want = _want(fr, W, H, ch, chroma, sp)
    x = torch.from_numpy(fr).cuda()
    for rb in (0, 1, 3):
        d.set_run_bands(rb)
        y = d(x)
        torch.cuda.synchronize()
        assert d.last_variant() == 2
        _same(y.cpu().numpy(), want, f"K-N1s {spec} {W}x{H} run_bands {rb}")


@pytest.mark.parametrize("spec", ["halo", "spec"])
@pytest.mark.parametrize("W,H,ch,chroma,n", [(720, 576, 3, 1, 4), (720, 288, 3, 1, 3), (360, 288, 1, 1, 5),
                                             (1400, 198, 3, 0, 2)])
def test_compiled_spec_rows_8_byte_aligned(spec, W, H, ch, chroma, n):
    """Rows that are not 16-byte multiples (PAL / NTSC SD chroma: 360 B; a
    360-wide luma plane; 1400 = 87.5 blocks): K-N1s with 8-byte loads, the
    windows crossing the row end computed word by word."""
    sp = HALO if spec == "halo" else None
    d = _handle(W, H, ch, chroma, sp)
    d.set_general_variant(ds.DS_GENERAL_COMPILED)
    fr = synth.random_frames(31, 2, n, W, H, ch, chroma)
    x = torch.from_numpy(fr).cuda()
    y = d(x)
    torch.cuda.synchronize()
    assert d.last_variant() == 2
    want = _want(fr, W, H, ch, chroma, sp)
    _same(y.cpu().numpy(), want, f"K-N1s {spec} {W}x{H}")
    # and from a 4-byte aligned pointer (4-byte loads) or none (funnel shifts)
    xb = torch.zeros(x.numel() + 16, dtype=torch.uint8, device="cuda")
    for off in (4, 3):
        xi = xb[off:off + x.numel()]
        xi.copy_(x.view(-1))
        y2 = d(xi.view(n, -1))
        torch.cuda.synchronize()
        assert d.last_variant() == 2
        _same(y2.cpu().numpy(), want, f"K-N1s {spec} {W}x{H} input offset {off}")


@pytest.mark.parametrize("W,H", [(88, 72), (104, 72), (88, 36), (136, 90)])
def test_runtime_taps_band_taller_than_plane(W, H):
    """Planes whose rows the TMA cannot copy (W % 16 == 8) are staged by the
    producer warp; when one band plus its V halo has more rows than the plane
    (QCIF chroma: 77 > 72 rows), the halo rows wrap past the plane bottom
    more than once.  Runtime taps and compiled spec, both exact."""
    fr = synth.random_frames(12, 0, 3, W, H, 1, 1)
    want = _want(fr, W, H, 1, 1, HALO)
    d = _handle(W, H, 1, 1, HALO)
    x = torch.from_numpy(fr).cuda()
    for variant in (ds.DS_GENERAL_RUNTIME, ds.DS_GENERAL_AUTO):
        d.set_general_variant(variant)
        y = d(x)
        torch.cuda.synchronize()
        _same(y.cpu().numpy(), want, f"{W}x{H} variant {d.last_variant()}")


def test_compiled_spec_planes_with_different_window_phases_fall_back():
    """An H origin of 200 reduces to 200 on 720-byte luma rows (phase 8) and
    to -160 on 360-byte chroma rows (phase 0): one compiled instance cannot
    serve both planes, so the runtime-tap kernel runs; results exact."""
    sp = (dict(HALO[0], origin=200), HALO[1])
    d = _handle(720, 576, 3, 1, sp)
    with pytest.raises(ds.DSError):
        d.set_general_variant(ds.DS_GENERAL_COMPILED)
    fr = synth.random_frames(4, 0, 2, 720, 576)
    y = d(torch.from_numpy(fr).cuda())
    torch.cuda.synchronize()
    assert d.last_variant() == 1
    _same(y.cpu().numpy(), _want(fr, 720, 576, 3, 1, sp), "phase mismatch")


def test_compiled_spec_every_unit_once_and_every_byte_written():
    W, H = 1920, 1080
    d = _handle(W, H, 3, 1, HALO)
    L = ds.lib()
    x = ds.generate_frames(23, d.in_frame_bytes, seed=2)
    for n in (1, 2, 7, 23):
        units = L.ds_units(d.handle, n, GENERAL)
        counts = torch.zeros(units, dtype=torch.int32, device="cuda")
        assert L.ds_set_debug_counter(d.handle, counts.data_ptr()) == 0
        d(x[:n])
        torch.cuda.synchronize()
        assert L.ds_set_debug_counter(d.handle, None) == 0
        assert d.last_variant() == 2
        c = counts.cpu().numpy()
        assert (c == 1).all(), (n, int((c == 0).sum()), int((c > 1).sum()))
    n = 3
    fr = synth.random_frames(2, 0, n, W, H)
    want = _want(fr, W, H, 3, 1, HALO)
    xs = torch.from_numpy(fr).cuda()
    guard = 4096
    for sentinel in (0x00, 0xA5):
        buf = torch.full((n * d.out_frame_bytes + 2 * guard,), sentinel, dtype=torch.uint8, device="cuda")
        y = buf[guard: guard + n * d.out_frame_bytes].view(n, -1)
        d(xs, y)
        torch.cuda.synchronize()
        assert d.last_variant() == 2
        _same(y.cpu().numpy(), want, f"sentinel {sentinel:#x}")
        b = buf.cpu().numpy()
        assert (b[:guard] == sentinel).all() and (b[-guard:] == sentinel).all(), "write outside output"


def test_compiled_spec_stream_every_frame():
    """The bench workload (--spec halo): 300 HD 4:2:0 frames in one launch,
    every frame against O1 with the halo stages, fanned out over host cores."""
    from oracle.verify import verify_stream

    W, H, N = 1920, 1080, 300
    d = _handle(W, H, 3, 1, HALO)
    x = ds.generate_frames(N, d.in_frame_bytes, seed=1)
    y = d(x).cpu().numpy()
    assert d.last_variant() == 2
    r = verify_stream(y, W, H, 3, 1, seed=1, stages=HALO)
    assert r["bit_exact"] and r["frames_checked"] == N, r


# a spec with no built-in instance: origins 3 / -5 (window phases 3 and 11), sparse
# and uneven taps, a pattern shorter than the paving in V's output 1
OTHER = (
    dict(pattern=13, paving=8, origin=3,
         weights=[[1, 2, 3, 0, 0, 0, 0, 0, 0, 0, 0, 1, 1], [0, 0, 0, 2, 2, 2, 0, 0, 0, 0, 0, 0, 2],
                  [0, 0, 0, 0, 0, 0, 4, 4, 1, 1, 0, 0, 0]], divisor=8, bias=4),
    dict(pattern=14, paving=9, origin=-5,
         weights=[[2, 2, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 4], [0, 0, 4, 4],
                  [0, 0, 0, 0, 0, 3, 3, 0, 0, 0, 0, 2], [0, 0, 0, 0, 0, 0, 0, 5, 3]], divisor=8, bias=4),
)


@pytest.mark.parametrize("spec,W,H,chroma", [("other", 1920, 1080, 1), ("other", 352, 288, 1),
                                            ("negative", 704, 576, 0), ("odd_divisor", 1024, 144, 1),
                                            ("other", 720, 576, 1), ("negative", 1400, 198, 0)])
def test_run_time_compiled_spec(spec, W, H, chroma):
    """A spec without a built-in instance: ds_set_general_variant(COMPILED)
    compiles K-N1s for it at run time (NVRTC, from the same kernel source);
    the output equals the oracle and the runtime-tap kernel."""
    rng = np.random.default_rng(len(spec) + W)
    if spec == "other":
        sp = OTHER
    elif spec == "negative":           # negative lobes: the clamp at 0 is live
        sp = (dict(pattern=12, paving=8, origin=-3, weights=[[-1, 4, 9, 4, -1], [0, 0, 0, -1, 5, 8, 5, -1],
                                                             [0, 0, 0, 0, 0, 0, -2, 6, 9, 6, -2]],
                   divisor=15, bias=7),
              dict(pattern=11, paving=9, origin=2, weights=[[-1, 6, 6, -1], [0, 0, 0, 1, 4, 4, 1], [0, 0, 0, 0, 0, 2, 3, 2],
                                                            [0, 0, 0, 0, 0, 0, 0, 1, 3, 3, 1]], divisor=10, bias=5))
    else:                              # odd divisors (float division path) with random taps
        wh = [[int(x) for x in rng.integers(0, 9, 10)] for _ in range(3)]
        wv = [[int(x) for x in rng.integers(0, 9, 12)] for _ in range(4)]
        sp = (dict(pattern=10, paving=8, origin=5, weights=wh, divisor=int(sum(wh[0])) | 1, bias=3),
              dict(pattern=12, paving=9, origin=-1, weights=wv, divisor=int(sum(wv[0])) | 1, bias=2))
    d = _handle(W, H, 3, chroma, sp)
    try:
        d.set_general_variant(ds.DS_GENERAL_COMPILED)
    except ds.DSError as e:
        pytest.fail(f"run-time compilation unavailable: {e}")
    assert d.launch_info(2, GENERAL)["variant"] == 3
    n = 3
    fr = synth.random_frames(91, 0, n, W, H, 3, chroma)
    x = torch.from_numpy(fr).cuda()
    y = d(x)
    torch.cuda.synchronize()
    assert d.last_variant() == 2
    want = _want(fr, W, H, 3, chroma, sp)
    _same(y.cpu().numpy(), want, f"K-N1s (run-time compiled) {spec} {W}x{H}")
    # the run-time compiled instance is built for the plan's row alignment only:
    # an input pointer less aligned than that runs the runtime-tap kernel
    plan_al = 16 if d.in_frame_bytes % 16 == 0 and W % 16 == 0 else 8
    xb = torch.zeros(x.numel() + 16, dtype=torch.uint8, device="cuda")
    xi = xb[4:4 + x.numel()].view(n, -1)
    xi.copy_(x)
    y4 = d(xi)
    torch.cuda.synchronize()
    assert d.last_variant() == (2 if plan_al == 4 else 1)
    _same(y4.cpu().numpy(), want, f"{spec} input offset 4")
    d.set_general_variant(ds.DS_GENERAL_RUNTIME)
    _same(d(x).cpu().numpy(), want, f"runtime taps {spec}")


def test_run_time_compilation_refused_outside_k1s():
    # taps outside s8 cannot go through dp4a: no compiled variant
    sp = (dict(pattern=8, paving=8, origin=0, weights=[[200, 5], [0, 0, 0, 3, 3], [0, 0, 0, 0, 0, 0, 5, 1]],
               divisor=206, bias=3), None)
    d = _handle(352, 288, 3, 1, (sp[0], HALO[1]))
    with pytest.raises(ds.DSError):
        d.set_general_variant(ds.DS_GENERAL_COMPILED)
