"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
byte for byte.  SPEC fixes integer pixel arithmetic,
so the tolerance is zero.  P:n = PAPER.md line n, S:n = SPEC.md line n."""
import numpy as np
import pytest

import oracle
import synth
from conftest import FUZZ_SCALE, fuzz_seed

torch = pytest.importorskip("torch")
ds = pytest.importorskip("paper_1103_4881_b200")

pytestmark = pytest.mark.gpu

FUSED, GENERIC = ds.DS_KERNEL_FUSED, ds.DS_KERNEL_GENERIC


def _run(d, frames_np, kernel=None):
    if kernel is not None:
        d.set_kernel(kernel)
    x = torch.from_numpy(np.ascontiguousarray(frames_np)).cuda()
    y = d(x)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def _assert_same(got, want, what=""):
    if not np.array_equal(got, want):
        idx = np.argwhere(got != want)
        raise AssertionError(f"{what}: {len(idx)} bytes differ; first at {idx[:5].tolist()} "
                             f"got {got[tuple(idx[0])]} want {want[tuple(idx[0])]}")


def _spec_chroma(chroma):
    s = ds.ds_default_spec()
    s.chroma = chroma
    return s


# ------------------------------------------------------------- config 0 --
@pytest.mark.parametrize("kernel", [FUSED, GENERIC])
def test_tiny_48x27(kernel):
    """BASELINE configs[0]: a tiny 48x27 1-channel frame (output frame of
    216 B is not 16-byte aligned: K-N1 takes its cooperative-store path)."""
    d = ds.Downscaler(48, 27, 1)
    for seed in range(5):
        fr = synth.random_frames(seed, 0, 3, 48, 27, 1)
        got = _run(d, fr, kernel)
        assert d.last_kernel() == kernel
        _assert_same(got, oracle.execute_frames(fr, 48, 27, 1, 1), f"tiny seed {seed}")
    # the golden of tests/golden/linear_48x27.json through the GPU
    fr = synth.linear_frames(1, 48, 27, 1)
    _assert_same(_run(d, fr, kernel), oracle.execute_frames(fr, 48, 27, 1, 1), "tiny linear")


# ---------------------------------------------------------- paper testbed --
@pytest.mark.parametrize("kernel", [FUSED, GENERIC])
def test_cif_420_100_seeded_frames(kernel):
    """100 random seeded CIF 4:2:0 frames bit-identical to the oracle."""
    d = ds.Downscaler(352, 288, 3)
    fr = synth.random_frames(0, 0, 100, 352, 288)
    got = _run(d, fr, kernel)
    assert d.last_kernel() == kernel
    _assert_same(got, oracle.execute_frames(fr, 352, 288), "cif")
    assert got.shape == (100, 132 * 128 + 2 * 66 * 64)


@pytest.mark.parametrize("chroma", [ds.DS_CHROMA_420, ds.DS_CHROMA_444])
def test_structured_frames_cif(chroma):
    d = ds.Downscaler(352, 288, 3, chroma=chroma)
    frames = [synth.constant_frames(c, 1, 352, 288, 3, chroma) for c in (0, 1, 100, 254, 255)]
    frames += [synth.checkerboard_frames(2, 352, 288, 3, chroma),
               synth.ramp_frames(4, 352, 288, 3, chroma),
               synth.linear_frames(2, 352, 288, 3, chroma)]
    fr = np.concatenate(frames)
    _assert_same(_run(d, fr), oracle.execute_frames(fr, 352, 288, 3, chroma), "structured")
    for c in (0, 1, 100, 254, 255):   # constants preserved
        one = synth.constant_frames(c, 1, 352, 288, 3, chroma)
        assert (_run(d, one) == c).all()


def test_impulses_every_tile_position():
    """An impulse at each of the 72 (row, col) positions of a 9x8 tile,
    tiled across a frame with varying amplitudes (dead taps included)."""
    W, H = 352, 288
    d = ds.Downscaler(W, H, 1)
    frames = []
    for r in range(9):
        for c in range(8):
            y, x = np.mgrid[0:H, 0:W]
            amp = ((x // 8 + 3 * (y // 9)) * 37) % 256
            fr = np.where((y % 9 == r) & (x % 8 == c), amp, 0).astype(np.uint8)
            frames.append(fr.reshape(1, -1))
    fr = np.concatenate(frames)
    _assert_same(_run(d, fr), oracle.execute_frames(fr, W, H, 1, 1), "impulses")


# ------------------------------------------------------- exhaustive pairs --
def test_exhaustive_h_pairs():
    """All 65,536 (a, b) pairs in every horizontal tap pair (p0,p1), (p3,p4),
    (p6,p7): row y carries a = y mod 256, packet p carries b = p."""
    W, H = 8 * 256, 9 * 256
    y, x = np.mgrid[0:H, 0:W]
    pos = x % 8
    a = y % 256
    b = x // 8
    plane = np.where(np.isin(pos, (0, 3, 6)), a, np.where(np.isin(pos, (1, 4, 7)), b, 77))
    fr = plane.astype(np.uint8).reshape(1, -1)
    d = ds.Downscaler(W, H, 1)
    _assert_same(_run(d, fr), oracle.execute_frames(fr, W, H, 1, 1), "h pairs")


def test_exhaustive_v_pairs():
    """All 65,536 (m_a, m_b) pairs in every vertical tap pair: constant
    packets make mid = the constant; rows 0,2,5,7 of group g hold g, rows
    1,3,6,8 hold the packet index, row 4 (dead) holds noise."""
    W, H = 8 * 256, 9 * 256
    y, x = np.mgrid[0:H, 0:W]
    g, r, p = y // 9, y % 9, x // 8
    noise = synth.random_frames(3, 0, 1, W, H, 1)[0].reshape(H, W)
    plane = np.where(np.isin(r, (0, 2, 5, 7)), g, np.where(np.isin(r, (1, 3, 6, 8)), p, noise))
    fr = plane.astype(np.uint8).reshape(1, -1)
    d = ds.Downscaler(W, H, 1)
    _assert_same(_run(d, fr), oracle.execute_frames(fr, W, H, 1, 1), "v pairs")


# -------------------------------------------------------------- HD / 4K --
@pytest.mark.parametrize("chroma", [ds.DS_CHROMA_420, ds.DS_CHROMA_444])
@pytest.mark.parametrize("kernel", [FUSED, GENERIC])
def test_one_hd_frame(chroma, kernel):
    """BASELINE configs[1]: one HD 1920x1080 frame."""
    d = ds.Downscaler(1920, 1080, 3, chroma=chroma)
    fr = np.concatenate([synth.random_frames(1, 0, 1, 1920, 1080, 3, chroma),
                         synth.ramp_frames(1, 1920, 1080, 3, chroma)])
    got = _run(d, fr, kernel)
    assert d.last_kernel() == kernel
    _assert_same(got, oracle.execute_frames(fr, 1920, 1080, 3, chroma), "hd")


@pytest.mark.parametrize("chroma", [ds.DS_CHROMA_420, ds.DS_CHROMA_444])
def test_4k_frames(chroma):
    d = ds.Downscaler(3840, 2160, 3, chroma=chroma)
    fr = synth.random_frames(5, 7, 2, 3840, 2160, 3, chroma)
    _assert_same(_run(d, fr), oracle.execute_frames(fr, 3840, 2160, 3, chroma), "4k")


# --------------------------------------------------------- ragged shapes --
@pytest.mark.parametrize("W,H,ch", [(16, 9, 1), (32, 18, 3), (400, 9, 1), (48, 99, 1),
                                    (40, 45, 1), (208, 90, 3), (1504, 54, 3), (2000, 27, 1),
                                    (176, 144, 3), (8, 9, 1), (720, 576, 3), (24, 9, 1),
                                    (1440, 1080, 3), (720, 486, 3)])
def test_ragged_geometries(W, H, ch):
    """Widths that are / are not multiples of 16 (K-N1 vs K-N2 auto choice),
    band counts that leave a ragged tail over the persistent grid."""
    d = ds.Downscaler(W, H, ch)
    fr = synth.random_frames(W + H, 0, 7, W, H, ch, 1)
    got = _run(d, fr)
    want_kernel = (FUSED if d.plan.fused_eligible else
                   ds.DS_KERNEL_FUSED_GENERAL if d.plan.fused_general_eligible else GENERIC)
    assert d.last_kernel() == want_kernel
    _assert_same(got, oracle.execute_frames(fr, W, H, ch, 1), f"{W}x{H}x{ch}")


@pytest.mark.parametrize("W,H,ch,chroma", [(16, 9, 1, 1), (8, 9, 1, 1), (16, 18, 3, 1), (32, 9, 1, 1),
                                           (1920, 9, 1, 1), (8, 900, 1, 1), (16, 18, 3, 0), (2048, 18, 3, 1)])
def test_degenerate_geometries_every_kernel(W, H, ch, chroma):
    """Smallest planes (one 8- or 16-byte row, one 9-row group), a single
    band over a wide plane and a tall narrow column, through every kernel that
    can take them (K-N1, K-N1g, K-N2), at 1, 2 and 5 frames."""
    d = ds.Downscaler(W, H, ch, chroma=chroma)
    kernels = [GENERIC, ds.DS_KERNEL_FUSED_GENERAL] + ([FUSED] if d.plan.fused_eligible else [])
    for n in (1, 2, 5):
        fr = synth.random_frames(W * 7 + H, 3, n, W, H, ch, chroma)
        want = oracle.execute_frames(fr, W, H, ch, chroma)
        for k in kernels:
            if k == ds.DS_KERNEL_FUSED_GENERAL and not d.plan.fused_general_eligible:
                continue
            got = _run(d, fr, k)
            assert d.last_kernel() == k
            _assert_same(got, want, f"{W}x{H}x{ch} chroma={chroma} n={n} kernel={k}")
    d.set_kernel(ds.DS_KERNEL_AUTO)


def test_zero_frames_noop():
    d = ds.Downscaler(352, 288, 3)
    x = torch.empty((0, d.in_frame_bytes), dtype=torch.uint8, device="cuda")
    y = d(x)
    assert y.shape == (0, d.out_frame_bytes)


# ----------------------------------------------------- general specs (K-N2) --
def _halo_spec():
    h = dict(pattern=13, paving=8, origin=3,
             weights=[[1, 2, 3, 0, 0, 0, 0, 0, 0, 0, 0, 1, 1], [0, 0, 0, 2, 2, 2, 0, 0, 0, 0, 0, 0, 2],
                      [0, 0, 0, 0, 0, 0, 4, 4, 1, 1, 0, 0, 0]], divisor=8, bias=4)
    v = dict(pattern=14, paving=9, origin=-5,
             weights=[[2, 2, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 4], [0, 0, 4, 4],
                      [0, 0, 0, 0, 0, 3, 3, 0, 0, 0, 0, 2], [0, 0, 0, 0, 0, 0, 0, 5, 3]],
             divisor=8, bias=4)
    return h, v


def _oracle_stage(d):
    return oracle.make_stage(d["pattern"], d["paving"], d["origin"], d["weights"], d["divisor"],
                             d["bias"])


@pytest.mark.parametrize("W,H,ch", [(48, 27, 1), (352, 288, 3), (64, 36, 3), (1920, 1080, 3)])
@pytest.mark.parametrize("kernel,variant", [(ds.DS_KERNEL_FUSED_GENERAL, ds.DS_GENERAL_RUNTIME),
                                            (ds.DS_KERNEL_FUSED_GENERAL, ds.DS_GENERAL_AUTO), (GENERIC, 0)])
def test_halo_and_origin_spec(W, H, ch, kernel, variant):
    """P > S halos with toroidal wrap and origin != 0:
    K-N1g with runtime taps (halo rows staged in smem, smem intermediate;
    runs of bands that reuse the halo's intermediate rows, forced from 1 band
    to whole planes), K-N1g's default (K-N1s compiled for this spec at run time
    where it can run) and K-N2."""
    hd, vd = _halo_spec()
    spec = ds.make_spec(h=hd, v=vd, chroma=ds.DS_CHROMA_420)
    d = ds.Downscaler(W, H, ch, spec=spec)
    d.set_general_variant(variant)
    assert d.plan.fused_general_eligible == 1 and d.plan.fused_eligible == 0
    fr = synth.random_frames(9, 0, 3, W, H, ch, 1)
    want = oracle.execute_frames(fr, W, H, ch, 1, _oracle_stage(hd), _oracle_stage(vd))
    for bands in ((0, 1, 2, 3, 1 << 20) if kernel == ds.DS_KERNEL_FUSED_GENERAL else (0,)):
        d.set_run_bands(bands)
        got = _run(d, fr, kernel)
        assert d.last_kernel() == kernel
        _assert_same(got, want, f"halo, run bands {bands}")


@pytest.mark.parametrize("stage_bytes", [1024, 2048, 3000])
@pytest.mark.parametrize("spec_kind", ["halo", "spec_taps", "negative"])
def test_general_column_strips(stage_bytes, spec_kind):
    """K-N1g column strips (ds_set_general_stage_bytes forces them on small
    frames): strip windows staged from 16-aligned supersets (wrapping the row
    end under origin != 0), the last strip narrower, runs reusing the V halo
    within a strip, strip-wise output rows -- against the oracle."""
    W, H, ch = 352, 288, 3
    if spec_kind == "halo":
        hd, vd = _halo_spec()
    elif spec_kind == "spec_taps":
        hd = vd = None
    else:
        hd = dict(pattern=6, paving=4, origin=-1, weights=[[-1, 3, 3, -1], [0, 0, -1, 3, 3, -1]],
                  divisor=4, bias=2)
        vd = dict(pattern=11, paving=6, origin=3, weights=[[1, 2, 1], [0, 0, 0, 1, 2, 1, 0, 0, 0, 0, 4]],
                  divisor=4, bias=-2)
        W, H = 352, 288
    spec = ds.make_spec(h=hd, v=vd, chroma=ds.DS_CHROMA_420)
    d = ds.Downscaler(W, H, ch, spec=spec)
    d.set_general_variant(ds.DS_GENERAL_RUNTIME)                 # strips are the runtime-tap kernel's
    d.set_general_stage_bytes(stage_bytes)
    assert d.plan.fused_general_eligible == 1 and d.plan.general_strips[0] > 1
    fr = synth.random_frames(7, 0, 4, W, H, ch, 1)
    if hd is None:
        want = oracle.execute_frames(fr, W, H, ch, 1)
    else:
        want = oracle.execute_frames(fr, W, H, ch, 1, _oracle_stage(hd), _oracle_stage(vd))
    for bands in (0, 1, 3):
        d.set_run_bands(bands)
        got = _run(d, fr, ds.DS_KERNEL_FUSED_GENERAL)
        assert d.last_kernel() == ds.DS_KERNEL_FUSED_GENERAL
        _assert_same(got, want, f"strips {stage_bytes} {spec_kind} run bands {bands}")
    # misaligned input: strip windows staged by the producer warp (plain loads)
    buf = torch.zeros(fr.size + 64, dtype=torch.uint8, device="cuda")
    x = buf[3: 3 + fr.size]
    x.copy_(torch.from_numpy(fr.ravel()).cuda())
    y = torch.zeros(want.size, dtype=torch.uint8, device="cuda")
    d.set_kernel(ds.DS_KERNEL_FUSED_GENERAL)
    ds.ds_run(d.handle, x.data_ptr(), 4, y.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    _assert_same(y.cpu().numpy().reshape(want.shape), want, f"strips coop {stage_bytes} {spec_kind}")
    d.set_general_stage_bytes(0)
    assert list(d.plan.general_strips) == [1, 1, 1]
    with pytest.raises(ds.DSError):
        d.set_general_stage_bytes(-1)


def test_general_strips_8k_halo():
    """8K 4:2:0 under the halo spec: whole rows exceed shared memory, so
    K-N1g runs in column strips (before strips this geometry fell back to
    K-N2) -- sampled whole frames against the oracle."""
    W, H = 7680, 4320
    hd, vd = _halo_spec()
    d = ds.Downscaler(W, H, 3, spec=ds.make_spec(h=hd, v=vd, chroma=ds.DS_CHROMA_420))
    d.set_general_variant(ds.DS_GENERAL_RUNTIME)
    assert d.plan.fused_general_eligible == 1 and d.plan.general_strips[0] > 1
    fr = synth.random_frames(11, 0, 2, W, H, 3, 1)
    got = _run(d, fr, ds.DS_KERNEL_FUSED_GENERAL)
    _assert_same(got, oracle.execute_frames(fr, W, H, 3, 1, _oracle_stage(hd), _oracle_stage(vd)), "8K strips")


def test_negative_weights_and_other_ratio():
    """Negative lobes (truncation toward zero, clamp) and a 4->2 / 3->1 ratio."""
    hd = dict(pattern=6, paving=4, origin=-1, weights=[[-1, 3, 3, -1], [0, 0, -1, 3, 3, -1]],
              divisor=4, bias=2)
    vd = dict(pattern=3, paving=3, origin=0, weights=[[1, 2, 1]], divisor=4, bias=-2)
    spec = ds.make_spec(h=hd, v=vd)
    d = ds.Downscaler(64, 30, 1, spec=spec)
    fr = synth.random_frames(4, 0, 4, 64, 30, 1)
    want = oracle.execute_frames(fr, 64, 30, 1, 1, _oracle_stage(hd), _oracle_stage(vd))
    _assert_same(_run(d, fr), want, "negative")
    assert d.last_kernel() == ds.DS_KERNEL_FUSED_GENERAL
    _assert_same(_run(d, fr, GENERIC), want, "negative K-N2")


@pytest.mark.parametrize("variant", [ds.DS_GENERAL_RUNTIME, ds.DS_GENERAL_AUTO])
@pytest.mark.parametrize("W,H,ch,chroma", [(352, 288, 3, 1), (1920, 1080, 3, 1), (1920, 1080, 3, 0),
                                           (48, 27, 1, 1)])
def test_general_kernel_on_spec_taps(W, H, ch, chroma, variant):
    """K-N1g forced on SPEC's own downscaler equals the oracle (and K-N1),
    with runtime taps and as K-N1s (the built-in SPEC instance)."""
    d = ds.Downscaler(W, H, ch, chroma=chroma)
    d.set_general_variant(variant)
    fr = synth.random_frames(17, 0, 3, W, H, ch, chroma)
    got = _run(d, fr, ds.DS_KERNEL_FUSED_GENERAL)
    assert d.last_kernel() == ds.DS_KERNEL_FUSED_GENERAL
    _assert_same(got, oracle.execute_frames(fr, W, H, ch, chroma), "K-N1g spec taps")


def _random_spec(rng):
    def stage(max_p):
        P = int(rng.integers(1, max_p + 1))
        S = int(rng.integers(1, P + 3))
        Q = int(rng.integers(1, 5))
        # 999983: M D - 2^32 = 959672, so large taps leave the FASTDIV bound
        # (K-N1g's reciprocal + correction instantiation)
        D = int(rng.choice([1, 2, 3, 5, 6, 7, 8, 16, 100, 1 << 20, 999983]))
        w = [[int(x) if rng.random() < 0.7 else 0 for x in rng.integers(-40, 120, P)] for _ in range(Q)]
        total = max(1, sum(max(0, x) for row in w for x in row))
        return dict(pattern=P, paving=S, origin=int(rng.integers(-50, 50)), weights=w,
                    divisor=max(D, total // 255 if D == 1 else D), bias=int(rng.integers(-200, 400)))
    return stage(16), stage(16)


def test_general_kernel_fuzz_random_specs():
    """Random separable specs (halos, gaps P < S, origins, negative taps,
    divisors incl. 1 and 2^20) on random geometries, K-N1g vs the oracle."""
    rng = np.random.default_rng(fuzz_seed(2024))
    checked = compiled = 0
    for trial in range(40 * FUZZ_SCALE):
        hd, vd = _random_spec(rng)
        ch = int(rng.choice([1, 3]))
        chroma = int(rng.integers(0, 2))
        mult_w = hd["paving"] * 16 * (2 if ch == 3 and chroma == 1 else 1)
        mult_h = vd["paving"] * (2 if ch == 3 and chroma == 1 else 1)
        W = mult_w * int(rng.integers(1, max(2, 200 // mult_w + 1)))
        H = mult_h * int(rng.integers(1, max(2, 60 // mult_h + 1)))
        spec = ds.make_spec(h=hd, v=vd, chroma=chroma)
        d = ds.Downscaler(W, H, ch, spec=spec)
        if not d.plan.fused_general_eligible:
            continue
        fr = synth.random_frames(trial, 0, 2, W, H, ch, chroma)
        want = oracle.execute_frames(fr, W, H, ch, chroma, _oracle_stage(hd), _oracle_stage(vd))
        d.set_run_bands(int(rng.choice([0, 1, 2, 3, 7, 1 << 20])))   # halo reuse across bands
        if rng.random() < 0.3:                                         # column strips
            d.set_general_stage_bytes(int(rng.choice([1024, 3000, 8000])))
            if not d.plan.fused_general_eligible:
                continue
        d.set_general_variant(ds.DS_GENERAL_RUNTIME)
        got = _run(d, fr, ds.DS_KERNEL_FUSED_GENERAL)
        assert d.last_kernel() == ds.DS_KERNEL_FUSED_GENERAL and d.last_variant() == 1
        _assert_same(got, want, f"fuzz {trial}: {W}x{H}x{ch} h={hd} v={vd} strips={list(d.plan.general_strips)}")
        checked += 1
        # the same spec with the spec compiled in (K-N1s, NVRTC) wherever it can run
        try:
            d.set_general_variant(ds.DS_GENERAL_COMPILED)
        except ds.DSError:
            continue
        got = _run(d, fr, ds.DS_KERNEL_FUSED_GENERAL)
        assert d.last_variant() == 2
        _assert_same(got, want, f"fuzz {trial} K-N1s: {W}x{H}x{ch} h={hd} v={vd}")
        compiled += 1
    assert checked >= 25 * FUZZ_SCALE
    assert compiled >= 1


def test_general_kernel_fuzz_unaligned_geometry():
    """Random specs on geometries the TMA cannot stage (any W % 16, planes
    shorter than one band plus its halo) from input pointers 0-15 bytes into
    their allocation: K-N1g (producer- or consumer-staged rows) and, where it
    can run (H paving % 4 == 0, rows 4-byte aligned), K-N1s with 16-, 8- or
    4-byte loads -- against the oracle."""
    rng = np.random.default_rng(fuzz_seed(77))
    checked = compiled = 0
    for trial in range(40 * FUZZ_SCALE):
        hd, vd = _random_spec(rng)
        if rng.random() < 0.5:                       # a paving K-N1s can take
            hd["paving"] = int(rng.choice([4, 8, 12]))
        ch = int(rng.choice([1, 3]))
        chroma = int(rng.integers(0, 2))
        sub = 2 if ch == 3 and chroma == 1 else 1
        mult_w = hd["paving"] * sub
        mult_h = vd["paving"] * sub
        W = mult_w * int(rng.integers(max(1, 32 // mult_w), max(2, 400 // mult_w + 1)))
        H = mult_h * int(rng.integers(1, max(2, 40 // mult_h + 1)))
        spec = ds.make_spec(h=hd, v=vd, chroma=chroma)
        d = ds.Downscaler(W, H, ch, spec=spec)
        if not d.plan.fused_general_eligible:
            continue
        n = int(rng.integers(1, 4))
        fr = synth.random_frames(trial, 0, n, W, H, ch, chroma)
        want = oracle.execute_frames(fr, W, H, ch, chroma, _oracle_stage(hd), _oracle_stage(vd))
        d.set_run_bands(int(rng.choice([0, 1, 2, 1 << 20])))
        d.set_kernel(ds.DS_KERNEL_FUSED_GENERAL)
        off = int(rng.choice([0, 4, 8, 12, 1, 2, 3, 5]))
        buf = torch.zeros(fr.size + 32, dtype=torch.uint8, device="cuda")
        x = buf[off:off + fr.size].view(n, -1)
        x.copy_(torch.from_numpy(fr).view(n, -1))
        what = f"unaligned fuzz {trial}: {W}x{H}x{ch}/{chroma} off {off} h={hd} v={vd}"
        for variant in (ds.DS_GENERAL_RUNTIME, ds.DS_GENERAL_COMPILED):
            try:
                d.set_general_variant(variant)
            except ds.DSError:
                continue
            y = d(x)
            torch.cuda.synchronize()
            _assert_same(y.cpu().numpy(), want, f"{what} variant {d.last_variant()}")
            checked += d.last_variant() == 1
            compiled += d.last_variant() == 2
    assert checked >= 25 * FUZZ_SCALE
    assert compiled >= 1


# ------------------------------------------------------- alignment / API --
@pytest.mark.parametrize("off", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("W,H,strips", [(352, 288, False), (352, 288, True), (32, 36, False)])
def test_general_rows_staged_by_producer(off, W, H, strips):
    """Input the TMA cannot copy (pointer `off` bytes into its allocation) is
    staged by K-N1g's producer warp: cp.async for 4/8-byte aligned rows,
    aligned words funnelled by the misalignment otherwise, strip windows the
    same way (with bytes for the word that straddles the row end), and the
    32-byte wrap pad from row[j mod W] (rows shorter than 32 bytes: the 16-byte
    chroma rows of 32x36) -- halo spec with origin -2, against the oracle."""
    hd, vd = _halo_spec()
    spec = ds.make_spec(h=hd, v=vd, chroma=ds.DS_CHROMA_420)
    d = ds.Downscaler(W, H, 3, spec=spec)
    if strips:
        d.set_general_stage_bytes(2048)
        assert d.plan.general_strips[0] > 1
    fr = synth.random_frames(9, 0, 3, W, H, 3, 1)
    want = oracle.execute_frames(fr, W, H, 3, 1, _oracle_stage(hd), _oracle_stage(vd))
    buf = torch.zeros(fr.size + 64, dtype=torch.uint8, device="cuda")
    x = buf[off: off + fr.size]
    x.copy_(torch.from_numpy(fr.ravel()).cuda())
    d.set_kernel(ds.DS_KERNEL_FUSED_GENERAL)
    # the runtime-tap kernel's staging; then whatever AUTO picks (K-N1s where it
    # can run: 4/8-byte loads or funnel-shifted words)
    for variant in (ds.DS_GENERAL_RUNTIME, ds.DS_GENERAL_AUTO):
        d.set_general_variant(variant)
        y = torch.zeros(want.size, dtype=torch.uint8, device="cuda")
        ds.ds_run(d.handle, x.data_ptr(), 3, y.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert d.last_kernel() == ds.DS_KERNEL_FUSED_GENERAL
        if variant == ds.DS_GENERAL_RUNTIME:
            assert d.last_variant() == 1
        _assert_same(y.cpu().numpy().reshape(want.shape), want,
                     f"off={off} {W}x{H} strips={strips} variant {d.last_variant()}")


def test_misaligned_pointers():
    """Misaligned input moves off K-N1 (TMA needs 16-byte sources) to K-N1g,
    which stages the rows with plain loads; misaligned output makes K-N1 fall
    back to cooperative stores -- results identical, never an error."""
    W, H = 352, 288
    d = ds.Downscaler(W, H, 3)
    fr = synth.random_frames(2, 0, 3, W, H)
    want = oracle.execute_frames(fr, W, H)
    buf = torch.zeros(fr.size + 64, dtype=torch.uint8, device="cuda")
    x = buf[1: 1 + fr.size]
    x.copy_(torch.from_numpy(fr.ravel()).cuda())
    obuf = torch.zeros(want.size + 64, dtype=torch.uint8, device="cuda")
    y = obuf[3: 3 + want.size]
    ds.ds_run(d.handle, x.data_ptr(), 3, y.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert d.last_kernel() == ds.DS_KERNEL_FUSED_GENERAL
    _assert_same(y.cpu().numpy().reshape(want.shape), want, "misaligned in")
    d.set_kernel(GENERIC)
    y.zero_()
    ds.ds_run(d.handle, x.data_ptr(), 3, y.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert d.last_kernel() == GENERIC
    _assert_same(y.cpu().numpy().reshape(want.shape), want, "misaligned in, K-N2")
    d.set_kernel(ds.DS_KERNEL_AUTO)
    x2 = torch.from_numpy(fr).cuda()
    ds.ds_run(d.handle, x2.data_ptr(), 3, y.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert d.last_kernel() == FUSED
    _assert_same(y.cpu().numpy().reshape(want.shape), want, "misaligned out")


def test_run_errors():
    d = ds.Downscaler(352, 288, 3)
    x = torch.zeros((2, d.in_frame_bytes), dtype=torch.uint8, device="cuda")
    L = ds.lib()
    s = torch.cuda.current_stream().cuda_stream
    assert L.ds_run(d.handle, x.data_ptr(), -1, x.data_ptr(), s) == ds.DS_EINVAL
    # overlapping in/out
    assert L.ds_run(d.handle, x.data_ptr(), 1, x.data_ptr() + 100, s) == ds.DS_EINVAL
    # host pointer is not a device pointer
    hx = torch.zeros((2, d.in_frame_bytes), dtype=torch.uint8)
    y = d.alloc_out(2)
    assert L.ds_run(d.handle, hx.data_ptr(), 2, y.data_ptr(), s) == ds.DS_EINVAL
    assert L.ds_run(d.handle, 0, 2, y.data_ptr(), s) == ds.DS_EINVAL
    assert L.ds_run(d.handle, x.data_ptr(), 0, y.data_ptr(), s) == ds.DS_OK
    # pinned host output: not device memory, and no peer can make it one
    hy = torch.zeros((2, d.out_frame_bytes), dtype=torch.uint8, pin_memory=True)
    assert L.ds_run(d.handle, x.data_ptr(), 2, hy.data_ptr(), s) == ds.DS_EINVAL
    # ds_enable_peer: own device is a no-op; a device that does not exist is EINVAL
    assert L.ds_enable_peer(d.handle, torch.cuda.current_device()) == ds.DS_OK
    assert L.ds_enable_peer(d.handle, torch.cuda.device_count()) == ds.DS_EINVAL
    assert L.ds_enable_peer(d.handle, -1) == ds.DS_EINVAL


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_peer_output_needs_explicit_enable():
    """ds_run returns DS_EINVAL for an output on another GPU and
    enables nothing itself; after ds_enable_peer the same call stores the
    frames on the peer (the fused gather's path) bit-exactly."""
    W, H = 352, 288
    torch.cuda.set_device(0)
    d = ds.Downscaler(W, H, 3)
    fr = synth.random_frames(21, 0, 4, W, H)
    x = torch.from_numpy(fr).cuda(0)
    y1 = torch.zeros((4, d.out_frame_bytes), dtype=torch.uint8, device="cuda:1")
    L = ds.lib()
    s = torch.cuda.current_stream().cuda_stream
    assert L.ds_run(d.handle, x.data_ptr(), 4, y1.data_ptr(), s) == ds.DS_EINVAL
    rc = L.ds_enable_peer(d.handle, 1)
    if rc == ds.DS_EUNSUPPORTED:
        pytest.skip("GPUs 0 and 1 cannot access each other")
    assert rc == ds.DS_OK
    assert L.ds_run(d.handle, x.data_ptr(), 4, y1.data_ptr(), s) == ds.DS_OK
    torch.cuda.synchronize()
    _assert_same(y1.cpu().numpy(), oracle.execute_frames(fr, W, H), "peer output")


def test_tuning_does_not_change_results():
    W, H = 1920, 1080
    d = ds.Downscaler(W, H, 3)
    fr = synth.random_frames(11, 0, 6, W, H)
    x = torch.from_numpy(fr).cuda()
    ref = d(x).cpu().numpy()
    _assert_same(ref, oracle.execute_frames(fr, W, H), "tuning ref")
    for band in (0, 8 * 1920, 64 * 1024, 1):
        d.set_band_bytes(band)
        for stages in (2, 3, 5, 8):
            for ctas in (0, 1, 2, 3):
                d.set_tuning(stages, ctas)
                y = d(x)
                torch.cuda.synchronize()
                assert d.last_kernel() == FUSED
                _assert_same(y.cpu().numpy(), ref, f"band={band} stages={stages} ctas={ctas}")


def test_two_streams_one_handle():
    W, H = 352, 288
    d = ds.Downscaler(W, H, 3)
    fr = synth.random_frames(6, 0, 40, W, H)
    x = torch.from_numpy(fr).cuda()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    y1, y2 = d.alloc_out(40), d.alloc_out(40)
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        d(x, y1)
    with torch.cuda.stream(s2):
        d(x, y2)
    torch.cuda.synchronize()
    want = oracle.execute_frames(fr, W, H)
    _assert_same(y1.cpu().numpy(), want, "s1")
    _assert_same(y2.cpu().numpy(), want, "s2")


def test_device_generator_matches_host_generator():
    fb = synth.in_frame_bytes(1920, 1080)
    g = ds.generate_frames(3, fb, seed=1, first_frame=5)
    torch.cuda.synchronize()
    _assert_same(g.cpu().numpy(), synth.random_frames(1, 5, 3, 1920, 1080), "generator")
    # unaligned / ragged tail
    buf = torch.zeros(1000, dtype=torch.uint8, device="cuda")
    ds.ds_generate(buf.data_ptr() + 3, 997, 9, 12345, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    _assert_same(buf.cpu().numpy()[3:], synth.random_bytes(9, 12345, 997), "gen tail")


# ------------------------------------------------------------- host path --
def test_run_host_pinned_and_pageable():
    W, H = 352, 288
    d = ds.Downscaler(W, H, 3)
    n = 50
    fr = synth.random_frames(8, 0, n, W, H)
    want = oracle.execute_frames(fr, W, H)
    for pinned in (True, False):
        hin = torch.from_numpy(fr)
        if pinned:
            hin = hin.pin_memory()
        d.set_host_chunk(7)                      # several chunks, ragged last one
        hout = d.run_host(hin)
        torch.cuda.current_stream().synchronize()
        _assert_same(hout.numpy(), want, f"host pinned={pinned}")


def test_run_host_general_spec():
    """The host path under a halo spec (K-N1g; every input row crosses PCIe,
    since only SPEC's taps have a dead row), chunked, pinned and pageable."""
    W, H = 352, 288
    hd, vd = _halo_spec()
    d = ds.Downscaler(W, H, 3, spec=ds.make_spec(h=hd, v=vd, chroma=ds.DS_CHROMA_420))
    n = 20
    fr = synth.random_frames(21, 0, n, W, H)
    want = oracle.execute_frames(fr, W, H, 3, 1, _oracle_stage(hd), _oracle_stage(vd))
    for pinned in (True, False):
        hin = torch.from_numpy(fr)
        if pinned:
            hin = hin.pin_memory()
        d.set_host_chunk(6)
        hout = d.run_host(hin)
        torch.cuda.current_stream().synchronize()
        assert d.last_kernel() == ds.DS_KERNEL_FUSED_GENERAL
        _assert_same(hout.numpy(), want, f"host halo pinned={pinned}")


def test_run_host_hd_auto_chunk():
    W, H = 1920, 1080
    d = ds.Downscaler(W, H, 3)
    n = 24
    fr = synth.random_frames(12, 0, n, W, H)
    hin = torch.from_numpy(fr).pin_memory()
    hout = d.run_host(hin)
    torch.cuda.current_stream().synchronize()
    idx = [0, 9, 10, 23]
    _assert_same(hout.numpy()[idx], oracle.execute_frames(fr[idx], W, H), "host hd")


# ------------------------------------------------- full-size, bench config --
def test_hd_300_frame_stream_bench_config():
    """BASELINE configs[2] at full size, in bench.py's launch configuration
    (device-generated frames, default tuning): whole-frame oracle checks on
    sampled frames, O3 per-pixel checks on many more, and frame-independence
    (no cross-frame contamination) via the last frame."""
    W, H, N = 1920, 1080, 300
    d = ds.Downscaler(W, H, 3)
    x = ds.generate_frames(N, d.in_frame_bytes, seed=1)
    y = d(x)
    torch.cuda.synchronize()
    assert d.last_kernel() == FUSED
    for f in (0, 1, 149, 298, 299):
        fr = synth.random_frames(1, f, 1, W, H)
        _assert_same(y[f].cpu().numpy()[None], oracle.execute_frames(fr, W, H), f"frame {f}")
    rng = np.random.default_rng(0)
    for f in rng.choice(N, 20, replace=False):
        fr = synth.random_frames(1, int(f), 1, W, H)[0]
        out = y[int(f)].cpu().numpy()
        ins = oracle.split_planes(fr, W, H)
        outs = oracle.split_planes(out, W, H, out=True)
        for pin, pout in zip(ins, outs):
            ho, wo = pout.shape
            for R, Cc in zip(rng.integers(0, ho, 200), rng.integers(0, wo, 200)):
                assert pout[R, Cc] == oracle.pixel(pin, int(R), int(Cc))


def test_hd_300_frame_stream_every_frame():
    """BASELINE configs[2], the bench workload, verified on EVERY frame: all
    300 device outputs against the oracle's direct nested loops (O2, pinned
    equal to the tiler executor O1 by the CPU tests), frames regenerated on
    the host by global index."""
    W, H, N = 1920, 1080, 300
    d = ds.Downscaler(W, H, 3)
    x = ds.generate_frames(N, d.in_frame_bytes, seed=1)
    y = d(x).cpu().numpy()
    assert d.last_kernel() == FUSED
    for f0 in range(0, N, 50):
        fr = synth.random_frames(1, f0, 50, W, H)
        _assert_same(y[f0: f0 + 50], oracle.direct_frames(fr, W, H), f"frames {f0}..{f0 + 49}")
    for chroma in (0,):                 # HD 4:4:4 (the three-equal-planes reading, A4) too
        d4 = ds.Downscaler(W, H, 3, chroma=chroma)
        y4 = d4(ds.generate_frames(N, d4.in_frame_bytes, seed=1)).cpu().numpy()
        from oracle.verify import verify_stream

        r = verify_stream(y4, W, H, 3, chroma, seed=1)
        assert r["frames_checked"] == N and r["bit_exact"], r


def test_cuda_graph_capture():
    """ds_run is capturable in a CUDA graph (the launch-bound 1-frame config
    replays a graph); replayed output equals the oracle."""
    W, H = 1920, 1080
    d = ds.Downscaler(W, H, 3)
    fr = synth.random_frames(21, 0, 1, W, H)
    x = torch.from_numpy(fr).cuda()
    y = d.alloc_out(1)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        d(x, y)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    y.zero_()
    with torch.cuda.graph(g, stream=s):
        d(x, y)
    y.zero_()
    g.replay()
    torch.cuda.synchronize()
    _assert_same(y.cpu().numpy(), oracle.execute_frames(fr, W, H), "graph replay")
    assert d.launch_shape(1) != d.launch_shape(300)     # small batches use the fine band plan


@pytest.mark.parametrize("kernel", [FUSED, ds.DS_KERNEL_FUSED_GENERAL, GENERIC])
@pytest.mark.parametrize("W,H,ch,n", [(1920, 1080, 3, 3), (352, 288, 3, 5), (48, 27, 1, 4),
                                      (720, 576, 3, 2), (176, 144, 3, 3)])
def test_every_output_byte_written(kernel, W, H, ch, n):
    """compute-sanitizer is closed on this pool; instead, outputs pre-filled
    with two different sentinels must both come back equal to the oracle, so
    every output byte is written by the kernel (and nothing else is)."""
    d = ds.Downscaler(W, H, ch)
    if kernel == FUSED and not d.plan.fused_eligible:
        pytest.skip("K-N1 needs 16-byte rows in every plane")
    d.set_kernel(kernel)
    fr = synth.random_frames(31, 0, n, W, H, ch, 1)
    want = oracle.execute_frames(fr, W, H, ch, 1)
    x = torch.from_numpy(fr).cuda()
    guard = 4096
    for sentinel in (0x00, 0xA5):
        buf = torch.full((n * d.out_frame_bytes + 2 * guard,), sentinel, dtype=torch.uint8, device="cuda")
        y = buf[guard: guard + n * d.out_frame_bytes].view(n, -1)
        d(x, y)
        torch.cuda.synchronize()
        assert d.last_kernel() == kernel
        _assert_same(y.cpu().numpy(), want, f"sentinel {sentinel:#x}")
        b = buf.cpu().numpy()
        assert (b[:guard] == sentinel).all() and (b[-guard:] == sentinel).all(), "write outside output"


@pytest.mark.parametrize("W,H,N,chroma", [(1920, 1080, 3000, 1), (3840, 2160, 1000, 1),
                                          (3840, 2160, 1000, 0)])
def test_full_size_streams_every_frame(W, H, N, chroma):
    """BASELINE configs[3] (3000 HD 4:2:0 frames: the whole stream on one GPU,
    i.e. every rank's shard at once) and configs[4] (1000 4K frames, 4:2:0 and
    4:4:4) at full size in bench.py's launch configuration (one ds_run over
    the stream, default tuning), verified on EVERY frame byte for byte
     against the oracle's direct loops (O2), fanned out
    over the host cores as single-threaded processes that regenerate the
    frames by global index (oracle/verify.py); plus O3 per-pixel samples."""
    from oracle.verify import verify_stream

    d = ds.Downscaler(W, H, 3, chroma=chroma)
    x = ds.generate_frames(N, d.in_frame_bytes, seed=1)
    y = d(x)
    torch.cuda.synchronize()
    assert d.last_kernel() == FUSED
    del x
    host = y.cpu().numpy()
    del y
    torch.cuda.empty_cache()
    r = verify_stream(host, W, H, 3, chroma, seed=1)
    assert r["frames_checked"] == N and r["bit_exact"], r
    rng = np.random.default_rng(N)
    for f in rng.choice(N, 4, replace=False):
        fr = synth.random_frames(1, int(f), 1, W, H, 3, chroma)[0]
        for pin, pout in zip(oracle.split_planes(fr, W, H, 3, chroma),
                             oracle.split_planes(host[int(f)], W, H, 3, chroma, out=True)):
            ho, wo = pout.shape
            for R, Cc in zip(rng.integers(0, ho, 100), rng.integers(0, wo, 100)):
                assert pout[R, Cc] == oracle.pixel(pin, int(R), int(Cc))


def test_fused_kernel_fuzz():
    """Random geometries (W % 16 == 0, H % 9 or 18 == 0), channel/chroma
    modes, frame counts, band sizes, ring depths and output-pointer
    alignments: K-N1 byte-for-byte against the oracle."""
    rng = np.random.default_rng(fuzz_seed(4242))
    checked = 0
    for trial in range(60 * FUZZ_SCALE):
        ch = int(rng.choice([1, 3]))
        chroma = int(rng.integers(0, 2))
        wmul = 16 if (ch == 3 and chroma == 1) else 8          # includes W % 16 == 8 planes
        hmul = 18 if (ch == 3 and chroma == 1) else 9
        W = wmul * int(rng.integers(1, 40))
        H = hmul * int(rng.integers(1, 30))
        n = int(rng.integers(1, 9))
        d = ds.Downscaler(W, H, ch, chroma=chroma)
        if not d.plan.fused_eligible:
            continue
        band = int(rng.choice([0, 1, 4096, 20000, 100000]))
        d.set_band_bytes(band)
        if rng.random() < 0.5:
            d.set_tuning(int(rng.integers(2, 9)), int(rng.integers(0, 3)))
        fr = synth.random_frames(trial, int(rng.integers(0, 1000)), n, W, H, ch, chroma)
        want = oracle.execute_frames(fr, W, H, ch, chroma)
        x = torch.from_numpy(fr).cuda()
        off = int(rng.choice([0, 0, 16, 1, 3]))
        buf = torch.full((n * d.out_frame_bytes + 64,), 0x5A, dtype=torch.uint8, device="cuda")
        y = buf[off: off + n * d.out_frame_bytes].view(n, -1)
        ds.ds_run(d.handle, x.data_ptr(), n, y.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert d.last_kernel() == FUSED
        _assert_same(y.cpu().numpy(), want, f"trial {trial}: {W}x{H}x{ch} chroma={chroma} n={n} "
                                              f"band={band} off={off}")
        checked += 1
    assert checked >= 30 * FUZZ_SCALE


@pytest.mark.parametrize("kernel,halo,strips", [(FUSED, False, False), (ds.DS_KERNEL_FUSED_GENERAL, False, False),
                                                (ds.DS_KERNEL_FUSED_GENERAL, True, False),
                                                (ds.DS_KERNEL_FUSED_GENERAL, True, True)])
def test_every_unit_processed_exactly_once(kernel, halo, strips):
    """Debug unit accounting (ds_set_debug_counter): over many frame counts,
    band sizes and ring/CTA tunings (K-N1), and automatic or forced run
    lengths (K-N1g with a V halo), the persistent schedule processes every
    work unit exactly once."""
    W, H = 1920, 1080
    spec = ds.make_spec(*_halo_spec(), chroma=ds.DS_CHROMA_420) if halo else None
    d = ds.Downscaler(W, H, 3, spec=spec)
    d.set_kernel(kernel)
    if strips:                                   # units = (frame, plane, column strip, run)
        d.set_general_variant(ds.DS_GENERAL_RUNTIME)
        d.set_general_stage_bytes(6000)
        assert d.plan.general_strips[0] > 1
    L = ds.lib()
    x = ds.generate_frames(40, d.in_frame_bytes, seed=2)
    rng = np.random.default_rng(1)
    for trial in range(12):
        n = int(rng.integers(1, 41))
        if kernel == FUSED and trial % 3 == 1:
            d.set_band_bytes(int(rng.choice([0, 8000, 16000, 64000])))
        if kernel == FUSED and trial % 3 == 2:
            d.set_tuning(int(rng.integers(2, 7)), int(rng.integers(0, 3)))
        if halo:
            d.set_run_bands(int(rng.choice([0, 0, 1, 5, 1 << 20])))
        units = L.ds_units(d.handle, n, kernel)
        assert units > 0
        counts = torch.zeros(units, dtype=torch.int32, device="cuda")
        assert L.ds_set_debug_counter(d.handle, counts.data_ptr()) == 0
        y = d(x[:n])
        torch.cuda.synchronize()
        assert L.ds_set_debug_counter(d.handle, None) == 0
        assert d.last_kernel() == kernel
        c = counts.cpu().numpy()
        assert (c == 1).all(), (trial, n, int((c == 0).sum()), int((c > 1).sum()))
    fr = synth.random_frames(2, 0, n, W, H)
    want = (oracle.execute_frames(fr, W, H, 3, 1, *[_oracle_stage(x) for x in _halo_spec()]) if halo
            else oracle.execute_frames(fr, W, H))
    _assert_same(y.cpu().numpy(), want, "after accounting")
