"""The seeded input generator (synth/): the C and numpy forms agree byte for
byte, and splitmix64 is the published SplitMix64 (first outputs from state 0
are 0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F)."""
import numpy as np

import synth


def test_splitmix64_known_values():
    # state 0: outputs k = 1, 2, 3 are mix(k * golden), i.e. splitmix64((k - 1) * golden)
    g = int(synth.GOLDEN)
    xs = np.array([0, g, (2 * g) % (1 << 64)], dtype=np.uint64)
    got = [int(v) for v in synth.splitmix64(xs)]
    assert got == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_c_generator_matches_numpy():
    assert synth._clib() is not None, "libsynth.so did not build"
    rng = np.random.default_rng(0)
    for seed in (0, 1, 5, 2**63 + 7):
        for start in (0, 1, 12345, 3_110_400 * 2999, 2**40 + 3):
            n = int(rng.integers(1, 5000))
            a = synth.random_bytes(seed, start, n)
            b = synth.random_bytes_numpy(seed, start, n)
            assert np.array_equal(a, b), (seed, start, n)


def test_frames_are_slices_of_one_stream():
    W, H = 64, 36
    a = synth.random_frames(3, 0, 5, W, H)
    b = synth.random_frames(3, 2, 2, W, H)
    assert np.array_equal(a[2:4], b)
    buf = np.empty((2, a.shape[1]), np.uint8)
    synth.random_frames(3, 2, 2, W, H, out=buf)
    assert np.array_equal(buf, b)
