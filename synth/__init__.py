"""Seeded synthetic frame generators shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no filter, no tiler): it
only produces input bytes.  It is the one module both `oracle/`-based tests
and the product-side tests/bench may import (task rule 3).

Random frames use a counter-based hash over the byte's index in the
*unsharded* stream, so any shard (any GPU, or the host) regenerates
identical bytes:

    byte(seed, i) = splitmix64(seed * 0x9E3779B97F4A7C15 + i) >> 56

`splitmix64` is Steele/Lea/Flood's SplitMix64 finaliser.  The CUDA library
implements the same generator on the device (`ds_generate`); the parity
tests compare the two byte for byte.

Frame layout: planes Y, plane 1, plane 2 back to back, row-major
u8, no headers; 4:2:0 chroma planes are (W/2, H/2).
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64, copy=True) + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


_CLIB = None


def build(force: bool = False) -> str:
    """Compile synth_gen.c (the same generator in C) to libsynth.so."""
    import os
    import subprocess

    here = os.path.dirname(os.path.abspath(__file__))
    src, so = os.path.join(here, "synth_gen.c"), os.path.join(here, "libsynth.so")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        tmp = so + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-o", tmp, src])
        os.replace(tmp, so)
    return so


def _clib():
    """libsynth.so, built on first use; None if no C compiler is at hand
    (then the numpy generator below serves alone)."""
    global _CLIB
    if _CLIB is None:
        import ctypes

        try:
            L = ctypes.CDLL(build())
            L.synth_random_bytes.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                             ctypes.c_void_p]
            L.synth_random_bytes.restype = None
            _CLIB = L
        except Exception:
            _CLIB = False
    return _CLIB or None


def random_bytes_numpy(seed: int, start: int, count: int, chunk: int = 1 << 24) -> np.ndarray:
    """Bytes i = start .. start+count-1 of the seeded stream (numpy form)."""
    out = np.empty(count, np.uint8)
    with np.errstate(over="ignore"):
        base = np.uint64(seed) * GOLDEN
        for lo in range(0, count, chunk):
            n = min(chunk, count - lo)
            idx = np.arange(start + lo, start + lo + n, dtype=np.uint64) + base
            out[lo: lo + n] = (splitmix64(idx) >> np.uint64(56)).astype(np.uint8)
    return out


def random_bytes(seed: int, start: int, count: int, out: np.ndarray | None = None) -> np.ndarray:
    """Bytes i = start .. start+count-1 of the seeded stream (C when built,
    else numpy; the two are byte-identical)."""
    if out is None:
        out = np.empty(count, np.uint8)
    L = _clib()
    if L is None:
        out[:] = random_bytes_numpy(seed, start, count)
        return out
    assert out.dtype == np.uint8 and out.flags.c_contiguous and out.size == count
    L.synth_random_bytes(seed % (1 << 64), start, count, out.ctypes.data)
    return out


def plane_dims(W: int, H: int, channels: int = 3, chroma: int = 1):
    """(w, h) of each plane; chroma 1 = 4:2:0, 0 = 4:4:4 (layout only)."""
    if channels == 1:
        return [(W, H)]
    if chroma == 1:
        return [(W, H), (W // 2, H // 2), (W // 2, H // 2)]
    return [(W, H)] * 3


def in_frame_bytes(W: int, H: int, channels: int = 3, chroma: int = 1) -> int:
    return sum(w * h for w, h in plane_dims(W, H, channels, chroma))


def random_frames(seed: int, first_frame: int, n: int, W: int, H: int, channels: int = 3,
                  chroma: int = 1, out: np.ndarray | None = None) -> np.ndarray:
    """Frames first_frame .. first_frame+n-1 of the seeded stream, (n, frame_bytes)."""
    fb = in_frame_bytes(W, H, channels, chroma)
    flat = None if out is None else out.reshape(-1)
    return random_bytes(seed, first_frame * fb, n * fb, out=flat).reshape(n, fb)


def _assemble(planes_fn, n, W, H, channels, chroma):
    fb = in_frame_bytes(W, H, channels, chroma)
    out = np.empty((n, fb), np.uint8)
    for f in range(n):
        off = 0
        for p, (w, h) in enumerate(plane_dims(W, H, channels, chroma)):
            y, x = np.mgrid[0:h, 0:w]
            out[f, off: off + w * h] = (planes_fn(f, p, y, x) & 255).astype(np.uint8).ravel()
            off += w * h
    return out


def constant_frames(value: int, n: int, W: int, H: int, channels: int = 3, chroma: int = 1):
    return np.full((n, in_frame_bytes(W, H, channels, chroma)), value, np.uint8)


def checkerboard_frames(n, W, H, channels=3, chroma=1):
    """255 where (x + y) is odd, else 0."""
    return _assemble(lambda f, p, y, x: ((x + y) & 1) * 255, n, W, H, channels, chroma)


def ramp_frames(n, W, H, channels=3, chroma=1, seed=0):
    """Video-like moving ramp (x + 2y + 3n + 5*plane) & 255 with +-2 hash noise."""
    noise = random_frames(seed, 0, n, W, H, channels, chroma).astype(np.int64) % 5 - 2

    def fn(f, p, y, x):
        return x + 2 * y + 3 * f + 5 * p

    base = _assemble(fn, n, W, H, channels, chroma).astype(np.int64)
    return np.clip(base + noise, 0, 255).astype(np.uint8)


def linear_frames(n, W, H, channels=3, chroma=1, a=7, b=3):
    """In[y][x] = (a*y + b*x) mod 256 per plane (Appendix B family)."""
    return _assemble(lambda f, p, y, x: a * y + b * x, n, W, H, channels, chroma)
