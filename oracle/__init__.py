"""CPU oracle for the arxiv 1103.4881 downscaler hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The
product path (``paper_1103_4881_b200``) never imports it and shares no code
with it.  The arithmetic lives in ``ds_oracle.c`` (plain C11, one thread);
this module is argument marshalling over ctypes plus the stage tables.

Citations: P:n = PAPER.md line n, S:n = SPEC.md line n (see ds_oracle.c).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ds_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

MAXDIM, MAXPAT, MAXOUT = 4, 16, 8


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc -O2 (no -march=native, no OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "ds_oracle.h"))
    ):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-std=c11", "-O2", "-Wall", "-Wextra", "-fPIC", "-shared", "-o", tmp, _SRC]
        )
        os.replace(tmp, _LIB)
    return _LIB


class Tiler(C.Structure):
    _fields_ = [
        ("ndim", C.c_int32),
        ("shape", C.c_int64 * MAXDIM),
        ("origin", C.c_int64 * MAXDIM),
        ("nrep", C.c_int32),
        ("paving", (C.c_int64 * MAXDIM) * MAXDIM),
        ("npat", C.c_int32),
        ("fitting", (C.c_int64 * MAXDIM) * MAXDIM),
        ("pattern", C.c_int64 * MAXDIM),
    ]


class Stage(C.Structure):
    _fields_ = [
        ("pattern", C.c_int32),
        ("paving", C.c_int32),
        ("origin", C.c_int32),
        ("outputs", C.c_int32),
        ("weight", (C.c_int32 * MAXPAT) * MAXOUT),
        ("divisor", C.c_int32),
        ("bias", C.c_int32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P8 = C.POINTER(C.c_uint8)
        P64 = C.POINTER(C.c_int64)
        PT = C.POINTER(Tiler)
        PS = C.POINTER(Stage)
        L.orc_element_index.argtypes = [PT, P64, P64, P64]
        L.orc_extract_pattern.argtypes = [P8, PT, P64, P8]
        L.orc_write_pattern.argtypes = [P8, PT, P64, P8]
        L.orc_check_coverage.argtypes = [PT, C.c_int32, P64, P64, C.c_int32, C.POINTER(C.c_int32)]
        L.orc_hfilter_8to3.argtypes = [P8, P8]
        L.orc_hfilter_8to3.restype = None
        L.orc_vfilter_9to4.argtypes = [P8, P8]
        L.orc_vfilter_9to4.restype = None
        L.orc_stage_apply.argtypes = [PS, P8, P8]
        L.orc_stage_apply.restype = None
        L.orc_default_stages.argtypes = [PS, PS]
        L.orc_default_stages.restype = None
        L.orc_execute_plane.argtypes = [P8, C.c_int32, C.c_int32, PS, PS, P8, C.c_int32]
        L.orc_execute_plane_mid.argtypes = [P8, C.c_int32, C.c_int32, PS, PS, P8, P8, C.c_int32]
        L.orc_run_task.argtypes = [P8, PT, P8, PT, C.c_int32, P64, PS, C.c_int32]
        L.orc_plane_dims.argtypes = [C.c_int32] * 5 + [C.POINTER(C.c_int32)] * 2
        L.orc_execute_frames.argtypes = [P8, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                         C.c_int32, PS, PS, P8]
        L.orc_direct_plane.argtypes = [P8, C.c_int32, C.c_int32, P8]
        L.orc_direct_frames.argtypes = [P8, C.c_int64] + [C.c_int32] * 4 + [P8]
        L.orc_pixel.argtypes = [P8, C.c_int32, C.c_int32, C.c_int32, C.c_int32]
        _lib = L
    return _lib


def _p8(a: np.ndarray):
    assert a.dtype == np.uint8 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def _p64(seq):
    arr = (C.c_int64 * max(1, len(seq)))(*[int(x) for x in seq])
    return arr


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: oracle error {code}")
        self.code = code


def _check(rc: int, what: str) -> None:
    if rc < 0:
        raise OracleError(rc, what)


# ---------------------------------------------------------------- tilers --
def make_tiler(shape, origin, paving, fitting, pattern) -> Tiler:
    """paving: array dims x repetition dims; fitting: array dims x pattern
    dims.  `pattern` is the pattern shape (may be empty)."""
    t = Tiler()
    t.ndim = len(shape)
    for d, s in enumerate(shape):
        t.shape[d] = s
        t.origin[d] = origin[d]
    t.nrep = len(paving[0]) if len(paving) else 0
    for d in range(len(shape)):
        for j in range(t.nrep):
            t.paving[d][j] = paving[d][j]
    t.npat = len(pattern)
    for d in range(len(shape)):
        for k in range(t.npat):
            t.fitting[d][k] = fitting[d][k]
    for k, s in enumerate(pattern):
        t.pattern[k] = s
    return t


def element_index(t: Tiler, r, f):
    out = (C.c_int64 * MAXDIM)()
    _check(lib().orc_element_index(C.byref(t), _p64(r), _p64(f), out), "element_index")
    return tuple(out[d] for d in range(t.ndim))


def extract_pattern(arr: np.ndarray, t: Tiler, r) -> np.ndarray:
    n = int(np.prod([t.pattern[k] for k in range(t.npat)])) if t.npat else 1
    out = np.zeros(n, np.uint8)
    a = np.ascontiguousarray(arr, dtype=np.uint8)
    _check(lib().orc_extract_pattern(_p8(a), C.byref(t), _p64(r), _p8(out)), "extract_pattern")
    return out


def write_pattern(arr: np.ndarray, t: Tiler, r, pat) -> None:
    assert arr.dtype == np.uint8 and arr.flags.c_contiguous
    p = np.ascontiguousarray(pat, dtype=np.uint8)
    _check(lib().orc_write_pattern(_p8(arr), C.byref(t), _p64(r), _p8(p)), "write_pattern")


def check_coverage(t: Tiler, rep_shape, max_wit: int = 10):
    """Returns ("exact"|"overlaps"|"gaps", [witness linear indices])."""
    wit = (C.c_int64 * max(1, max_wit))()
    nw = C.c_int32(0)
    rc = lib().orc_check_coverage(C.byref(t), len(rep_shape), _p64(rep_shape), wit, max_wit,
                                  C.byref(nw))
    _check(rc, "check_coverage")
    return ("exact", "overlaps", "gaps")[rc], [wit[i] for i in range(nw.value)]


def run_task(arr_in: np.ndarray, tin: Tiler, out_shape, tout: Tiler, rep_shape, body,
             order: int = 0, out_init: np.ndarray | None = None) -> np.ndarray:
    """A general repetitive task executed as S:517-520; body is a
    Stage whose pattern = input pattern elements, outputs = output pattern
    elements.  Elements of out not covered by tout keep out_init (zeros)."""
    a = np.ascontiguousarray(arr_in, dtype=np.uint8)
    out = np.zeros(out_shape, np.uint8) if out_init is None else np.ascontiguousarray(out_init).copy()
    _check(lib().orc_run_task(_p8(a), C.byref(tin), _p8(out), C.byref(tout), len(rep_shape),
                              _p64(rep_shape), C.byref(body), order), "run_task")
    return out


# ---------------------------------------------------------------- stages --
def make_stage(pattern, paving, origin, weights, divisor, bias) -> Stage:
    s = Stage()
    s.pattern, s.paving, s.origin = pattern, paving, origin
    s.outputs = len(weights)
    for k, row in enumerate(weights):
        assert len(row) <= pattern
        for i, w in enumerate(row):
            s.weight[k][i] = w
    s.divisor, s.bias = divisor, bias
    return s


def default_stages():
    h, v = Stage(), Stage()
    lib().orc_default_stages(C.byref(h), C.byref(v))
    return h, v


def stage_to_dict(s: Stage) -> dict:
    return dict(pattern=s.pattern, paving=s.paving, origin=s.origin,
                weights=[[s.weight[k][i] for i in range(s.pattern)] for k in range(s.outputs)],
                divisor=s.divisor, bias=s.bias)


def stage_from_dict(d: dict) -> Stage:
    return make_stage(d["pattern"], d["paving"], d["origin"], d["weights"], d["divisor"], d["bias"])


def hfilter_8to3(pat) -> np.ndarray:
    i = np.ascontiguousarray(pat, dtype=np.uint8)
    o = np.zeros(3, np.uint8)
    lib().orc_hfilter_8to3(_p8(i), _p8(o))
    return o


def vfilter_9to4(pat) -> np.ndarray:
    i = np.ascontiguousarray(pat, dtype=np.uint8)
    o = np.zeros(4, np.uint8)
    lib().orc_vfilter_9to4(_p8(i), _p8(o))
    return o


def stage_apply(s: Stage, pat) -> np.ndarray:
    i = np.zeros(MAXPAT, np.uint8)
    i[: len(pat)] = np.asarray(pat, dtype=np.uint8)
    o = np.zeros(MAXOUT, np.uint8)
    lib().orc_stage_apply(C.byref(s), _p8(i), _p8(o))
    return o[: s.outputs].copy()


# ---------------------------------------------------------------- planes --
def plane_dims(W, H, channels=3, chroma=1):
    dims = []
    for p in range(channels):
        pw, ph = C.c_int32(), C.c_int32()
        _check(lib().orc_plane_dims(W, H, channels, chroma, p, C.byref(pw), C.byref(ph)),
               "plane_dims")
        dims.append((pw.value, ph.value))
    return dims


def out_plane_dims(W, H, channels=3, chroma=1, h: Stage | None = None, v: Stage | None = None):
    if h is None:
        h, v = default_stages()
    return [(h.outputs * (pw // h.paving), v.outputs * (ph // v.paving))
            for pw, ph in plane_dims(W, H, channels, chroma)]


def frame_bytes(W, H, channels=3, chroma=1, h=None, v=None):
    fin = sum(pw * ph for pw, ph in plane_dims(W, H, channels, chroma))
    fout = sum(ow * oh for ow, oh in out_plane_dims(W, H, channels, chroma, h, v))
    return fin, fout


def execute_plane(plane: np.ndarray, h: Stage | None = None, v: Stage | None = None,
                  order: int = 0) -> np.ndarray:
    """O1 on one (H, W) u8 plane."""
    if h is None:
        h, v = default_stages()
    Hh, W = plane.shape
    a = np.ascontiguousarray(plane, dtype=np.uint8)
    if W % h.paving or Hh % v.paving:
        raise OracleError(-2, "execute_plane")
    out = np.zeros((v.outputs * (Hh // v.paving), h.outputs * (W // h.paving)), np.uint8)
    _check(lib().orc_execute_plane(_p8(a), W, Hh, C.byref(h), C.byref(v), _p8(out), order),
           "execute_plane")
    return out


def execute_plane_mid(plane: np.ndarray, h: Stage | None = None, v: Stage | None = None):
    """O1 on one plane, returning (Mid, Out): Mid is the H task's u8 output
    array, the array the paper's unfused kernels keep in global memory."""
    if h is None:
        h, v = default_stages()
    Hh, W = plane.shape
    a = np.ascontiguousarray(plane, dtype=np.uint8)
    if W % h.paving or Hh % v.paving:
        raise OracleError(-2, "execute_plane_mid")
    mid = np.zeros((Hh, h.outputs * (W // h.paving)), np.uint8)
    out = np.zeros((v.outputs * (Hh // v.paving), h.outputs * (W // h.paving)), np.uint8)
    _check(lib().orc_execute_plane_mid(_p8(a), W, Hh, C.byref(h), C.byref(v), _p8(mid), _p8(out),
                                       0), "execute_plane_mid")
    return mid, out


def execute_frames_mid(frames: np.ndarray, W, H, channels=3, chroma=1,
                       h: Stage | None = None, v: Stage | None = None):
    """O1 over a stream returning (mids, outs); mids is (n, mid_frame_bytes)
    with the planes' Mid arrays back to back (same layout rule as S:583)."""
    if h is None:
        h, v = default_stages()
    fin, fout = frame_bytes(W, H, channels, chroma, h, v)
    a = np.ascontiguousarray(frames, dtype=np.uint8).reshape(-1, fin)
    dims = plane_dims(W, H, channels, chroma)
    fmid = sum(ph * h.outputs * (pw // h.paving) for pw, ph in dims)
    mids = np.zeros((a.shape[0], fmid), np.uint8)
    outs = np.zeros((a.shape[0], fout), np.uint8)
    for f in range(a.shape[0]):
        ip = split_planes(a[f], W, H, channels, chroma)
        mo = oo = 0
        for (pw, ph), pl in zip(dims, ip):
            m, o = execute_plane_mid(pl, h, v)
            mids[f, mo: mo + m.size] = m.ravel()
            outs[f, oo: oo + o.size] = o.ravel()
            mo += m.size
            oo += o.size
    return mids, outs


def execute_frames(frames: np.ndarray, W, H, channels=3, chroma=1,
                   h: Stage | None = None, v: Stage | None = None) -> np.ndarray:
    """O1 over a stream: frames is (n, in_frame_bytes) u8."""
    if h is None:
        h, v = default_stages()
    fin, fout = frame_bytes(W, H, channels, chroma, h, v)
    a = np.ascontiguousarray(frames, dtype=np.uint8).reshape(-1, fin)
    out = np.zeros((a.shape[0], fout), np.uint8)
    _check(lib().orc_execute_frames(_p8(a), a.shape[0], W, H, channels, chroma, C.byref(h),
                                    C.byref(v), _p8(out)), "execute_frames")
    return out


def direct_plane(plane: np.ndarray) -> np.ndarray:
    """O2 on one plane (default taps)."""
    Hh, W = plane.shape
    a = np.ascontiguousarray(plane, dtype=np.uint8)
    if W % 8 or Hh % 9:
        raise OracleError(-2, "direct_plane")
    out = np.zeros((Hh // 9 * 4, W // 8 * 3), np.uint8)
    _check(lib().orc_direct_plane(_p8(a), W, Hh, _p8(out)), "direct_plane")
    return out


def direct_frames(frames: np.ndarray, W, H, channels=3, chroma=1) -> np.ndarray:
    fin, fout = frame_bytes(W, H, channels, chroma)
    a = np.ascontiguousarray(frames, dtype=np.uint8).reshape(-1, fin)
    out = np.zeros((a.shape[0], fout), np.uint8)
    _check(lib().orc_direct_frames(_p8(a), a.shape[0], W, H, channels, chroma, _p8(out)),
           "direct_frames")
    return out


def pixel(plane: np.ndarray, R: int, Cc: int) -> int:
    """O3: one output pixel of a plane from its closed form."""
    Hh, W = plane.shape
    a = np.ascontiguousarray(plane, dtype=np.uint8)
    rc = lib().orc_pixel(_p8(a), W, Hh, R, Cc)
    _check(rc, "pixel")
    return rc


def split_planes(frame: np.ndarray, W, H, channels=3, chroma=1, out=False, h=None, v=None):
    """View one flat frame (in or out layout) as its list of 2-D planes."""
    dims = out_plane_dims(W, H, channels, chroma, h, v) if out else plane_dims(W, H, channels,
                                                                                chroma)
    planes, off = [], 0
    for pw, ph in dims:
        planes.append(frame[off: off + pw * ph].reshape(ph, pw))
        off += pw * ph
    return planes
