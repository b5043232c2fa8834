"""Python binding of libds.so (include/ds.h): the B200 downscaler of
arxiv 1103.4881.

Argument marshalling only -- every step of the hot path runs in the CUDA
kernels of ``csrc/``.  Functions keep the C names (``ds_create``,
``ds_run``, ...); ``Downscaler`` wraps them for ``torch.uint8`` CUDA
tensors, using PyTorch only for device memory and streams.  There is no CPU
fallback: if libds.so is missing or cannot be built this module raises.

Citation key: P:n = PAPER.md line n, S:n = SPEC.md line n.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from . import _build

DS_OK, DS_EINVAL, DS_ESHAPE, DS_EUNSUPPORTED, DS_ECUDA, DS_ENOMEM = 0, -1, -2, -3, -4, -5
DS_CHROMA_444, DS_CHROMA_420 = 0, 1
DS_KERNEL_AUTO, DS_KERNEL_FUSED, DS_KERNEL_GENERIC, DS_KERNEL_FUSED_GENERAL = 0, 1, 2, 3
DS_GENERAL_AUTO, DS_GENERAL_RUNTIME, DS_GENERAL_COMPILED = 0, 1, 2
VARIANT_NAMES = {0: None, 1: "runtime taps (ds_general.cuh)", 2: "compiled taps, built-in (K-N1s, ds_spec.cuh)",
                 3: "compiled taps, NVRTC (K-N1s, ds_spec.cuh)"}
DS_MAX_PATTERN, DS_MAX_OUTPUTS, DS_MAX_PLANES = 16, 8, 3
KERNEL_NAMES = {DS_KERNEL_AUTO: "none", DS_KERNEL_FUSED: "K-N1 fused band (TMA ring)",
                DS_KERNEL_GENERIC: "K-N2 generic",
                DS_KERNEL_FUSED_GENERAL: "K-N1g fused band, any spec (variant: runtime taps or K-N1s)"}


class ds_stage_spec(C.Structure):
    _fields_ = [
        ("pattern", C.c_int32),
        ("paving", C.c_int32),
        ("origin", C.c_int32),
        ("outputs", C.c_int32),
        ("weight", (C.c_int32 * DS_MAX_PATTERN) * DS_MAX_OUTPUTS),
        ("divisor", C.c_int32),
        ("bias", C.c_int32),
    ]


class ds_filter_spec(C.Structure):
    _fields_ = [("h", ds_stage_spec), ("v", ds_stage_spec), ("chroma", C.c_int32)]


class ds_plan_info(C.Structure):
    _fields_ = [
        ("in_frame_bytes", C.c_int64),
        ("out_frame_bytes", C.c_int64),
        ("n_planes", C.c_int32),
        ("in_w", C.c_int32 * DS_MAX_PLANES),
        ("in_h", C.c_int32 * DS_MAX_PLANES),
        ("out_w", C.c_int32 * DS_MAX_PLANES),
        ("out_h", C.c_int32 * DS_MAX_PLANES),
        ("in_offset", C.c_int64 * DS_MAX_PLANES),
        ("out_offset", C.c_int64 * DS_MAX_PLANES),
        ("fused_eligible", C.c_int32),
        ("band_groups", C.c_int32 * DS_MAX_PLANES),
        ("units_per_frame", C.c_int64),
        ("unit_in_bytes_max", C.c_int64),
        ("unit_out_bytes_max", C.c_int64),
        ("fused_general_eligible", C.c_int32),
        ("general_band_reps", C.c_int32 * DS_MAX_PLANES),
        ("general_units_per_frame", C.c_int64),
        ("general_stage_bytes_max", C.c_int64),
        ("general_strips", C.c_int32 * 3),
    ]


class ds_schedule_stats(C.Structure):
    _fields_ = [
        ("frames", C.c_int64),
        ("h2d_count", C.c_int64),
        ("d2h_count", C.c_int64),
        ("h2d_bytes", C.c_int64),
        ("d2h_bytes", C.c_int64),
        ("launches", C.c_int64),
        ("h2d_ms", C.c_double),
        ("d2h_ms", C.c_double),
        ("kernel_ms", C.c_double),
        ("kernel_ms_plane", C.c_double * DS_MAX_PLANES),
        ("total_ms", C.c_double),
    ]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "kernel_ms_plane"}
        d["kernel_ms_plane"] = list(self.kernel_ms_plane)
        return d


class ds_tiler(C.Structure):
    _fields_ = [
        ("ndim", C.c_int32),
        ("shape", C.c_int64 * 4),
        ("origin", C.c_int64 * 4),
        ("nrep", C.c_int32),
        ("paving", (C.c_int64 * 4) * 4),
        ("npat", C.c_int32),
        ("fitting", (C.c_int64 * 4) * 4),
        ("pattern", C.c_int64 * 4),
    ]


class ds_task_body(C.Structure):
    _fields_ = [
        ("n_in", C.c_int32),
        ("n_out", C.c_int32),
        ("weight", (C.c_int32 * DS_MAX_PATTERN) * DS_MAX_OUTPUTS),
        ("divisor", C.c_int32),
        ("bias", C.c_int32),
    ]


class ds_launch(C.Structure):
    _fields_ = [
        ("kernel", C.c_int32),
        ("grid", C.c_int32),
        ("block", C.c_int32),
        ("smem_bytes", C.c_int32),
        ("stages", C.c_int32),
        ("ctas_per_sm", C.c_int32),
        ("consumer_warps", C.c_int32),
        ("units", C.c_int64),
        ("unit_in_bytes_max", C.c_int64),
        ("variant", C.c_int32),
        ("reserved_", C.c_int32),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved_"}


class ds_topology(C.Structure):
    _fields_ = [
        ("ndim", C.c_int32),
        ("multiplicity", C.c_int64 * 3),
        ("local", C.c_int32 * 3),
        ("global_", C.c_int64 * 3),
        ("guarded", C.c_int32),
    ]

    def as_dict(self):
        n = self.ndim
        return dict(multiplicity=list(self.multiplicity[:n]), local=list(self.local[:n]),
                    global_=list(self.global_[:n]), guarded=bool(self.guarded))


DS_TOPO_FLAT, DS_TOPO_SPEC = 0, 1

DS_SCHED_NAIVE, DS_SCHED_OPTIMIZED, DS_SCHED_FUSED, DS_SCHED_STREAMED = 0, 1, 2, 3
SCHED_NAMES = {DS_SCHED_NAIVE: "naive", DS_SCHED_OPTIMIZED: "optimized", DS_SCHED_FUSED: "fused",
               DS_SCHED_STREAMED: "streamed"}


class DSError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: {ds_strerror(code)} ({code})")
        self.code = code


_lib = None
_lock = threading.Lock()

# (name, restype, argtypes) of every entry point declared in include/ds.h
_P8 = C.POINTER(C.c_uint8)
_PI32 = C.POINTER(C.c_int32)
SIGNATURES = [
    ("ds_default_spec", C.c_int, [C.POINTER(ds_filter_spec)]),
    ("ds_plan", C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(ds_filter_spec),
                          C.POINTER(ds_plan_info)]),
    ("ds_create", C.c_void_p, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(ds_filter_spec)]),
    ("ds_run", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    ("ds_enable_peer", C.c_int, [C.c_void_p, C.c_int32]),
    ("ds_run_host", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    ("ds_set_host_chunk", C.c_int, [C.c_void_p, C.c_int64]),
    ("ds_destroy", None, [C.c_void_p]),
    ("ds_last_error", C.c_int, []),
    ("ds_strerror", C.c_char_p, [C.c_int]),
    ("ds_in_frame_bytes", C.c_int64, [C.c_void_p]),
    ("ds_out_frame_bytes", C.c_int64, [C.c_void_p]),
    ("ds_get_plan", C.c_int, [C.c_void_p, C.POINTER(ds_plan_info)]),
    ("ds_plane_dims", C.c_int, [C.c_void_p, C.c_int, _PI32, _PI32, _PI32, _PI32]),
    ("ds_set_kernel", C.c_int, [C.c_void_p, C.c_int32]),
    ("ds_set_general_variant", C.c_int, [C.c_void_p, C.c_int32]),
    ("ds_last_variant", C.c_int, [C.c_void_p]),
    ("ds_last_kernel", C.c_int, [C.c_void_p]),
    ("ds_set_tuning", C.c_int, [C.c_void_p, C.c_int32, C.c_int32]),
    ("ds_set_band_bytes", C.c_int, [C.c_void_p, C.c_int64]),
    ("ds_set_run_bands", C.c_int, [C.c_void_p, C.c_int32]),
    ("ds_set_general_stage_bytes", C.c_int, [C.c_void_p, C.c_int64]),
    ("ds_launch_shape", C.c_int, [C.c_void_p, C.c_int64, _PI32, _PI32, _PI32]),
    ("ds_launch_info", C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.POINTER(ds_launch)]),
    ("ds_mid_frame_bytes", C.c_int64, [C.c_void_p]),
    ("ds_run_htask", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_int32,
                               C.c_void_p]),
    ("ds_run_vtask", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_int32,
                               C.c_void_p]),
    ("ds_schedule_plan", C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(ds_filter_spec),
                                   C.c_int32, C.POINTER(ds_schedule_stats)]),
    ("ds_run_schedule", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32,
                                  C.POINTER(ds_schedule_stats), C.c_void_p]),
    ("ds_compute_topology", C.c_int, [C.c_int32, C.POINTER(C.c_int64), C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.POINTER(ds_topology)]),
    ("ds_run_task", C.c_int, [C.c_void_p, C.POINTER(ds_tiler), C.c_void_p, C.POINTER(ds_tiler), C.c_int32,
                              C.POINTER(C.c_int64), C.POINTER(ds_task_body), C.c_int32, C.c_void_p]),
    ("ds_tiler_coverage", C.c_int, [C.POINTER(ds_tiler), C.c_int32, C.POINTER(C.c_int64),
                                    C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_void_p]),
    ("ds_set_debug_counter", C.c_int, [C.c_void_p, C.c_void_p]),
    ("ds_units", C.c_int64, [C.c_void_p, C.c_int64, C.c_int32]),
    ("ds_generate", C.c_int, [C.c_void_p, C.c_int64, C.c_uint64, C.c_int64, C.c_void_p]),
]


def lib():
    """Load (building in-tree first if stale) libds.so.  Raises if it cannot."""
    global _lib
    with _lock:
        if _lib is None:
            path = _build.LIB
            if _build.stale():
                try:
                    _build.build()
                except Exception as e:  # no silent fallback: the CUDA path is the product
                    if not os.path.exists(path):
                        raise ImportError(f"libds.so is missing and could not be built: {e}")
            L = C.CDLL(path)
            for name, res, args in SIGNATURES:
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def lib_path() -> str:
    return _build.LIB


# ----------------------------------------------------------- thin C names --
def ds_strerror(code: int) -> str:
    return lib().ds_strerror(code).decode()


def ds_last_error() -> int:
    return lib().ds_last_error()


def _stage_from(d) -> ds_stage_spec:
    if isinstance(d, ds_stage_spec):
        return d
    s = ds_stage_spec()
    s.pattern, s.paving, s.origin = d["pattern"], d["paving"], d.get("origin", 0)
    s.outputs = len(d["weights"])
    for k, row in enumerate(d["weights"]):
        for i, w in enumerate(row):
            s.weight[k][i] = int(w)
    s.divisor, s.bias = d["divisor"], d["bias"]
    return s


def make_spec(h=None, v=None, chroma: int = DS_CHROMA_420) -> ds_filter_spec:
    """Build a ds_filter_spec from dicts {pattern, paving, origin, weights
    (Q rows of <= P ints), divisor, bias}; None = SPEC's stage."""
    spec = ds_default_spec()
    if h is not None:
        spec.h = _stage_from(h)
    if v is not None:
        spec.v = _stage_from(v)
    spec.chroma = chroma
    return spec


def stage_to_dict(s: ds_stage_spec) -> dict:
    return dict(pattern=s.pattern, paving=s.paving, origin=s.origin,
                weights=[[s.weight[k][i] for i in range(s.pattern)] for k in range(s.outputs)],
                divisor=s.divisor, bias=s.bias)


def ds_default_spec() -> ds_filter_spec:
    s = ds_filter_spec()
    rc = lib().ds_default_spec(C.byref(s))
    if rc:
        raise DSError(rc, "ds_default_spec")
    return s


def ds_plan(frame_w: int, frame_h: int, channels: int = 3, spec: ds_filter_spec | None = None):
    info = ds_plan_info()
    rc = lib().ds_plan(frame_w, frame_h, channels, C.byref(spec) if spec is not None else None,
                       C.byref(info))
    if rc:
        raise DSError(rc, "ds_plan")
    return info


def ds_schedule_plan(frame_w: int, frame_h: int, channels: int, schedule: int,
                     spec: ds_filter_spec | None = None) -> dict:
    st = ds_schedule_stats()
    rc = lib().ds_schedule_plan(frame_w, frame_h, channels,
                                C.byref(spec) if spec is not None else None, schedule, C.byref(st))
    if rc:
        raise DSError(rc, "ds_schedule_plan")
    return st.as_dict()


def ds_create(frame_w: int, frame_h: int, channels: int = 3, spec: ds_filter_spec | None = None):
    h = lib().ds_create(frame_w, frame_h, channels,
                        C.byref(spec) if spec is not None else None)
    if not h:
        raise DSError(lib().ds_last_error(), "ds_create")
    return h


def ds_run(h, in_ptr: int, n_frames: int, out_ptr: int, stream: int = 0) -> None:
    rc = lib().ds_run(h, in_ptr, n_frames, out_ptr, stream or None)
    if rc:
        raise DSError(rc, "ds_run")


def ds_run_host(h, in_ptr: int, n_frames: int, out_ptr: int, stream: int = 0) -> None:
    rc = lib().ds_run_host(h, in_ptr, n_frames, out_ptr, stream or None)
    if rc:
        raise DSError(rc, "ds_run_host")


def ds_destroy(h) -> None:
    lib().ds_destroy(h)


def ds_generate(dev_ptr: int, n_bytes: int, seed: int, start_index: int, stream: int = 0) -> None:
    rc = lib().ds_generate(dev_ptr, n_bytes, seed, start_index, stream or None)
    if rc:
        raise DSError(rc, "ds_generate")


# ------------------------------------------------- general tasks --
def make_tiler(shape, origin, paving, fitting, pattern) -> ds_tiler:
    """Array-OL tiler: paving is array dims x repetition dims,
    fitting array dims x pattern dims, pattern the pattern shape."""
    t = ds_tiler()
    t.ndim = len(shape)
    for d, x in enumerate(shape):
        t.shape[d] = x
        t.origin[d] = origin[d]
    t.nrep = len(paving[0]) if len(paving) else 0
    t.npat = len(pattern)
    for d in range(len(shape)):
        for j in range(t.nrep):
            t.paving[d][j] = paving[d][j]
        for k in range(t.npat):
            t.fitting[d][k] = fitting[d][k]
    for k, x in enumerate(pattern):
        t.pattern[k] = x
    return t


def make_body(weights, divisor=1, bias=0, n_in=None) -> ds_task_body:
    b = ds_task_body()
    b.n_out = len(weights)
    b.n_in = n_in if n_in is not None else max(len(r) for r in weights)
    for k, row in enumerate(weights):
        for i, w in enumerate(row):
            b.weight[k][i] = int(w)
    b.divisor, b.bias = divisor, bias
    return b


def _i64(seq):
    return (C.c_int64 * max(1, len(seq)))(*[int(x) for x in seq])


def ds_compute_topology(multiplicity, max_wg=1024, max_dims=3, min_items=64, wg_threshold=256) -> dict:
    t = ds_topology()
    rc = lib().ds_compute_topology(len(multiplicity), _i64(multiplicity), max_wg, max_dims, min_items,
                                   wg_threshold, C.byref(t))
    if rc:
        raise DSError(rc, "ds_compute_topology")
    return t.as_dict()


def run_task(x, t_in: ds_tiler, out, t_out: ds_tiler, rep_shape, body: ds_task_body,
             policy: int = DS_TOPO_FLAT, stream=None):
    """One repetitive task on torch uint8 CUDA tensors x -> out (in place)."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    rc = lib().ds_run_task(x.data_ptr(), C.byref(t_in), out.data_ptr(), C.byref(t_out), len(rep_shape),
                           _i64(rep_shape), C.byref(body), policy, s.cuda_stream)
    if rc:
        raise DSError(rc, "ds_run_task")
    return out


def tiler_coverage(t: ds_tiler, rep_shape, stream=None):
    """("exact"|"overlaps"|"gaps", n_overlapping_elements, n_gap_elements), on the device."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    ov, gp = C.c_int64(), C.c_int64()
    rc = lib().ds_tiler_coverage(C.byref(t), len(rep_shape), _i64(rep_shape), C.byref(ov), C.byref(gp),
                                 s.cuda_stream)
    if rc:
        raise DSError(rc, "ds_tiler_coverage")
    kind = "overlaps" if ov.value else ("gaps" if gp.value else "exact")
    return kind, ov.value, gp.value


# ------------------------------------------------------------ torch facade --
def _torch_uint8():
    import torch

    return torch.uint8


def _current_raw_stream(device_index):
    """cudaStream_t of torch's current stream on the device (the raw query
    when this torch has it: ~10x cheaper than torch.cuda.current_stream())."""
    import torch

    f = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if f is not None:
        return f(device_index)
    return torch.cuda.current_stream(device_index).cuda_stream


def _check_u8(t, what: str, cuda: bool, numel: int | None = None, unit: int | None = None) -> int:
    """Argument checks shared by the facade's calls: a contiguous uint8 tensor
    on the right side of the bus, holding a whole number of `unit`-byte
    frames (returns that number) and, if given, exactly `numel` elements."""
    if t.dtype is not _torch_uint8() or bool(t.is_cuda) != cuda or not t.is_contiguous():
        raise ValueError(f"{what} must be a contiguous {'CUDA' if cuda else 'CPU'} torch.uint8 tensor")
    n = t.numel()
    if numel is not None and n != numel:
        raise ValueError(f"{what} holds {n} bytes, expected {numel}")
    if unit is not None:
        if n % unit:
            raise ValueError(f"{what} does not hold a whole number of {unit}-byte frames")
        return n // unit
    return n


class Downscaler:
    """``Downscaler(w, h, channels=3, chroma="420", spec=None)(frames)``.

    frames: ``torch.uint8`` CUDA tensor holding n whole frames (shape
    ``(n, in_frame_bytes)`` or anything with n*in_frame_bytes elements,
    contiguous).  Returns (or fills ``out``) ``(n, out_frame_bytes)``.
    Runs on ``torch.cuda.current_stream()``.
    """

    def __init__(self, w: int, h: int, channels: int = 3, chroma: str | int | None = None,
                 spec: ds_filter_spec | None = None, kernel: int = DS_KERNEL_AUTO):
        """chroma: "420" / "444" / DS_CHROMA_*; None = the spec's own (4:2:0 by default)."""
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("Downscaler needs a CUDA device (no CPU fallback)")
        if spec is None:
            spec = ds_default_spec()
        else:
            spec = ds_filter_spec.from_buffer_copy(spec)
        if chroma is not None:
            spec.chroma = chroma if isinstance(chroma, int) else {
                "420": DS_CHROMA_420, "444": DS_CHROMA_444}[str(chroma)]
        self.spec = spec
        self.w, self.h, self.channels = w, h, channels
        self.device = torch.cuda.current_device()
        self._h = ds_create(w, h, channels, spec)       # loads libds.so (module-level _lib)
        self.in_frame_bytes = lib().ds_in_frame_bytes(self._h)
        self.out_frame_bytes = lib().ds_out_frame_bytes(self._h)
        self.plan = self.get_plan()
        if kernel != DS_KERNEL_AUTO:
            self.set_kernel(kernel)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                ds_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def plane_dims(self):
        out = []
        for p in range(self.channels):
            a, b, c, d = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
            rc = lib().ds_plane_dims(self._h, p, C.byref(a), C.byref(b), C.byref(c), C.byref(d))
            if rc:
                raise DSError(rc, "ds_plane_dims")
            out.append(((a.value, b.value), (c.value, d.value)))
        return out

    def enable_peer(self, peer_device: int) -> None:
        """ds_enable_peer: let ds_run store its output on GPU ``peer_device``
        (a buffer mapped from another rank, the fused gather of dist.py)."""
        rc = lib().ds_enable_peer(self._h, int(peer_device))
        if rc:
            raise DSError(rc, "ds_enable_peer")

    def set_kernel(self, kernel: int) -> None:
        rc = lib().ds_set_kernel(self._h, kernel)
        if rc:
            raise DSError(rc, "ds_set_kernel")

    def last_kernel(self) -> int:
        return lib().ds_last_kernel(self._h)

    def set_general_variant(self, variant: int) -> None:
        """K-N1g variant: DS_GENERAL_AUTO, _RUNTIME (taps as data) or _COMPILED (K-N1s)."""
        rc = lib().ds_set_general_variant(self._h, variant)
        if rc:
            raise DSError(rc, "ds_set_general_variant")

    def last_variant(self) -> int:
        return lib().ds_last_variant(self._h)

    def set_tuning(self, stages: int, ctas_per_sm: int = 0) -> None:
        rc = lib().ds_set_tuning(self._h, stages, ctas_per_sm)
        if rc:
            raise DSError(rc, "ds_set_tuning")

    def set_band_bytes(self, target: int) -> None:
        rc = lib().ds_set_band_bytes(self._h, target)
        if rc:
            raise DSError(rc, "ds_set_band_bytes")
        self.plan = self.get_plan()

    def set_run_bands(self, bands: int) -> None:
        """K-N1g: bands per run when the V stage has a halo (0 = automatic)."""
        rc = lib().ds_set_run_bands(self._h, bands)
        if rc:
            raise DSError(rc, "ds_set_run_bands")

    def set_general_stage_bytes(self, target: int) -> None:
        """K-N1g: staged bytes per band (0 = default); wide planes split into column strips."""
        rc = lib().ds_set_general_stage_bytes(self._h, target)
        if rc:
            raise DSError(rc, "ds_set_general_stage_bytes")
        self.plan = self.get_plan()

    def get_plan(self):
        info = ds_plan_info()
        rc = lib().ds_get_plan(self._h, C.byref(info))
        if rc:
            raise DSError(rc, "ds_get_plan")
        return info

    def set_host_chunk(self, frames: int) -> None:
        rc = lib().ds_set_host_chunk(self._h, frames)
        if rc:
            raise DSError(rc, "ds_set_host_chunk")

    def launch_shape(self, n_frames: int):
        g, b, s = C.c_int32(), C.c_int32(), C.c_int32()
        rc = lib().ds_launch_shape(self._h, n_frames, C.byref(g), C.byref(b), C.byref(s))
        if rc:
            raise DSError(rc, "ds_launch_shape")
        return g.value, b.value, s.value

    def launch_info(self, n_frames: int, kernel: int | None = None) -> dict:
        """ds_launch_info for `kernel` (default: the kernel of the last ds_run)."""
        li = ds_launch()
        k = self.last_kernel() if kernel is None else kernel
        rc = lib().ds_launch_info(self._h, n_frames, k, C.byref(li))
        if rc:
            raise DSError(rc, "ds_launch_info")
        return li.as_dict()

    # ---- the paper's unfused structure / schedules --------
    @property
    def mid_frame_bytes(self) -> int:
        return lib().ds_mid_frame_bytes(self._h)

    def htask(self, frames, mid=None, planes=None, stream=None):
        """H task alone (K-N3): frames -> Mid (n, mid_frame_bytes) in HBM."""
        import torch

        n = _check_u8(frames, "frames", True, unit=self.in_frame_bytes)
        if mid is None:
            mid = torch.empty((n, self.mid_frame_bytes), dtype=torch.uint8, device=frames.device)
        _check_u8(mid, "mid", True, numel=n * self.mid_frame_bytes)
        p0, pc = planes if planes is not None else (0, self.channels)
        s = stream if stream is not None else torch.cuda.current_stream()
        rc = lib().ds_run_htask(self._h, frames.data_ptr(), n, mid.data_ptr(), p0, pc, s.cuda_stream)
        if rc:
            raise DSError(rc, "ds_run_htask")
        return mid

    def vtask(self, mid, out=None, planes=None, stream=None):
        """V task alone (K-N3): Mid -> frames out."""
        import torch

        n = _check_u8(mid, "mid", True, unit=self.mid_frame_bytes)
        if out is None:
            out = self.alloc_out(n)
        _check_u8(out, "out", True, numel=n * self.out_frame_bytes)
        p0, pc = planes if planes is not None else (0, self.channels)
        s = stream if stream is not None else torch.cuda.current_stream()
        rc = lib().ds_run_vtask(self._h, mid.data_ptr(), n, out.data_ptr(), p0, pc, s.cuda_stream)
        if rc:
            raise DSError(rc, "ds_run_vtask")
        return out

    def schedule_plan(self, schedule: int) -> dict:
        return ds_schedule_plan(self.w, self.h, self.channels, schedule, self.spec)

    def run_schedule(self, host_frames, schedule: int, host_out=None, stream=None):
        """Synchronous host-resident run under a transfer schedule; returns
        (host_out, stats dict)."""
        import torch

        n = _check_u8(host_frames, "host_frames", False, unit=self.in_frame_bytes)
        if host_out is None:
            host_out = torch.empty((n, self.out_frame_bytes), dtype=torch.uint8,
                                   pin_memory=host_frames.is_pinned())
        _check_u8(host_out, "host_out", False, numel=n * self.out_frame_bytes)
        st = ds_schedule_stats()
        s = stream if stream is not None else torch.cuda.current_stream()
        rc = lib().ds_run_schedule(self._h, host_frames.data_ptr(), n, host_out.data_ptr(), schedule,
                                   C.byref(st), s.cuda_stream)
        if rc:
            raise DSError(rc, "ds_run_schedule")
        return host_out, st.as_dict()

    def alloc_out(self, n: int):
        import torch

        return torch.empty((n, self.out_frame_bytes), dtype=torch.uint8,
                           device=f"cuda:{self.device}")

    def __call__(self, frames, out=None, stream=None):
        # Hot path for small batches: identity dtype checks, the raw current
        # stream, and the library call directly (tools/host_overhead.py).
        u8 = _torch_uint8()
        if frames.dtype is not u8 or not frames.is_cuda or not frames.is_contiguous():
            raise ValueError("frames must be a contiguous torch.uint8 CUDA tensor")
        total = frames.numel()
        n = total // self.in_frame_bytes
        if n * self.in_frame_bytes != total:
            raise ValueError("frames does not hold a whole number of frames")
        if out is None:
            out = self.alloc_out(n)
        elif (out.dtype is not u8 or not out.is_cuda or not out.is_contiguous()
              or out.numel() != n * self.out_frame_bytes):
            raise ValueError("out has the wrong dtype, device, layout or size")
        sp = stream.cuda_stream if stream is not None else _current_raw_stream(frames.device.index)
        rc = _lib.ds_run(self._h, frames.data_ptr(), n, out.data_ptr(), sp or None)
        if rc:
            raise DSError(rc, "ds_run")
        return out

    def run_host(self, host_frames, host_out=None, stream=None):
        """Host-resident path (ds_run_host): pinned CPU uint8 tensors in/out.
        Asynchronous on the stream; synchronise before reading host_out."""
        import torch

        n = _check_u8(host_frames, "host_frames", False, unit=self.in_frame_bytes)
        if host_out is None:
            host_out = torch.empty((n, self.out_frame_bytes), dtype=torch.uint8,
                                   pin_memory=host_frames.is_pinned())
        _check_u8(host_out, "host_out", False, numel=n * self.out_frame_bytes)
        s = stream if stream is not None else torch.cuda.current_stream()
        ds_run_host(self._h, host_frames.data_ptr(), n, host_out.data_ptr(), s.cuda_stream)
        return host_out


def generate_frames(n: int, in_frame_bytes: int, seed: int = 1, first_frame: int = 0,
                    device=None, out=None):
    """Synthetic frames on the device by global frame index (ds_generate),
    byte-identical to synth.random_frames(seed, first_frame, n, ...)."""
    import torch

    if out is None:
        out = torch.empty((n, in_frame_bytes), dtype=torch.uint8,
                          device=device if device is not None else "cuda")
    ds_generate(out.data_ptr(), n * in_frame_bytes, seed, first_frame * in_frame_bytes,
                torch.cuda.current_stream(out.device).cuda_stream)
    return out


__all__ = [n for n, _, _ in SIGNATURES] + [
    "Downscaler", "DSError", "make_spec", "generate_frames", "lib", "lib_path", "stage_to_dict",
]
