/*
 * ds.h -- C ABI of libds.so, the B200 (sm_100a) downscaler of
 * arxiv 1103.4881 ("Programming Massively Parallel Architectures using
 * MARTE: a Case Study").
 *
 * Citation key: P:n = PAPER.md line n; S:n = SPEC.md line n; SURVEY sec. n.
 *
 * The operation (PAPER sec. 3, P:64-90 and sec. 3.1): a stream of N
 * frames, each made of u8 colour planes, goes in; every plane goes through
 * an Array-OL horizontal repetitive task (pattern 8 -> 3, "interpolating
 * packets of 8 pixels"; taps S:530) and then a vertical one
 * (pattern 9 -> 4, 288 -> 128 lines; taps S:540), each applied via
 * tilers (origin, paving, fitting).  N frames of
 * (3W/8) x (4H/9) planes come out (352x288 -> 132x128).  Pixel
 * arithmetic is integer; the intermediate array is u8;
 * results are bit-exact and independent of kernel, grid and GPU count.
 *
 * Frame layout: plane 0 (Y), plane 1, plane 2 back to back, each
 * row-major u8, no headers, frames contiguous.  4:2:0 chroma planes are
 * (W/2, H/2); 4:4:4 is three equal planes ("24-bit RGB").
 *
 * Threading: every function is thread-safe.  A handle holds immutable
 * tables plus (after the first ds_run_host) staging buffers guarded by a
 * mutex; ds_run itself has no mutable state, so one handle may run
 * concurrently on several streams.
 *
 * Plain C: no C++ or torch types cross this boundary.
 */
#ifndef DS_H
#define DS_H

#include <stdint.h>

#if defined(__GNUC__)
#define DS_API __attribute__((visibility("default")))
#else
#define DS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ds_handle ds_handle;        /* opaque; owned by the library   */
typedef struct CUstream_st* ds_stream_t;   /* == cudaStream_t; NULL = legacy
                                              default stream                 */

/* Error codes (negative).  S:551 "non-divisible shape -> error"
 * "missing input array; shape mismatch" -> error. */
enum {
    DS_OK = 0,
    DS_EINVAL = -1,        /* bad argument: NULL, negative n, overlap, wrong device */
    DS_ESHAPE = -2,        /* plane not divisible by the paving steps       */
    DS_EUNSUPPORTED = -3,  /* channels not 1/3, spec over its limits               */
    DS_ECUDA = -4,         /* CUDA runtime / launch failure                         */
    DS_ENOMEM = -5         /* allocation failure                                    */
};

/* Colour layouts. */
enum { DS_CHROMA_444 = 0, DS_CHROMA_420 = 1 };

enum { DS_MAX_PATTERN = 16, DS_MAX_OUTPUTS = 8, DS_MAX_PLANES = 3 };

/* Kernel selection (ds_set_kernel / ds_last_kernel). */
enum {
    DS_KERNEL_AUTO = 0,     /* K-N1 when eligible, else K-N1g, else K-N2         */
    DS_KERNEL_FUSED = 1,    /* K-N1: TMA-staged fused H+V band kernel            */
    DS_KERNEL_GENERIC = 2,  /* K-N2: one thread per output pixel, any spec       */
    DS_KERNEL_FUSED_GENERAL = 3  /* K-N1g: TMA-staged fused band kernel for any spec:
                                    halo rows staged in smem, smem intermediate,
                                    runs of bands reusing the V halo, column strips
                                    for wide planes                                 */
};

/*
 * One separable Array-OL stage, i.e. one repetitive task with its tilers
 * along one axis, plus its elementary function:
 *   input tiler : origin `origin` (along the axis), paving step `paving`,
 *                 fitting 1, pattern [pattern]   (toroidal modulo)
 *   output tiler: origin 0, paving step `outputs`, fitting 1, pattern
 *                 [outputs]  -- exact coverage by construction
 *   body        : out[k] = clamp_0^255( trunc( (sum_i weight[k][i]*in[i]
 *                 + bias) / divisor ) )
 * pattern > paving gives a halo of pattern - paving elements.
 * Limits: 1 <= pattern <= 16, 1 <= paving <= 4096, 1 <= outputs <= 8,
 * 1 <= divisor <= 2^24, |weight| <= 65535, |bias| <= 2^24,
 * |origin| <= 2^20; otherwise DS_EUNSUPPORTED.
 */
typedef struct {
    int32_t pattern;
    int32_t paving;
    int32_t origin;
    int32_t outputs;
    int32_t weight[DS_MAX_OUTPUTS][DS_MAX_PATTERN];
    int32_t divisor;
    int32_t bias;
} ds_stage_spec;

/* h applies along rows ("horizontal filter"), v along columns of the
 * intermediate.  chroma is used when channels == 3. */
typedef struct {
    ds_stage_spec h;
    ds_stage_spec v;
    int32_t chroma;
} ds_filter_spec;

/* Geometry of a frame under a spec (host-only, no GPU needed). */
typedef struct {
    int64_t in_frame_bytes;              /* e.g. 3,110,400 for HD 4:2:0          */
    int64_t out_frame_bytes;             /* e.g.   518,400                       */
    int32_t n_planes;
    int32_t in_w[DS_MAX_PLANES], in_h[DS_MAX_PLANES];
    int32_t out_w[DS_MAX_PLANES], out_h[DS_MAX_PLANES];
    int64_t in_offset[DS_MAX_PLANES];    /* byte offset of each plane in a frame */
    int64_t out_offset[DS_MAX_PLANES];
    int32_t fused_eligible;              /* 1 if K-N1 can run this geometry+spec:
                                            SPEC's taps, every plane W % 16 in {0, 8}
                                            (8 also needs in_frame_bytes % 16 == 0),
                                            one 9-row group staged within smem      */
    int32_t band_groups[DS_MAX_PLANES];  /* K-N1: 9-row groups per work unit (band);
                                            rows < 512 B and W % 16 == 8 planes stage
                                            the whole band, dead rows included       */
    int64_t units_per_frame;             /* K-N1 work units per frame            */
    int64_t unit_in_bytes_max;           /* K-N1 bytes staged per unit (max)     */
    int64_t unit_out_bytes_max;
    int32_t fused_general_eligible;      /* 1 if K-N1g can run this geometry+spec  */
    int32_t general_band_reps[DS_MAX_PLANES];  /* K-N1g: V repetitions per band */
    int64_t general_units_per_frame;     /* K-N1g bands per frame (strips x bands); a
                                            launch groups them into runs (ds_units)  */
    int64_t general_stage_bytes_max;     /* K-N1g: staged bytes per unit: R rows (band + halo)
                                            at a pitch of round_up(W, 16) + 32 (wrap pad), or
                                            a column strip's window pitch */
    int32_t general_strips[DS_MAX_PLANES];  /* K-N1g: column strips per plane (1 = whole rows) */
} ds_plan_info;

/* Fill *out with SPEC's downscaler (hfilter_8to3 S:527-535, vfilter_9to4
 * S:537-545); chroma = DS_CHROMA_420.  Returns DS_OK. */
DS_API int ds_default_spec(ds_filter_spec* out);

/* Validate (frame_w, frame_h, channels, spec) and describe the geometry.
 * spec NULL = ds_default_spec.  Returns DS_OK or DS_EINVAL / DS_ESHAPE /
 * DS_EUNSUPPORTED (same rules as ds_create).  Host-only. */
DS_API int ds_plan(int32_t frame_w, int32_t frame_h, int32_t channels,
                   const ds_filter_spec* spec, ds_plan_info* out);

/* Create a downscaler bound to the CUDA device current at the call.
 * channels in {1, 3}.  spec NULL = SPEC's downscaler, 4:2:0 when
 * channels == 3.  Every plane must satisfy W_p % h.paving == 0 and
 * H_p % v.paving == 0 (4:2:0 with the default spec: W % 16 == 0 and
 * H % 18 == 0), else NULL with ds_last_error() == DS_ESHAPE.
 * The spec is copied.  Returns NULL on error (see ds_last_error). */
DS_API ds_handle* ds_create(int32_t frame_w, int32_t frame_h, int32_t channels,
                            const ds_filter_spec* filter_spec);

/* Downscale n_frames device-resident frames.
 *   in_frames : device pointer, n_frames * ds_in_frame_bytes(h) bytes, read
 *               only ("const", the read-only flowPort of P:132-135)
 *   out_frames: device pointer, n_frames * ds_out_frame_bytes(h) bytes
 * in_frames and out_frames on the handle's device.  out_frames may instead
 * lie on a peer GPU that was enabled for this handle with ds_enable_peer
 * (e.g. another rank's buffer mapped with CUDA IPC): the kernel's output
 * stores then travel over NVLink, fusing the gather of frame shards
 * into the filtering.  ds_run itself never enables peer access
 * and has no context-wide side effects.  Caller-owned, not retained, must
 * not overlap and must stay alive until work on `stream` completes.
 * Asynchronous on `stream`; faults surface at the caller's sync.
 * n_frames == 0 is a successful no-op.  Any alignment is accepted
 * (misalignment selects K-N1g's plain-load staging or plain stores, never
 * an error).
 * Returns DS_OK, DS_EINVAL (NULL handle/pointer with n > 0, n < 0,
 * overlapping ranges, a pointer that is not device memory, in_frames not on
 * the handle's device, out_frames neither on it nor on an enabled peer) or
 * DS_ECUDA. */
DS_API int ds_run(ds_handle* h, const uint8_t* in_frames, int64_t n_frames,
                  uint8_t* out_frames, ds_stream_t stream);

/* Allow ds_run on this handle to store its output into memory of GPU
 * peer_device (the gather of frame shards fused into the
 * kernels' output stores over NVLink / NVSwitch).  Enables CUDA peer access
 * from the handle's device to peer_device -- a context-wide setting of the
 * calling process, made here once and explicitly, never inside ds_run.
 * peer_device == the handle's device is a no-op.  Idempotent.
 * Returns DS_OK, DS_EINVAL (NULL handle, no such device), DS_EUNSUPPORTED
 * (the devices cannot access each other) or DS_ECUDA. */
DS_API int ds_enable_peer(ds_handle* h, int32_t peer_device);

/* Same result from HOST buffers (the paper's host-resident setting, P:146,
 * P:148): the library streams chunks of frames host -> device, runs the
 * downscaler and copies results device -> host, overlapping the three on
 * internal streams and staging buffers it owns (allocated on first use,
 * freed by ds_destroy).  In the spirit of the paper's transfer tuning
 * ("avoid extra data transfers"), with SPEC's taps the input rows
 * 9g+4 -- zero V weight, read by no kernel -- are not transferred
 * (8/9 of the input bytes cross PCIe).  host_in / host_out should be page-locked
 * (cudaHostAlloc / cudaHostRegister) for the copies to be asynchronous;
 * pageable memory works but serialises.  Asynchronous on `stream`:
 * host_out is valid after `stream` synchronises; both buffers must stay
 * alive until then.  Calls on one handle are serialised internally.
 * Returns as ds_run, plus DS_ENOMEM. */
DS_API int ds_run_host(ds_handle* h, const uint8_t* host_in, int64_t n_frames,
                       uint8_t* host_out, ds_stream_t stream);

/* Frames per chunk for ds_run_host (0 = automatic, ~96 MiB per chunk). */
DS_API int ds_set_host_chunk(ds_handle* h, int64_t frames_per_chunk);

/* Release the handle and its staging buffers (synchronises them).
 * NULL-safe. */
DS_API void ds_destroy(ds_handle* h);

/* Thread-local code of the last failed ds_create (DS_OK if none). */
DS_API int ds_last_error(void);

/* Static description of an error code; never NULL. */
DS_API const char* ds_strerror(int code);

/* The handle's current plan (band sizes follow ds_set_band_bytes). */
DS_API int ds_get_plan(const ds_handle* h, ds_plan_info* out);

/* Geometry queries; -1 / DS_EINVAL on a NULL handle. */
DS_API int64_t ds_in_frame_bytes(const ds_handle* h);
DS_API int64_t ds_out_frame_bytes(const ds_handle* h);
DS_API int ds_plane_dims(const ds_handle* h, int plane, int32_t* in_w, int32_t* in_h,
                         int32_t* out_w, int32_t* out_h);

/* K-N1g comes in two variants with identical results.  The runtime-tap
 * kernel (ds_general.cuh) reads the taps as data and runs any spec and
 * alignment.  K-N1s (ds_spec.cuh) has the spec compiled in -- taps, pattern,
 * paving, divisor, origin phase as constants, so zero taps, dead clamps and
 * byte shifting vanish -- and needs an H paving that is a multiple of 4,
 * taps in [-128, 127], at most 3 planes, rows of at least 64 bytes that hold
 * one H window, and an H origin with the same phase mod 16 on every plane
 * once reduced to (-W/2, W/2].  Any input and output alignment: rows are
 * read with 16-, 8- or 4-byte loads by their alignment, or as words
 * funnel-shifted out of aligned ones.  Specs with a built-in instance
 * (SPEC's downscaler, the halo reading of bench.py) use it directly; any
 * other spec is compiled at ds_create with NVRTC (about 0.3 s, once per spec
 * and process) when the runtime compiler is present (environment
 * DS_SPEC_JIT=0 turns that off; DS_GENERAL_COMPILED still compiles on
 * request) for the plan's row alignment only: calls from a less aligned
 * input pointer then run the runtime-tap kernel.  AUTO (default) picks
 * K-N1s whenever it can run a call. */
enum { DS_GENERAL_AUTO = 0, DS_GENERAL_RUNTIME = 1, DS_GENERAL_COMPILED = 2 };

/* Select the K-N1g variant.  Returns DS_OK, DS_EINVAL, or DS_EUNSUPPORTED
 * when the handle has no such variant (COMPILED: geometry/spec outside
 * K-N1s; RUNTIME: K-N1g cannot run the handle). */
DS_API int ds_set_general_variant(ds_handle* h, int32_t variant);

/* Variant used by the most recent ds_run when it ran a K-N1g kernel: 1
 * runtime taps, 2 compiled taps; 0 if the last kernel was not K-N1g. */
DS_API int ds_last_variant(const ds_handle* h);

/* Force a kernel (DS_KERNEL_*).  DS_KERNEL_FUSED / DS_KERNEL_FUSED_GENERAL
 * on an ineligible geometry/spec returns DS_EUNSUPPORTED and leaves the
 * setting unchanged.  A forced fused kernel still yields to K-N2 when the
 * input pointer is not 16-byte aligned.  AUTO picks K-N1 (SPEC taps), then
 * K-N1g, then K-N2. */
DS_API int ds_set_kernel(ds_handle* h, int32_t kernel);

/* Kernel used by the most recent ds_run on this handle (any thread), or
 * DS_KERNEL_AUTO if none yet. */
DS_API int ds_last_kernel(const ds_handle* h);

/* K-N1 tuning: ring stages per CTA (2..8) and CTAs per SM (0 = maximum
 * occupancy), for every call size.  Defaults: up to 3 CTAs per SM (as many as
 * fit) whose rings together hold ~120 KB, at least 2 stages each (120 KB in
 * flight per SM is the TMA read optimum measured by tools/bw_probe); where
 * that is 2 CTAs per SM (HD and wider), calls of at most 3 GiB of input run
 * one CTA per SM with 4 stages (measured faster below ~3 GB, slower above).
 * Returns DS_EINVAL when out of range.  Not synchronised with ds_run calls
 * in flight on other threads. */
DS_API int ds_set_tuning(ds_handle* h, int32_t stages, int32_t ctas_per_sm);

/* K-N1 work-unit (band) size: the largest number of 9-row groups whose
 * staged bytes stay <= target_bytes for plane 0, other planes matched to
 * it (0 = default: 32 KiB, or 8 KiB for frames under 64 KiB such as QCIF).  An explicit ds_set_tuning is kept (re-applied
 * to the new unit size).  On error the handle is left unchanged.  Output is
 * unaffected.  Not synchronised with ds_run calls in flight on other threads. */
DS_API int ds_set_band_bytes(ds_handle* h, int64_t target_bytes);

/* K-N1g run length: with a V halo (v.pattern > v.paving) a work unit is a
 * run of consecutive bands of one plane, and each band after the first
 * reuses the previous band's intermediate rows for the Pv - Sv halo rows
 * instead of staging and H-filtering them again.  bands > 0 forces that
 * many bands per run (clamped to the plane); 0 (default) picks runs per
 * launch, split evenly within each plane, sized for a few units per CTA
 * slot (K-N1s: ~4).  No effect
 * without a V halo.  Output is unaffected.  Not synchronised with ds_run
 * calls in flight on other threads. */
DS_API int ds_set_run_bands(ds_handle* h, int32_t bands);

/* K-N1g stage size: the staged bytes one band may occupy (0 = default:
 * 28 KiB with a V halo, 40 KiB without).  Planes whose k = 1 band does not
 * fit are split into column strips (ds_plan_info.general_strips).  Output is
 * unaffected; K-N1g stays ineligible if the result still exceeds shared
 * memory.  An explicit ds_set_tuning is kept; on error the handle is left
 * unchanged.  Not synchronised with ds_run calls in flight on other threads. */
DS_API int ds_set_general_stage_bytes(ds_handle* h, int64_t target_bytes);

/* K-N1 launch shape that ds_run would use for n_frames:
 * grid CTAs, threads per CTA, dynamic shared memory bytes. */
DS_API int ds_launch_shape(const ds_handle* h, int64_t n_frames, int32_t* grid,
                           int32_t* block, int32_t* smem_bytes);

/* Launch description of a kernel for a ds_run over n frames (bench.py's
 * report row: kernel, stages, ctas_per_sm). */
typedef struct {
    int32_t kernel;              /* DS_KERNEL_FUSED / _FUSED_GENERAL / _GENERIC        */
    int32_t grid, block, smem_bytes;
    int32_t stages;              /* ring slots per CTA (persistent kernels; 0 for K-N2) */
    int32_t ctas_per_sm;         /* resident CTAs per SM the grid is sized for         */
    int32_t consumer_warps;      /* compute warps per CTA (plus one producer warp)     */
    int64_t units;               /* work units of the launch (K-N2: output bytes)      */
    int64_t unit_in_bytes_max;   /* bytes staged per unit                              */
    int32_t variant;             /* K-N1g family: 1 runtime taps, 2 compiled taps
                                    (built-in instance), 3 compiled taps (run-time
                                    compiled); 0 otherwise                             */
    int32_t reserved_;
} ds_launch;

/* Fill *out for `kernel` (DS_KERNEL_FUSED, DS_KERNEL_FUSED_GENERAL or
 * DS_KERNEL_GENERIC) as ds_run would launch it for n_frames on this handle.
 * Host-only.  Returns DS_OK, DS_EINVAL, or DS_EUNSUPPORTED if that kernel
 * cannot run the handle. */
DS_API int ds_launch_info(const ds_handle* h, int64_t n_frames, int32_t kernel, ds_launch* out);

/* ---- the paper's unfused structure and its transfer schedules
 *
 * Bytes of one frame's intermediate arrays Mid (the H task's u8 output,
 * S:365): planes' (H_p x Qh*W_p/Sh) arrays back to back, the same layout
 * rule as frames.  -1 on a NULL handle. */
DS_API int64_t ds_mid_frame_bytes(const ds_handle* h);

/* K-N3: one repetitive task per launch, as the paper's generated code does
 * ("the six repetitive tasks ... allocated onto the GPU in order to
 * generate kernels"), with Mid in HBM.  ds_run_htask: in -> mid (H task);
 * ds_run_vtask: mid -> out (V task); over planes [plane_first,
 * plane_first + plane_count) of n frames.  Pointers are frame-base device
 * pointers (n * in/mid/out frame bytes), caller-owned, non-overlapping.
 * SPEC taps with aligned geometry take vectorised kernels, anything else a
 * literal tiler kernel.  Asynchronous on `stream`.  Returns as ds_run. */
DS_API int ds_run_htask(ds_handle* h, const uint8_t* in_frames, int64_t n_frames, uint8_t* mid,
                        int32_t plane_first, int32_t plane_count, ds_stream_t stream);
DS_API int ds_run_vtask(ds_handle* h, const uint8_t* mid, int64_t n_frames, uint8_t* out_frames,
                        int32_t plane_first, int32_t plane_count, ds_stream_t stream);

/* Host <-> device transfer schedules of a host-resident stream. */
enum {
    DS_SCHED_NAIVE = 0,      /* H2D every task input, D2H every task
                                output -> 12 transfers/frame ("not optimized") */
    DS_SCHED_OPTIMIZED = 1,  /* residency-aware -> 3 H2D + 3 D2H per frame
                                ("performance tuning")                   */
    DS_SCHED_FUSED = 2,      /* per frame: 1 H2D, one fused K-N1 launch, 1 D2H      */
    DS_SCHED_STREAMED = 3    /* ds_run_host: chunked, overlapped on 3 streams       */
};

typedef struct {
    int64_t frames;
    int64_t h2d_count, d2h_count;         /* transfers                                */
    int64_t h2d_bytes, d2h_bytes;
    int64_t launches;
    double h2d_ms, d2h_ms, kernel_ms;     /* device time per phase: CUDA events around
                                             every step, steps serialised on one stream
                                             (STREAMED: 0, steps overlap)              */
    double kernel_ms_plane[DS_MAX_PLANES];/* per colour component ("y-component") */
    double total_ms;                      /* first to last event                       */
} ds_schedule_stats;

/* Per-frame transfer counts / bytes / launches of a schedule for a frame
 * geometry (host-only, like ds_plan; the deterministic quantities behind
 * P:148's "about 30% and 70% faster transfer times"; for STREAMED one
 * transfer each way per chunk).  Returns DS_OK, DS_EINVAL or ds_plan's
 * errors. */
DS_API int ds_schedule_plan(int32_t frame_w, int32_t frame_h, int32_t channels,
                            const ds_filter_spec* spec, int32_t schedule,
                            ds_schedule_stats* per_frame);

/* Run n host-resident frames (host_in -> host_out, pinned memory advised)
 * frame by frame under `schedule`, on `stream`, and fill *stats (totals
 * over the call).  SYNCHRONOUS: returns after host_out is written.  Uses
 * one frame of library-owned device scratch (and a pinned host copy of Mid
 * for NAIVE), freed by ds_destroy; calls on one handle are serialised.
 * Returns as ds_run_host. */
DS_API int ds_run_schedule(ds_handle* h, const uint8_t* host_in, int64_t n_frames,
                           uint8_t* host_out, int32_t schedule, ds_schedule_stats* stats,
                           ds_stream_t stream);

/* ---- general Array-OL repetitive tasks --------------------------
 *
 * A tiler: element_index(r, f) = (origin + paving.r + fitting.f)
 * mod shape, component-wise, non-negative modulo.  paving is
 * array dims x repetition dims, fitting array dims x pattern dims (row-major
 * [array dim][k]).  Limits: 1..4 array dims, 1..4 repetition dims, 0..4
 * pattern dims; every extent >= 1; product(shape) <= 2^32; repetition
 * extents < 2^31; origin/paving/fitting entries |x| <= 2^40. */
typedef struct {
    int32_t ndim;
    int64_t shape[4];
    int64_t origin[4];
    int32_t nrep;
    int64_t paving[4][4];
    int32_t npat;
    int64_t fitting[4][4];
    int64_t pattern[4];
} ds_tiler;

/* Elementary function of a task: a linear integer body over the
 * row-major flattened input pattern (n_in <= 16 elements) producing n_out
 * <= 8 elements in the output pattern's row-major order:
 * out[k] = clamp_0^255(trunc((sum_i weight[k][i] * in[i] + bias) / divisor))
 * (the form of S:530/S:540; limits as ds_stage_spec). */
typedef struct {
    int32_t n_in, n_out;
    int32_t weight[DS_MAX_OUTPUTS][DS_MAX_PATTERN];
    int32_t divisor, bias;
} ds_task_body;

/* Launch topology (rule S:349-357; the paper's lost Fig. 3,
 * P:122-130): collapse dimensions beyond max_dims by multiplying trailing
 * extents; below min_items one work-group sized to the multiplicity;
 * otherwise a power-of-two local box, product <= min(max_wg, wg_threshold),
 * grown one dimension at a time round-robin from the largest dimension while
 * the padded global size stays < 2 x the multiplicity; global[d] = smallest
 * multiple of local[d] >= multiplicity[d]; guarded iff padded. */
typedef struct {
    int32_t ndim;                 /* collapsed dims, 1..3            */
    int64_t multiplicity[3];      /* collapsed repetition extents    */
    int32_t local[3];
    int64_t global[3];
    int32_t guarded;
} ds_topology;

enum { DS_TOPO_FLAT = 0, DS_TOPO_SPEC = 1 };

/* Host-only.  max_wg = device max work-group size (0 -> DS_EINVAL);
 * max_dims 1..3; min_items default 64 and wg_threshold default 256. */
DS_API int ds_compute_topology(int32_t nrep, const int64_t* multiplicity, int32_t max_wg,
                               int32_t max_dims, int32_t min_items, int32_t wg_threshold,
                               ds_topology* out);

/* Run one repetitive task on the current device (S:72-77 executed as
 * S:517-520): for every repetition index r of rep_shape, pattern =
 * extract(in, t_in, r); write(out, t_out, r, body(pattern)).  in / out are
 * device arrays of product(t_in.shape) / product(t_out.shape) bytes,
 * caller-owned, non-overlapping; elements not covered by t_out are left
 * untouched.  Repetitions run in parallel: if t_out is not an exact
 * cover (ds_tiler_coverage) multiply-written elements are unspecified.
 * policy DS_TOPO_FLAT: grid-stride over repetitions; DS_TOPO_SPEC: the
 * ds_compute_topology launch (B200 limits), guarded.  Asynchronous on
 * `stream`.  Returns DS_OK, DS_EINVAL (bad tiler/body/pointers),
 * DS_EUNSUPPORTED (over the limits) or DS_ECUDA. */
DS_API int ds_run_task(const uint8_t* in, const ds_tiler* t_in, uint8_t* out, const ds_tiler* t_out,
                       int32_t nrep, const int64_t* rep_shape, const ds_task_body* body,
                       int32_t policy, ds_stream_t stream);

/* check_coverage on the device: count, for every element of
 * t's array, the (r, f) pairs that hit it; *overlaps = elements hit more
 * than once, *gaps = elements never hit (exact iff both are 0).
 * SYNCHRONOUS on `stream`; allocates a temporary 4-byte counter per
 * element.  Returns as ds_run_task, plus DS_ENOMEM. */
DS_API int ds_tiler_coverage(const ds_tiler* t, int32_t nrep, const int64_t* rep_shape,
                             int64_t* overlaps, int64_t* gaps, ds_stream_t stream);

/* ---- debug: work-unit accounting (stand-in for compute-sanitizer, which is
 * closed on this GPU pool).  When counts != NULL, every K-N1 / K-N1g work
 * unit u processed by a later ds_run / ds_run_host adds 1 to counts[u]
 * (device array of ds_units(h, n, kernel) u32, caller-zeroed); a correct
 * persistent schedule leaves every entry exactly 1.  NULL switches it off
 * (the default; costs one predicate per unit). */
DS_API int ds_set_debug_counter(ds_handle* h, uint32_t* counts);

/* Work units of a ds_run over n frames with K-N1 (DS_KERNEL_FUSED) or K-N1g
 * (DS_KERNEL_FUSED_GENERAL); -1 if that kernel cannot run the handle. */
DS_API int64_t ds_units(const ds_handle* h, int64_t n_frames, int32_t kernel);

/* Synthetic input (bench / test infrastructure, not part of the method):
 * fills dev[0 .. n_bytes) on the current device with
 *   byte(i) = splitmix64(seed * 0x9E3779B97F4A7C15 + start_index + i) >> 56
 * (the counter hash of synth/__init__.py).  Asynchronous on `stream`. */
DS_API int ds_generate(uint8_t* dev, int64_t n_bytes, uint64_t seed, int64_t start_index,
                       ds_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* DS_H */
