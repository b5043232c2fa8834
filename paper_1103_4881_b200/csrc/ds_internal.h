// ds_internal.h -- shared internals of libds.so (not part of the C ABI).
#pragma once
#include <atomic>
#include <cstdint>
#include <mutex>
#include <vector>

#include <cuda_runtime.h>

#include "ds.h"

namespace dsi {

constexpr int kHostSlots = 3;                       // ds_run_host pipeline depth
constexpr int64_t kUnitTargetBytes = 32 * 1024;     // K-N1 band size target (bytes staged)
constexpr int64_t kSmallFrameBytes = 64 * 1024;     // frames below this (QCIF: 38 KB) ...
constexpr int64_t kSmallUnitTargetBytes = 8 * 1024; // ... take 8 KB bands: more, smaller units and CTAs
                                                    // (QCIF x 2000: 0.58 -> 0.66 of the copy peak,
                                                    // profiles/r02/k1_small_sweep.txt)
inline int64_t default_band_target(int64_t in_frame_bytes) {
    return in_frame_bytes < kSmallFrameBytes ? kSmallUnitTargetBytes : kUnitTargetBytes;
}
constexpr int64_t kInFlightTarget = 120 * 1024;     // K-N1 bytes in flight per SM (measured
                                                    // optimum of tools/bw_probe tma_read)
constexpr int kK1Ctas = 3;                          // K-N1 CTAs per SM (cap; what fits runs)
constexpr int64_t kOneCtaMaxBytes = 3LL << 30;      // K-N1 calls up to this much input (wide
                                                    // plans) run one CTA per SM x 4 stages:
                                                    // measured crossover 2.8-3.7 GB
                                                    // (profiles/r02/k1_cta_ab4.txt)
constexpr int kSmemLimit = 227 * 1024;              // per-CTA opt-in maximum
constexpr int64_t kHostChunkBytes = 96LL << 20;     // ds_run_host chunk target (tools/e2e_sweep.py)

struct HostSlot {
    uint8_t* d_in = nullptr;
    uint8_t* d_out = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
};

// ds_run_schedule scratch: one frame of device arrays + a pinned host copy of
// the intermediate (the naive schedule moves it to the host and back).
struct SchedState {
    uint8_t* d_in = nullptr;
    uint8_t* d_mid = nullptr;
    uint8_t* d_out = nullptr;
    uint8_t* h_mid = nullptr;
    std::vector<cudaEvent_t> events;
    bool ready = false;
};

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// One K-N1 launch configuration: a band plan plus its launch shape.
struct FusedCfg {
    ds_plan_info plan{};
    int ncw = 4;                 // consumer warps per CTA
    int stages = 4;              // ring depth
    int ctas_per_sm = 1;         // 0 = occupancy maximum
    int32_t stage_stride = 0, out_stride = 0;
    bool valid = false;
    // cached launch shape (computed when the configuration is set, so ds_run
    // makes no occupancy / attribute calls)
    int grid_per_sm = 0, threads = 0, smem = 0, run_stages = 0;
};

#ifndef DS_HTASK_TMA
#define DS_HTASK_TMA 1
#endif
constexpr bool kHtaskTma = DS_HTASK_TMA != 0;      // K-N3 H task on the TMA pipeline (flat ranges)
constexpr int64_t kHtaskUnit = 24 * 1024;          // its unit: input bytes per ring slot (x 128)
constexpr int64_t kFineUnitTarget = 16 * 1024;      // small batches: more, smaller units
#ifndef DS_GEN_STAGE_TARGET
#define DS_GEN_STAGE_TARGET (40 * 1024)
#endif
constexpr int64_t kGeneralStageTarget = DS_GEN_STAGE_TARGET;  // K-N1g staged rows per band
#ifndef DS_GEN_STAGE_TARGET_REUSE
#define DS_GEN_STAGE_TARGET_REUSE (28 * 1024)
#endif
constexpr int64_t kGeneralStageTargetReuse = DS_GEN_STAGE_TARGET_REUSE;  // ... when bands reuse a V halo

// K-N1g per-plane geometry (ds_api.cu general_plane_geom)
struct GenGeom {
    int32_t strips = 1, sw = 0, np_last = 0;   // column strips, H repetitions per strip (last: np_last)
    int32_t k = 0, R = 0, pitch = 0;          // V repetitions per band, staged rows, staged row stride
    int32_t wm_max = 0;                       // widest mid / output row of a unit (bytes)
};

// K-N1g launch configuration (any stage spec).
struct GeneralCfg {
    bool valid = false;
    GenGeom geom[DS_MAX_PLANES];
    int32_t k[DS_MAX_PLANES] = {0, 0, 0};     // V repetitions per band
    int32_t nb[DS_MAX_PLANES] = {0, 0, 0};    // bands per plane
    int32_t R[DS_MAX_PLANES] = {0, 0, 0};     // staged rows per band (first band of a run)
    int32_t ovl = 0;                          // Pv - Sv > 0: halo rows shared by consecutive bands
    int32_t mid_alt = 0;                      // second mid buffer offset (0: one buffer)
    int32_t stage_stride = 0, mid_stride = 0, out_stride = 0;
    int stages = 2, ncw = 8;
    int fast = 0;                             // division mode (ds_general.cuh g_out): 0, 1 or 2
    int grid_per_sm = 0, threads = 0, smem = 0;
};

// K-N1s (ds_spec.cu): the fused band kernel with the spec compiled in
using SpecFn = void (*)(void);
struct SpecPlaneCfg {
    int32_t strips = 1, sw = 0, k = 0, nb = 0, R = 0, pitch = 0, mp = 0, unit_start = 0;
    int32_t rows_alloc = 0;        // K-N1s: intermediate rows per buffer (R + rows per warp - 1)
};
struct SpecCfg {
    bool valid = false;
    int jit = 0;                   // 0: built-in instance, 1: compiled at run time (NVRTC)
    SpecFn fn = nullptr;           // kernel entry for the plan's row alignment (runtime-API function, or a JIT CUfunction)
    SpecFn fn_al[7] = {};          // entries by call row alignment 16 / 8 / 4 / not 4 / 16-byte rows 4, 8, 12
                                   // bytes off (built-in: all that apply; JIT: the plan's alignment only)
    int al = 16;                   // row alignment of the plan (frame size, plane offsets, widths)
    SpecPlaneCfg plane[DS_MAX_PLANES];
    int32_t upf = 0, stages = 2, stage_stride = 0, mid_stride = 0;
    int threads = 0, smem = 0, grid_per_sm = 0;
};

// K-N1: planes with W % 16 == 0 and rows shorter than this stage whole bands
// (dead rows included) with one bulk copy per band instead of k + 1 copies of
// 8 live rows: short rows make those copies small (CIF luma: 2.8 KB)
#ifndef DS_K1_WHOLE_MAX_W
#define DS_K1_WHOLE_MAX_W 512
#endif
inline bool k1_whole_band(int64_t W) { return W % 16 == 0 && W < DS_K1_WHOLE_MAX_W; }

// K-N1g staged row stride: the row, rounded to 16 bytes, then the 32-byte wrap pad
inline int64_t general_pitch(int64_t W) { return (W + 15) / 16 * 16 + 32; }

}  // namespace dsi

struct ds_handle {
    int device = 0;
    int sm_count = 0;
    int32_t W = 0, H = 0, channels = 0;
    ds_filter_spec spec{};
    ds_plan_info plan{};
    // K-N1 launch configurations: `fused` (bands of ~band_target bytes, used
    // for streams) and `fine` (~16 KiB bands, used when a call has fewer
    // coarse units than 2 per SM, e.g. one HD frame)
    int64_t band_target = dsi::kUnitTargetBytes;
    dsi::FusedCfg fused, fine;
    // `onecta`: the coarse plan at one CTA per SM and a 4-deep ring, for calls
    // of at most kOneCtaMaxBytes of input when `fused` runs 2 CTAs per SM
    dsi::FusedCfg onecta;
    dsi::GeneralCfg general;
    dsi::SpecCfg spec_cfg;                  // K-N1s (compiled-spec K-N1g)
    int32_t general_variant = 0;            // ds_set_general_variant: 0 auto, 1 runtime taps, 2 compiled taps
    bool spec_jit_req = false;              // compile K-N1s at run time for a spec without a built-in instance
    int kernel_pref = DS_KERNEL_AUTO;
    int32_t run_bands = 0;                  // ds_set_run_bands (0 = automatic)
    int32_t tune_stages = 0, tune_ctas = 0; // explicit ds_set_tuning (0 stages = none)
    bool htask_tma_ready = false;           // smem attribute set for ds_htask_tma_kernel
    int64_t general_target = 0;             // ds_set_general_stage_bytes (0 = default)
    uint32_t* debug_unit_count = nullptr;   // ds_set_debug_counter
    std::atomic<int> last_kernel{DS_KERNEL_AUTO};
    std::atomic<int> last_variant{0};       // K-N1g family: 1 runtime taps, 2 compiled taps (K-N1s)
    std::atomic<uint64_t> peer_mask{0};     // ds_enable_peer: peer devices ds_run may store to
    // ds_run_host / ds_run_schedule state (lazily allocated, guarded by host_mu)
    std::mutex host_mu;
    int64_t host_chunk = 0;      // frames per chunk, 0 = auto
    int64_t host_alloc_frames = 0;
    dsi::HostSlot slots[dsi::kHostSlots];
    cudaEvent_t fork_ev = nullptr;
    bool host_init = false;
    dsi::SchedState sched;
};

namespace dsi {

void default_spec(ds_filter_spec* s);
bool stage_equal(const ds_stage_spec& a, const ds_stage_spec& b);
bool aligned16(const void* p);
bool device_ptr_on(const void* p, int dev);
bool out_ptr_ok(const ds_handle* h, const void* p);
bool ranges_overlap(const void* a, int64_t na, const void* b, int64_t nb);
int run_device(ds_handle* h, const uint8_t* in, int64_t n, uint8_t* out, cudaStream_t st);
void free_sched_state(ds_handle* h);
int configure_spec(ds_handle* h);
bool spec_call_ok(const ds_handle* h, const uint8_t* in, const uint8_t* out);
int launch_spec(ds_handle* h, const uint8_t* in, int64_t n, uint8_t* out, cudaStream_t st);
SpecFn spec_jit_kernel(ds_handle* h, int phase, int align);
bool spec_jit_available();
const char* spec_jit_log();
int spec_jit_set_smem(SpecFn fn, int smem);
int spec_jit_occupancy(SpecFn fn, int threads, int smem, int* occ);
int spec_jit_launch(SpecFn fn, unsigned grid, unsigned threads, unsigned smem, cudaStream_t st, void** args);
void spec_runs(const ds_handle* h, int64_t n, int32_t* L, int32_t* upf);
int make_plan(int32_t W, int32_t H, int32_t channels, const ds_filter_spec* spec_in,
              ds_filter_spec* spec_out, ds_plan_info* info, int64_t unit_target = kUnitTargetBytes,
              int64_t general_target = 0);
// K-N1g stage target: explicit (ds_set_general_stage_bytes) or the default for the spec
inline int64_t general_stage_target(const ds_filter_spec& spec, int64_t explicit_target) {
    if (explicit_target > 0) return explicit_target;
    return spec.v.pattern > spec.v.paving ? kGeneralStageTargetReuse : kGeneralStageTarget;
}

// Device binding: run with the handle's device current, restore after.
struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) { ok = false; return; }
        if (prev != dev && cudaSetDevice(dev) != cudaSuccess) ok = false;
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

}  // namespace dsi
