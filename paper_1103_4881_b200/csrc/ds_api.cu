// ds_api.cu -- the C ABI of include/ds.h: validation, planning, launches,
// and the host-resident streaming path.  Citations: P:n = PAPER.md line n,
// S:n = SPEC.md line n, SURVEY sec. n.
#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "ds.h"
#include "ds_internal.h"
#include "ds_kernels.cuh"
#include "ds_general.cuh"
#include "ds_spec.cuh"

namespace {
thread_local int g_last_error = DS_OK;
}  // namespace

using namespace dsi;

namespace dsi {

void default_spec(ds_filter_spec* s) {
    std::memset(s, 0, sizeof *s);
    // hfilter_8to3
    s->h.pattern = 8; s->h.paving = 8; s->h.origin = 0; s->h.outputs = 3;
    s->h.weight[0][0] = 1; s->h.weight[0][1] = 5;
    s->h.weight[1][3] = 3; s->h.weight[1][4] = 3;
    s->h.weight[2][6] = 5; s->h.weight[2][7] = 1;
    s->h.divisor = 6; s->h.bias = 3;
    // vfilter_9to4
    s->v.pattern = 9; s->v.paving = 9; s->v.origin = 0; s->v.outputs = 4;
    s->v.weight[0][0] = 3; s->v.weight[0][1] = 5;
    s->v.weight[1][2] = 1; s->v.weight[1][3] = 7;
    s->v.weight[2][5] = 7; s->v.weight[2][6] = 1;
    s->v.weight[3][7] = 5; s->v.weight[3][8] = 3;
    s->v.divisor = 8; s->v.bias = 4;
    s->chroma = DS_CHROMA_420;
}

bool stage_equal(const ds_stage_spec& a, const ds_stage_spec& b) {
    return std::memcmp(&a, &b, sizeof a) == 0;
}

int check_stage(const ds_stage_spec& s) {
    if (s.pattern < 1 || s.pattern > DS_MAX_PATTERN) return DS_EUNSUPPORTED;
    if (s.paving < 1 || s.paving > 4096) return DS_EUNSUPPORTED;
    if (s.outputs < 1 || s.outputs > DS_MAX_OUTPUTS) return DS_EUNSUPPORTED;
    if (s.divisor < 1 || s.divisor > (1 << 24)) return DS_EUNSUPPORTED;
    if (s.bias < -(1 << 24) || s.bias > (1 << 24)) return DS_EUNSUPPORTED;
    if (s.origin < -(1 << 20) || s.origin > (1 << 20)) return DS_EUNSUPPORTED;
    for (int k = 0; k < DS_MAX_OUTPUTS; ++k)
        for (int i = 0; i < DS_MAX_PATTERN; ++i) {
            const int32_t w = s.weight[k][i];
            if (w < -65535 || w > 65535) return DS_EUNSUPPORTED;
            if ((k >= s.outputs || i >= s.pattern) && w != 0) return DS_EUNSUPPORTED;
        }
    return DS_OK;
}

// K-N1 band choice: luma takes the largest
// divisor k of its 9-row group count with 8 k W <= target; the other planes
// take the divisor whose staged bytes are closest to luma's, so units are
// (near-)equal in bytes and a static round-robin balances the SMs.
int largest_divisor_below(int G, int64_t per_group, int64_t target) {
    int best = 1;
    for (int d = 1; d <= G; ++d)
        if (G % d == 0 && per_group * d <= target) best = d;
    return best;
}
int closest_divisor(int G, int64_t per_group, int64_t target) {
    int best = 1;
    int64_t bestd = INT64_MAX;
    for (int d = 1; d <= G; ++d) {
        if (G % d) continue;
        const int64_t diff = std::llabs(per_group * d - target);
        if (diff < bestd) { bestd = diff; best = d; }
    }
    return best;
}

int64_t fused_smem_bytes(int stages, int32_t stage_stride, int32_t out_stride) {
    return (int64_t)stages * stage_stride + (int64_t)ds::kOutSlots * out_stride +
           (int64_t)2 * stages * 8;
}

// K-N1g per-plane geometry.  A band of k V repetitions stages
// R = Sv (k-1) + Pv rows.  Whole rows (row + 32-byte wrap pad) when a k = 1
// band fits the stage target; otherwise column strips of sw H repetitions
// (a multiple of 16, so strip outputs start 16-byte aligned) whose input
// window Sh (sw-1) + Ph is staged from its 16-aligned superset (+15 bytes of
// phase, +20 bytes of window over-read slack).  k is then the largest divisor
// of the band count whose rows still fit.
GenGeom general_plane_geom(const ds_filter_spec& spec, int32_t W, int32_t Hp, int64_t target) {
    GenGeom g;
    const int Sh = spec.h.paving, Ph = spec.h.pattern;
    const int np = W / Sh;
    const int G = Hp / spec.v.paving;
    const int64_t R1 = spec.v.pattern;
    int64_t pitch = general_pitch(W);
    g.strips = 1; g.sw = np; g.np_last = np;
    auto strip_pitch = [&](int64_t sw) { return round_up((int64_t)Sh * (sw - 1) + Ph + 15 + 20, 16); };
    if (R1 * pitch > target && np >= 32) {
        int64_t sw = np / 16 * 16;
        while (sw > 16 && (R1 * strip_pitch(sw) > target || strip_pitch(sw) > W)) sw -= 16;
        if (sw >= 16 && sw < np && strip_pitch(sw) <= W) {
            g.sw = (int32_t)sw;
            g.strips = (int32_t)((np + sw - 1) / sw);
            g.np_last = (int32_t)(np - (int64_t)(g.strips - 1) * sw);
            pitch = strip_pitch(sw);
        }
    }
    int best = 1;
    for (int d = 1; d <= G; ++d) {
        if (G % d) continue;
        if (((int64_t)spec.v.paving * (d - 1) + spec.v.pattern) * pitch <= target) best = d;
    }
    g.k = best;
    g.R = spec.v.paving * (best - 1) + spec.v.pattern;
    g.pitch = (int32_t)pitch;
    g.wm_max = spec.h.outputs * g.sw;
    return g;
}

int make_plan(int32_t W, int32_t H, int32_t channels, const ds_filter_spec* spec_in,
              ds_filter_spec* spec_out, ds_plan_info* info, int64_t unit_target, int64_t general_target) {
    ds_filter_spec spec;
    if (spec_in) spec = *spec_in; else default_spec(&spec);
    if (W < 1 || H < 1) return DS_ESHAPE;
    if (channels != 1 && channels != 3) return DS_EUNSUPPORTED;
    if (channels == 3 && spec.chroma != DS_CHROMA_444 && spec.chroma != DS_CHROMA_420)
        return DS_EUNSUPPORTED;
    int rc = check_stage(spec.h);
    if (rc) return rc;
    rc = check_stage(spec.v);
    if (rc) return rc;

    ds_plan_info pi;
    std::memset(&pi, 0, sizeof pi);
    pi.n_planes = channels;
    int64_t inb = 0, outb = 0;
    for (int p = 0; p < channels; ++p) {
        int32_t pw = W, ph = H;
        if (channels == 3 && spec.chroma == DS_CHROMA_420 && p > 0) {
            if (W % 2 || H % 2) return DS_ESHAPE;
            pw = W / 2; ph = H / 2;
        }
        if (pw % spec.h.paving || ph % spec.v.paving) return DS_ESHAPE;
        pi.in_w[p] = pw; pi.in_h[p] = ph;
        pi.out_w[p] = spec.h.outputs * (pw / spec.h.paving);    // 3W/8
        pi.out_h[p] = spec.v.outputs * (ph / spec.v.paving);    // 4H/9
        pi.in_offset[p] = inb; pi.out_offset[p] = outb;
        inb += (int64_t)pw * ph;
        outb += (int64_t)pi.out_w[p] * pi.out_h[p];
    }
    pi.in_frame_bytes = inb;
    pi.out_frame_bytes = outb;

    ds_filter_spec def;
    default_spec(&def);
    // K-N1 eligibility: SPEC's taps (the kernel hard-codes them and skips the
    // dead row 4 of every 9-row group).  SPEC's H paving makes every width a
    // multiple of 8: W % 16 == 0 planes stage their 8 live rows per group by
    // 16-byte-aligned bulk copies, W % 16 == 8 planes as below.
    bool fused = stage_equal(spec.h, def.h) && stage_equal(spec.v, def.v);
    // planes with W % 16 == 8 ("narrow") are staged as whole bands from a
    // 16-aligned superset, which needs 16-aligned frames
    bool any_narrow = false;
    for (int p = 0; p < channels; ++p) any_narrow |= (pi.in_w[p] % 16 != 0);
    if (any_narrow && pi.in_frame_bytes % 16 != 0) fused = false;
    if (fused) {
        // staged bytes per 9-row group: 8 live rows, or all 9 for narrow planes
        // and for short aligned rows staged as whole bands (k1_whole_band)
        auto per_group = [&](int p) { return (k1_whole_band(pi.in_w[p]) || pi.in_w[p] % 16 ? 9LL : 8LL) * pi.in_w[p]; };
        // shrink the band target until a 2-deep ring fits one CTA's shared
        // memory (a caller's large ds_set_band_bytes never loses K-N1)
        const int G0 = pi.in_h[0] / 9;
        int64_t want = unit_target;
        for (;;) {
            const int k0 = largest_divisor_below(G0, per_group(0), want);
            const int64_t target = per_group(0) * k0;
            int64_t units = 0, umax = 0, omax = 0;
            for (int p = 0; p < channels; ++p) {
                const int G = pi.in_h[p] / 9;
                const int k = p == 0 ? k0 : closest_divisor(G, per_group(p), target);
                pi.band_groups[p] = k;
                units += G / k;
                umax = std::max<int64_t>(umax, per_group(p) * k + (pi.in_w[p] % 16 ? 16 : 0));
                omax = std::max<int64_t>(omax, 4LL * k * pi.out_w[p]);
            }
            pi.units_per_frame = units;
            pi.unit_in_bytes_max = umax;
            pi.unit_out_bytes_max = omax;
            fused = fused_smem_bytes(2, (int32_t)round_up(umax, 128), (int32_t)round_up(omax, 128)) <=
                    kSmemLimit;
            if (fused || k0 == 1) break;
            want = per_group(0) * k0 - 1;      // next smaller luma band
        }
    }
    pi.fused_eligible = fused ? 1 : 0;
    if (!fused) {
        for (int p = 0; p < DS_MAX_PLANES; ++p) pi.band_groups[p] = 0;
        pi.units_per_frame = pi.unit_in_bytes_max = pi.unit_out_bytes_max = 0;
    }
    // K-N1g (any spec, any width): bands of k V repetitions stage
    // R = Sv (k-1) + Pv rows (band + halo), each at a pitch of
    // round_up(W, 16) + 32 (row + wrap pad) -- by TMA when rows are 16-byte
    // multiples, else by the producer warp with plain loads.
    bool general = true;         // any width: unaligned rows are staged with plain loads
    if (general) {
        int64_t units = 0, smax = 0, mmax = 0, omax = 0;
        // with a V halo (Pv > Sv) consecutive bands of a run reuse the halo's mid
        // rows, so small bands cost little and leave smem for a second mid buffer
        const int64_t stage_target = general_stage_target(spec, general_target);
        for (int p = 0; p < channels; ++p) {
            const int G = pi.in_h[p] / spec.v.paving;
            const GenGeom gg = general_plane_geom(spec, pi.in_w[p], pi.in_h[p], stage_target);
            const int64_t R = gg.R, best = gg.k;
            pi.general_band_reps[p] = gg.k;
            pi.general_strips[p] = gg.strips;
            units += (int64_t)gg.strips * (G / best);
            smax = std::max<int64_t>(smax, R * gg.pitch);
            mmax = std::max<int64_t>(mmax, (R + 3) * gg.wm_max);   // +3: dp4a row blocks
            omax = std::max<int64_t>(omax, (int64_t)spec.v.outputs * best * gg.wm_max);
            // exact reciprocal index division: items * divisor < 2^32
            const int64_t np = gg.sw;
            if (R * np * np >= (1LL << 32) ||
                (int64_t)spec.v.outputs * best * gg.wm_max * gg.wm_max >= (1LL << 32))
                general = false;
        }
        const int64_t mids = spec.v.pattern > spec.v.paving ? 2 : 1;
        const int64_t need = 2 * round_up(smax, 128) + mids * round_up(mmax, 128) + 2 * round_up(omax, 128) +
                             2 * DS_MAX_OUTPUTS * DS_MAX_PATTERN * 4 + 64;
        if (need > kSmemLimit) general = false;
        pi.general_units_per_frame = units;
        pi.general_stage_bytes_max = smax;
    }
    pi.fused_general_eligible = general ? 1 : 0;
    if (!general) {
        for (int p = 0; p < DS_MAX_PLANES; ++p) pi.general_band_reps[p] = pi.general_strips[p] = 0;
        pi.general_units_per_frame = pi.general_stage_bytes_max = 0;
    }
    *info = pi;
    if (spec_out) *spec_out = spec;
    return DS_OK;
}

// ----------------------------------------------------------- K-N1 launch --
// Launch shape from a band plan: enough consumer warps for one task each
// (cap 8), up to kK1Ctas CTAs per SM, and rings that together hold
// ~kInFlightTarget bytes in flight per SM (tools/bw_probe: ~120 KB/SM is the
// TMA optimum), at least 2 stages each.  Several CTAs per SM overlap one
// unit's synchronisation with another's work.  Measured against one CTA with a
// ~120 KB ring (profiles/r01/k1_small_sweep.txt, k1_ctas_ab.txt): PAL SD, CIF
// and QCIF +28-34%, 4K 4:2:0 +5%, HD 4:4:4 +2.4%, HD 4:2:0 even.
int max_tasks(const ds_plan_info& pi) {
    int t = 0;
    for (int p = 0; p < pi.n_planes; ++p)
        t = std::max(t, 2 * pi.band_groups[p] * ((pi.in_w[p] + 15) / 16));
    return t;
}

// plane kinds of a K-N1 plan: bit 0 wide, bit 1 whole-band, bit 2 narrow
int plan_modes(const ds_plan_info& pi) {
    int m = 0;
    for (int p = 0; p < pi.n_planes; ++p)
        m |= pi.in_w[p] % 16 != 0 ? 4 : k1_whole_band(pi.in_w[p]) ? 2 : 1;
    return m;
}

// Consumer warps for K-N1: fewer than 8 only for tiny planes.  (More than 8
// was measured: no gain on CIF / SD at 11-12 warps, and 16 warps were slower
// on HD, so a unit's 2 k chunks tasks are spread over 256 threads in rounds.)
int pick_ncw(const ds_plan_info& pi) {
    const int w = (max_tasks(pi) + 31) / 32;
    return w <= 1 ? 1 : w <= 2 ? 2 : w <= 4 ? 4 : 8;
}

FusedCfg make_cfg(const ds_plan_info& pi) {
    FusedCfg c;
    c.plan = pi;
    if (!pi.fused_eligible) return c;
    c.ncw = pick_ncw(pi);
    c.stage_stride = (int32_t)round_up(pi.unit_in_bytes_max, 128);
    c.out_stride = (int32_t)round_up(pi.unit_out_bytes_max, 128);
    c.stages = (int)std::max<int64_t>(
        2, std::min<int64_t>(8, (kInFlightTarget + kK1Ctas * c.stage_stride / 2) / (kK1Ctas * c.stage_stride)));
    c.ctas_per_sm = kK1Ctas;
    if (pi.in_frame_bytes < kSmallFrameBytes) {
        // small frames (8 KB bands): as many CTAs per SM as fit, 3-deep rings
        // (QCIF x 2000: 0.58 -> 0.66 of the copy peak, profiles/r02/k1_small_sweep.txt)
        c.stages = 3;
        c.ctas_per_sm = 0;
    }
    c.valid = true;
    return c;
}

int prepare_cfg(FusedCfg& c);
int configure_fused(ds_handle* h) {
    h->fused = make_cfg(h->plan);
    h->fine = FusedCfg{};
    if (!h->plan.fused_eligible) return DS_OK;
    ds_plan_info fp;
    if (make_plan(h->W, h->H, h->channels, &h->spec, nullptr, &fp,
                  std::min<int64_t>(kFineUnitTarget, h->band_target)) == DS_OK &&
        fp.fused_eligible && fp.units_per_frame > h->plan.units_per_frame)
        h->fine = make_cfg(fp);
    DeviceGuard g(h->device);
    int rc = prepare_cfg(h->fused);
    if (!rc) rc = prepare_cfg(h->fine);
    // Wide plans (2 CTAs per SM) on calls of up to ~3 GB of input: one CTA per
    // SM with a 4-deep ring of the same units measured 2-4% faster (HD 4:2:0
    // 150-900 frames, HD 4:4:4 300, 4K 100-150), and 1.5-7% slower on longer
    // calls (HD 1200/3000, HD 4:4:4 600, 4K 300/1000); CIF/SD plans (3 CTAs
    // per SM) lose 20-26% at one CTA (profiles/r02/k1_cta_ab*.txt).
    h->onecta = FusedCfg{};
    if (!rc && h->fused.valid && h->fused.grid_per_sm == 2) {
        FusedCfg c = h->fused;
        c.stages = 4;
        c.ctas_per_sm = 1;
        if (prepare_cfg(c) == DS_OK && c.grid_per_sm == 1) h->onecta = c;
    }
    return rc;
}

using FusedFn = void (*)(const ds::FusedParams);

// Instantiations: 8 consumer warps for every combination of plane kinds a
// plan can have (bit 0 wide, 1 whole-band, 2 narrow); tiny plans (1/2/4
// warps) get the all-kinds kernel.
FusedFn fused_fn(int ncw, int modes) {
    switch (ncw) {
        case 1: return ds::ds_fused_band_kernel<1, 7>;
        case 2: return ds::ds_fused_band_kernel<2, 7>;
        case 4: return ds::ds_fused_band_kernel<4, 7>;
        default: break;
    }
    switch (modes) {
        case 1: return ds::ds_fused_band_kernel<8, 1>;
        case 2: return ds::ds_fused_band_kernel<8, 2>;
        case 3: return ds::ds_fused_band_kernel<8, 3>;
        case 4: return ds::ds_fused_band_kernel<8, 4>;
        case 5: return ds::ds_fused_band_kernel<8, 5>;
        case 6: return ds::ds_fused_band_kernel<8, 6>;
        default: return ds::ds_fused_band_kernel<8, 7>;
    }
}

// Ring depth that fits, capped by the request.
int fit_stages(const FusedCfg& c, int want) {
    int s = std::max(2, std::min(8, want));
    while (s > 2 && fused_smem_bytes(s, c.stage_stride, c.out_stride) > kSmemLimit) --s;
    return s;
}

// Which configuration a call of n frames uses.
const FusedCfg& pick_cfg(const ds_handle* h, int64_t n) {
    if (h->fine.valid && n * h->fused.plan.units_per_frame < 2LL * h->sm_count) return h->fine;
    if (h->onecta.valid && n * h->plan.in_frame_bytes <= kOneCtaMaxBytes) return h->onecta;
    return h->fused;
}

// Resolve and cache the launch shape of a configuration on the current
// device (sets the kernel's dynamic shared-memory attribute once).
int prepare_cfg(FusedCfg& c) {
    if (!c.valid) return DS_OK;
    const int stages = fit_stages(c, c.stages);
    const int sm = (int)fused_smem_bytes(stages, c.stage_stride, c.out_stride);
    const int threads = (c.ncw + 1) * 32;
    FusedFn fn = fused_fn(c.ncw, plan_modes(c.plan));
    // the attribute belongs to the kernel function (shared by every handle and
    // configuration using this instantiation): always the opt-in maximum
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit) !=
        cudaSuccess) {
        cudaGetLastError();
        return DS_ECUDA;
    }
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, sm) != cudaSuccess ||
        occ < 1) {
        cudaGetLastError();
        return DS_ECUDA;
    }
    if (c.ctas_per_sm > 0) occ = std::min(occ, c.ctas_per_sm);
    c.grid_per_sm = occ;
    c.threads = threads;
    c.smem = sm;
    c.run_stages = stages;
    return DS_OK;
}

int fused_grid(const ds_handle* h, const FusedCfg& c, int64_t n_units, int* grid, int* block,
               int* smem) {
    if (c.grid_per_sm < 1) return DS_ECUDA;
    const int64_t g = std::min<int64_t>(n_units, (int64_t)c.grid_per_sm * h->sm_count);
    *grid = (int)std::max<int64_t>(g, 1);
    *block = c.threads;
    *smem = c.smem;
    return DS_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int launch_fused(ds_handle* h, const uint8_t* in, int64_t n, uint8_t* out, cudaStream_t st) {
    const FusedCfg& c = pick_cfg(h, n);
    const ds_plan_info& pi = c.plan;
    ds::FusedParams p;
    std::memset(&p, 0, sizeof p);
    p.in = in; p.out = out;
    p.unit_count = h->debug_unit_count;
    p.in_frame = pi.in_frame_bytes; p.out_frame = pi.out_frame_bytes;
    p.upf = (int32_t)pi.units_per_frame;
    p.n_units = n * pi.units_per_frame;
    p.n_planes = pi.n_planes;
    p.stage_stride = c.stage_stride;
    p.out_stride = c.out_stride;
    const bool out_al = aligned16(out) && pi.out_frame_bytes % 16 == 0;
    int32_t start = 0;
    for (int q = 0; q < pi.n_planes; ++q) {
        ds::FusedPlane& P = p.pl[q];
        P.in_off = pi.in_offset[q];
        P.out_off = pi.out_offset[q];
        P.W = pi.in_w[q];
        P.Wout = pi.out_w[q];
        P.k = pi.band_groups[q];
        P.narrow = (P.W % 16 != 0) ? 1 : 0;
        P.whole = k1_whole_band(P.W) ? 1 : 0;
        P.chunks = (P.W + 15) / 16;
        P.tasks = 2 * P.k * P.chunks;
        P.chunks_rcp = P.chunks > 1 ? (uint32_t)((0x100000000ULL + P.chunks - 1) / P.chunks) : 0u;
        P.unit_start = start;
        P.unit_in = (P.narrow || P.whole ? 9 : 8) * P.k * P.W;
        P.unit_out = 4 * P.k * P.Wout;
        P.bulk_store = (out_al && P.out_off % 16 == 0 && P.unit_out % 16 == 0) ? 1 : 0;
        start += pi.in_h[q] / (9 * P.k);
    }
    int grid, block, smem;
    int rc = fused_grid(h, c, p.n_units, &grid, &block, &smem);
    if (rc) return rc;
    p.stages = c.run_stages;
    fused_fn(c.ncw, plan_modes(c.plan))<<<grid, block, smem, st>>>(p);
    return cudaGetLastError() == cudaSuccess ? DS_OK : DS_ECUDA;
}

// ------------------------------------------------------------ K-N1g launch --
using GeneralFn = void (*)(const ds::GeneralParams);

int64_t general_smem(const GeneralCfg& c, int stages) {
    return (int64_t)stages * c.stage_stride + c.mid_stride + c.mid_alt + 2LL * c.out_stride + (2LL * stages + 1) * 8;
}

// K-N1g run lengths for a launch over n frames: with a V halo, a unit is a
// run of L_p consecutive bands of one plane (the halo's mid rows carry over).
// Runs grow (by work per band, split evenly within a plane) while the
// launch keeps >= 16 units per CTA slot, so the persistent schedule's tail
// stays <= ~1/16 (tools/general_perf.py --run-bands sweep: 8 HD luma bands
// per run beat 1, 2, 4, 16 and whole planes).  Returns units per frame.
int32_t general_runs(const ds_handle* h, int64_t n, int32_t* L) {
    const GeneralCfg& c = h->general;
    const ds_plan_info& pi = h->plan;
    int64_t bb[DS_MAX_PLANES], bbmax = 1;
    for (int q = 0; q < pi.n_planes; ++q) {
        L[q] = 1;
        bb[q] = (int64_t)c.R[q] * c.geom[q].pitch;
        bbmax = std::max(bbmax, bb[q]);
    }
    auto upf_of = [&](const int32_t* l) {
        int32_t u = 0;
        for (int q = 0; q < pi.n_planes; ++q) u += c.geom[q].strips * ((c.nb[q] + l[q] - 1) / l[q]);
        return u;
    };
    if (c.mid_alt == 0) return upf_of(L);
    if (h->run_bands > 0) {
        for (int q = 0; q < pi.n_planes; ++q) L[q] = std::min<int32_t>(h->run_bands, c.nb[q]);
        return upf_of(L);
    }
    const int64_t slots = std::max<int64_t>(1, (int64_t)c.grid_per_sm * h->sm_count);
    for (int64_t T = 2 * bbmax; T <= 64 * bbmax; T *= 2) {
        int32_t l[DS_MAX_PLANES];
        for (int q = 0; q < pi.n_planes; ++q) {
            const int64_t want = std::max<int64_t>(1, std::min<int64_t>(c.nb[q], T / bb[q]));
            const int64_t runs = (c.nb[q] + want - 1) / want;
            l[q] = (int32_t)((c.nb[q] + runs - 1) / runs);      // equal runs within the plane
        }
        if (n * upf_of(l) < 16 * slots) break;
        for (int q = 0; q < pi.n_planes; ++q) L[q] = l[q];
    }
    return upf_of(L);
}

// cs: some plane of the call is staged by the consumers (ds_fused_general_kernel)
GeneralFn general_fn(int fast, bool cs) {
    if (cs)
        return fast == 2 ? ds::ds_fused_general_kernel<2, true>
                         : fast == 1 ? ds::ds_fused_general_kernel<1, true> : ds::ds_fused_general_kernel<0, true>;
    return fast == 2 ? ds::ds_fused_general_kernel<2, false>
                     : fast == 1 ? ds::ds_fused_general_kernel<1, false> : ds::ds_fused_general_kernel<0, false>;
}

// Stage constants for K-N1g.  FASTDIV (M != 0): floor(a / D) = umulhi(a, M)
// with M = ceil(2^32 / D) is exact for 0 <= a <= amax when amax * e < 2^32,
// e = M D - 2^32 (the error a e / (D 2^32) stays below 1 / D).  amax is the
// largest accumulator any window can reach: bias + 255 * (sum of positive taps).
// D = 1 uses M = 2^32 - 1 with the accumulator biased by +1 (umulhi(a + 1,
// 2^32 - 1) = a) and a clamp floor of 1 instead of 0.
ds::GenStage gen_stage(const ds_stage_spec& s) {
    ds::GenStage g;
    std::memset(&g, 0, sizeof g);
    g.P = s.pattern; g.S = s.paving; g.Q = s.outputs; g.bias = s.bias;
    g.D = (uint32_t)s.divisor;
    g.D_rcp = s.divisor == 1 ? 0xffffffffu : (uint32_t)((1ULL << 32) / (uint64_t)s.divisor);
    std::memcpy(g.w, s.weight, sizeof g.w);
    g.s8 = 1;
    int64_t amax = 0, amin = INT64_MAX;
    for (int k = 0; k < DS_MAX_OUTPUTS; ++k) {
        int64_t pos = 0, neg = 0;
        for (int i = 0; i < DS_MAX_PATTERN; ++i) {
            const int32_t w = s.weight[k][i];
            if (w < -128 || w > 127) g.s8 = 0;
            g.wp[k][i / 4] |= (uint32_t)(uint8_t)(int8_t)(w < -128 ? 0 : w > 127 ? 0 : w) << (8 * (i % 4));
            if (k < s.outputs && i < s.pattern) (w > 0 ? pos : neg) += w;
        }
        if (k < s.outputs) {
            amax = std::max<int64_t>(amax, (int64_t)s.bias + 255 * pos);
            amin = std::min<int64_t>(amin, (int64_t)s.bias + 255 * neg);
        }
    }
    if (s.divisor == 1) {
        if (amax < (int64_t)0x7fffffff) { g.M = 0xffffffffu; g.lo = 1; g.fbias = s.bias + 1; }
    } else {
        const uint64_t D = (uint64_t)s.divisor;
        const uint64_t M = ((1ULL << 32) + D - 1) / D;
        const uint64_t e = M * D - (1ULL << 32);
        if (amax < (int64_t)0x7fffffff && (unsigned __int128)(uint64_t)amax * e < ((unsigned __int128)1 << 32)) {
            g.M = (uint32_t)M; g.lo = 0; g.fbias = s.bias;
        }
    }
    // both clamps dead: every accumulator is >= 0 and its quotient <= 255
    g.exact = (g.M != 0 && amin >= 0 && amax < 256 * (int64_t)s.divisor) ? 1 : 0;
    return g;
}

int configure_general(ds_handle* h) {
    GeneralCfg c;
    const ds_plan_info& pi = h->plan;
    if (!pi.fused_general_eligible) { h->general = c; return DS_OK; }
    const ds_filter_spec& sp = h->spec;
    int64_t smax = 0, mmax = 0, omax = 0;
    for (int p = 0; p < pi.n_planes; ++p) {
        c.geom[p] = general_plane_geom(sp, pi.in_w[p], pi.in_h[p], general_stage_target(sp, h->general_target));
        c.k[p] = c.geom[p].k;
        c.nb[p] = (pi.in_h[p] / sp.v.paving) / c.k[p];
        c.R[p] = c.geom[p].R;
        smax = std::max<int64_t>(smax, (int64_t)c.R[p] * c.geom[p].pitch);
        mmax = std::max<int64_t>(mmax, (int64_t)(c.R[p] + 3) * c.geom[p].wm_max);   // V reads 4-row blocks
        omax = std::max<int64_t>(omax, (int64_t)sp.v.outputs * c.k[p] * c.geom[p].wm_max);
    }
    c.stage_stride = (int32_t)round_up(smax, 128);
    c.mid_stride = (int32_t)round_up(mmax, 128);
    c.ovl = std::max(0, sp.v.pattern - sp.v.paving);
    c.mid_alt = c.ovl > 0 ? c.mid_stride : 0;     // second mid buffer for halo reuse
    c.out_stride = (int32_t)round_up(omax, 128);
    // K-N1g is issue-bound (tools/general_perf.py sweep, profiles/r01/general.md):
    // 2 CTAs x 8 consumer warps per SM with a 2-deep ring beat deeper rings
    // and 16-warp CTAs
    c.stages = 2;
    c.ncw = DS_GEN_NCW;
#ifndef DS_GEN_CTAS
#define DS_GEN_CTAS 2
#endif
    const int want_ctas = DS_GEN_CTAS;
    c.threads = (c.ncw + 1) * 32;
    c.smem = (int)general_smem(c, c.stages);
    const ds::GenStage gh = gen_stage(sp.h), gv = gen_stage(sp.v);
    c.fast = (gh.M == 0 || gv.M == 0) ? 0 : (gh.exact && gv.exact) ? 2 : 1;
    DeviceGuard g(h->device);
    int occ_min = 1 << 30;
    for (bool cs : {false, true}) {
        GeneralFn fn = general_fn(c.fast, cs);
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSmemLimit - 2 * DS_MAX_OUTPUTS * DS_MAX_PATTERN * 4) != cudaSuccess) {
            cudaGetLastError();
            return DS_ECUDA;
        }
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, c.threads, c.smem) != cudaSuccess || occ < 1) {
            cudaGetLastError();
            return DS_ECUDA;
        }
        occ_min = std::min(occ_min, occ);
    }
    c.grid_per_sm = std::min(occ_min, want_ctas);

    c.valid = true;
    h->general = c;
    return DS_OK;
}

uint32_t rcp32(int32_t d) { return d > 1 ? (uint32_t)((0x100000000ULL + d - 1) / (uint64_t)d) : 0u; }

int launch_general(ds_handle* h, const uint8_t* in, int64_t n, uint8_t* out, cudaStream_t st) {
    const GeneralCfg& c = h->general;
    const ds_plan_info& pi = h->plan;
    const ds_filter_spec& sp = h->spec;
    ds::GeneralParams p;
    std::memset(&p, 0, sizeof p);
    p.in = in; p.out = out;
    p.unit_count = h->debug_unit_count;
    p.in_frame = pi.in_frame_bytes; p.out_frame = pi.out_frame_bytes;
    int32_t L[DS_MAX_PLANES] = {1, 1, 1};
    p.upf = general_runs(h, n, L);
    p.n_units = n * p.upf;
    bool cs = false;
    p.n_planes = pi.n_planes;
    p.stages = c.stages;
    p.stage_stride = c.stage_stride;
    p.mid_stride = c.mid_stride;
    p.out_stride = c.out_stride;
    p.ovl = c.ovl;
    p.mid_alt = c.mid_alt;
    p.h = gen_stage(sp.h);
    p.v = gen_stage(sp.v);
    const bool out_al = aligned16(out) && pi.out_frame_bytes % 16 == 0;
    const bool in_al = aligned16(in);
    int32_t start = 0;
    for (int q = 0; q < pi.n_planes; ++q) {
        ds::GenPlane& P = p.pl[q];
        P.in_off = pi.in_offset[q];
        P.out_off = pi.out_offset[q];
        P.W = pi.in_w[q];
        P.H = pi.in_h[q];
        P.Wm = pi.out_w[q];
        P.k = c.k[q];
        P.R = c.R[q];
        P.np = P.W / sp.h.paving;
        P.np_rcp = rcp32(P.np);
        P.wm_rcp = rcp32(P.Wm);
        P.quads_rcp = rcp32(P.Wm / 4);
        P.oh = (int32_t)(((int64_t)sp.h.origin % P.W + P.W) % P.W);
        P.ov = (int32_t)(((int64_t)sp.v.origin % P.H + P.H) % P.H);
        P.unit_start = start;
        P.nb = c.nb[q];
        P.L = L[q];
        const GenGeom& gg = c.geom[q];
        P.strips = gg.strips;
        P.sw = gg.sw;
        P.runs = (P.nb + P.L - 1) / P.L;
        P.runs_rcp = rcp32(P.runs);
        auto groups = [](int np) { return np <= DS_GEN_NCW * 32 ? (DS_GEN_NCW * 32) / np : 1; };   // threads / np
        if (gg.strips > 1) {
            // per-strip geometry: regular strips (sw repetitions) and the last one
            P.np_rcp = rcp32(gg.sw);
            P.wm_rcp = rcp32(sp.h.outputs * gg.sw);
            P.quads_rcp = rcp32(sp.h.outputs * gg.sw / 4);
            P.hgroups = groups(gg.sw);
            P.np_last = gg.np_last;
            P.np_rcp_last = rcp32(gg.np_last);
            P.wm_rcp_last = rcp32(sp.h.outputs * gg.np_last);
            P.quads_rcp_last = rcp32(sp.h.outputs * gg.np_last / 4);
            P.hgroups_last = groups(gg.np_last);
        } else {
            P.hgroups = groups(P.np);
        }
        P.unit_out = sp.v.outputs * P.k * P.Wm;
        P.bulk_store = (out_al && P.out_off % 16 == 0 && P.unit_out % 16 == 0) ? 1 : 0;
        P.bulk_rows = (out_al && P.out_off % 16 == 0 && P.Wm % 16 == 0) ? 1 : 0;
        P.coop = (in_al && P.W % 16 == 0 && P.W >= 32 && P.in_off % 16 == 0 && pi.in_frame_bytes % 16 == 0)
                     ? 0 : 1;
        P.pitch = gg.pitch;
        // consumer staging (the device's g_coop_async test, for every frame)
        if (P.coop && (P.strips > 1 || ((reinterpret_cast<uintptr_t>(in) + P.in_off) & 3) != 0 || (P.W & 3) != 0 ||
                       (n > 1 && (pi.in_frame_bytes & 3) != 0)))
            cs = true;
        start += P.strips * P.runs;
    }
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(p.n_units, (int64_t)c.grid_per_sm * h->sm_count));
    general_fn(c.fast, cs)<<<(unsigned)grid, c.threads, c.smem, st>>>(p);
    return cudaGetLastError() == cudaSuccess ? DS_OK : DS_ECUDA;
}

int launch_generic(ds_handle* h, const uint8_t* in, int64_t n, uint8_t* out, cudaStream_t st) {
    const ds_plan_info& pi = h->plan;
    ds::GenericParams p;
    std::memset(&p, 0, sizeof p);
    p.in = in; p.out = out;
    p.in_frame = pi.in_frame_bytes; p.out_frame = pi.out_frame_bytes;
    p.total_out = n * pi.out_frame_bytes;
    p.n_planes = pi.n_planes;
    for (int q = 0; q < pi.n_planes; ++q) {
        p.in_off[q] = pi.in_offset[q];
        p.out_off[q] = pi.out_offset[q];
        p.W[q] = pi.in_w[q];
        p.H[q] = pi.in_h[q];
        p.Wout[q] = pi.out_w[q];
    }
    p.h = h->spec.h;
    p.v = h->spec.v;
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>((p.total_out + threads - 1) / threads,
                                             (int64_t)h->sm_count * 8);
    ds::ds_generic_kernel<<<(int)std::max<int64_t>(blocks, 1), threads, 0, st>>>(p);
    return cudaGetLastError() == cudaSuccess ? DS_OK : DS_ECUDA;
}

// K-N1 needs 16-byte rows and a 16-byte-aligned input (TMA); K-N1g stages
// unaligned rows itself; K-N2 takes whatever neither can (no smem fit).
int choose_kernel(const ds_handle* h, const uint8_t* in) {
    if (h->kernel_pref == DS_KERNEL_GENERIC) return DS_KERNEL_GENERIC;
    const bool k1 = h->plan.fused_eligible && h->fused.valid && aligned16(in);
    const bool k1g = h->plan.fused_general_eligible && h->general.valid;
    if (h->kernel_pref == DS_KERNEL_FUSED) return k1 ? DS_KERNEL_FUSED : DS_KERNEL_GENERIC;
    if (h->kernel_pref == DS_KERNEL_FUSED_GENERAL) return k1g ? DS_KERNEL_FUSED_GENERAL : DS_KERNEL_GENERIC;
    return k1 ? DS_KERNEL_FUSED : k1g ? DS_KERNEL_FUSED_GENERAL : DS_KERNEL_GENERIC;
}


bool device_ptr_on(const void* p, int dev) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) return false;
    return a.device == dev;
}

// Output memory the kernels of handle h may write: device memory of h's
// device, or of a peer GPU the caller has enabled explicitly with
// ds_enable_peer (e.g. another rank's buffer mapped with CUDA IPC: the fused
// compute + gather of dist.py).  No side effects: ds_run never enables peer
// access itself (a pointer not on the handle's device is DS_EINVAL).
bool out_ptr_ok(const ds_handle* h, const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) return false;
    if (a.device == h->device) return true;
    return a.device >= 0 && a.device < 64 && ((h->peer_mask.load() >> a.device) & 1ull);
}

bool ranges_overlap(const void* a, int64_t na, const void* b, int64_t nb) {
    const uintptr_t x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
    return x < y + (uintptr_t)nb && y < x + (uintptr_t)na;
}

// K-N1g family: the compiled-spec instance (K-N1s) when the handle has one
// and the call's pointers allow it, else the runtime-tap kernel
bool use_spec(const ds_handle* h, const uint8_t* in, const uint8_t* out) {
    return h->general_variant != 1 && spec_call_ok(h, in, out);
}

int run_device(ds_handle* h, const uint8_t* in, int64_t n, uint8_t* out, cudaStream_t st) {
    const int k = choose_kernel(h, in);
    int rc, variant = 0;
    if (k == DS_KERNEL_FUSED) {
        rc = launch_fused(h, in, n, out, st);
    } else if (k == DS_KERNEL_FUSED_GENERAL) {
        variant = use_spec(h, in, out) ? 2 : 1;
        rc = variant == 2 ? launch_spec(h, in, n, out, st) : launch_general(h, in, n, out, st);
    } else {
        rc = launch_generic(h, in, n, out, st);
    }
    if (rc == DS_OK) {
        h->last_kernel.store(k);
        h->last_variant.store(variant);
    }
    return rc;
}

// Host -> device copy of m frames for the fused path.  With SPEC's taps row
// 9g+4 of every plane has zero V weight and no kernel reads it, so
// only rows 0..3 and 5..8 of each 9-row group cross PCIe: per plane one
// strided 3-D copy per half when the frame stride is a whole number of
// 9-row pitches, else one 2-D copy per frame and half.  Returns bytes copied
// (< 0 on error).  The skipped rows of the device buffer stay stale.
int64_t live_rows_h2d(const ds_handle* h, uint8_t* dst, const uint8_t* src, int64_t m,
                      cudaStream_t st) {
    const ds_plan_info& pi = h->plan;
    ds_filter_spec def;
    default_spec(&def);
    const int64_t fin = pi.in_frame_bytes;
    if (!(stage_equal(h->spec.v, def.v) && stage_equal(h->spec.h, def.h) && pi.fused_eligible)) {
        if (cudaMemcpyAsync(dst, src, m * fin, cudaMemcpyHostToDevice, st) != cudaSuccess) return -1;
        return m * fin;
    }
    int64_t bytes = 0;
    for (int p = 0; p < pi.n_planes; ++p) {
        const int64_t W = pi.in_w[p], G = pi.in_h[p] / 9, pitch = 9 * W;
        for (int half = 0; half < 2; ++half) {
            const int64_t off = pi.in_offset[p] + (half ? 5 : 0) * W;
            if (fin % pitch == 0) {
                cudaMemcpy3DParms c;
                std::memset(&c, 0, sizeof c);
                c.srcPtr = make_cudaPitchedPtr(const_cast<uint8_t*>(src) + off, (size_t)pitch, (size_t)(4 * W),
                                               (size_t)(fin / pitch));
                c.dstPtr = make_cudaPitchedPtr(dst + off, (size_t)pitch, (size_t)(4 * W), (size_t)(fin / pitch));
                c.extent = make_cudaExtent((size_t)(4 * W), (size_t)G, (size_t)m);
                c.kind = cudaMemcpyHostToDevice;
                if (cudaMemcpy3DAsync(&c, st) != cudaSuccess) return -1;
            } else {
                for (int64_t f = 0; f < m; ++f)
                    if (cudaMemcpy2DAsync(dst + f * fin + off, (size_t)pitch, src + f * fin + off, (size_t)pitch,
                                          (size_t)(4 * W), (size_t)G, cudaMemcpyHostToDevice, st) != cudaSuccess)
                        return -1;
            }
            bytes += m * G * 4 * W;
        }
    }
    return bytes;
}

void free_host_state(ds_handle* h) {
    for (auto& s : h->slots) {
        if (s.stream) cudaStreamSynchronize(s.stream);
        if (s.d_in) cudaFree(s.d_in);
        if (s.d_out) cudaFree(s.d_out);
        if (s.done) cudaEventDestroy(s.done);
        if (s.stream) cudaStreamDestroy(s.stream);
        s = HostSlot{};
    }
    if (h->fork_ev) cudaEventDestroy(h->fork_ev);
    h->fork_ev = nullptr;
    h->host_alloc_frames = 0;
    h->host_init = false;
}

}  // namespace dsi


// ================================================================ C ABI ==
extern "C" {

DS_API int ds_default_spec(ds_filter_spec* out) {
    if (!out) return DS_EINVAL;
    default_spec(out);
    return DS_OK;
}

DS_API int ds_plan(int32_t frame_w, int32_t frame_h, int32_t channels,
                   const ds_filter_spec* spec, ds_plan_info* out) {
    if (!out) return DS_EINVAL;
    return make_plan(frame_w, frame_h, channels, spec, nullptr, out);
}

DS_API ds_handle* ds_create(int32_t frame_w, int32_t frame_h, int32_t channels,
                            const ds_filter_spec* filter_spec) {
    ds_filter_spec spec;
    ds_plan_info pi;
    int rc = make_plan(frame_w, frame_h, channels, filter_spec, &spec, &pi);
    if (rc) { g_last_error = rc; return nullptr; }
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
        cudaGetLastError();
        g_last_error = DS_ECUDA;
        return nullptr;
    }
    ds_handle* h = new (std::nothrow) ds_handle();
    if (!h) { g_last_error = DS_ENOMEM; return nullptr; }
    h->device = dev;
    h->sm_count = sms;
    h->W = frame_w; h->H = frame_h; h->channels = channels;
    h->spec = spec;
    h->plan = pi;
    h->band_target = default_band_target(pi.in_frame_bytes);
    if (h->band_target != kUnitTargetBytes) {
        ds_plan_info ps;
        if (make_plan(frame_w, frame_h, channels, &spec, nullptr, &ps, h->band_target) == DS_OK) h->plan = ps;
    }
    int crc = configure_fused(h);
    if (!crc) crc = configure_general(h);
    if (!crc) crc = configure_spec(h);
    if (crc) {
        delete h;
        g_last_error = crc;
        return nullptr;
    }
    g_last_error = DS_OK;
    return h;
}

DS_API int ds_run(ds_handle* h, const uint8_t* in, int64_t n, uint8_t* out, ds_stream_t stream) {
    if (!h || n < 0) return DS_EINVAL;
    if (n == 0) return DS_OK;
    if (!in || !out) return DS_EINVAL;
    const int64_t nin = n * h->plan.in_frame_bytes, nout = n * h->plan.out_frame_bytes;
    if (ranges_overlap(in, nin, out, nout)) return DS_EINVAL;
    DeviceGuard g(h->device);
    if (!g.ok) { cudaGetLastError(); return DS_ECUDA; }
    if (!device_ptr_on(in, h->device) || !out_ptr_ok(h, out)) return DS_EINVAL;
    return run_device(h, in, n, out, reinterpret_cast<cudaStream_t>(stream));
}

DS_API int ds_enable_peer(ds_handle* h, int32_t peer_device) {
    if (!h || peer_device < 0 || peer_device >= 64) return DS_EINVAL;
    if (peer_device == h->device) return DS_OK;
    int count = 0, can = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) { cudaGetLastError(); return DS_ECUDA; }
    if (peer_device >= count) return DS_EINVAL;
    if (cudaDeviceCanAccessPeer(&can, h->device, peer_device) != cudaSuccess) {
        cudaGetLastError();
        return DS_ECUDA;
    }
    if (!can) return DS_EUNSUPPORTED;
    DeviceGuard g(h->device);
    if (!g.ok) { cudaGetLastError(); return DS_ECUDA; }
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return DS_ECUDA;
    }
    cudaGetLastError();                            // clear "already enabled"
    h->peer_mask.fetch_or(1ull << peer_device);
    return DS_OK;
}

DS_API int ds_set_host_chunk(ds_handle* h, int64_t frames) {
    if (!h || frames < 0) return DS_EINVAL;
    std::lock_guard<std::mutex> lk(h->host_mu);
    h->host_chunk = frames;
    return DS_OK;
}

DS_API int ds_run_host(ds_handle* h, const uint8_t* host_in, int64_t n, uint8_t* host_out,
                       ds_stream_t stream) {
    if (!h || n < 0) return DS_EINVAL;
    if (n == 0) return DS_OK;
    if (!host_in || !host_out) return DS_EINVAL;
    const int64_t fin = h->plan.in_frame_bytes, fout = h->plan.out_frame_bytes;
    if (ranges_overlap(host_in, n * fin, host_out, n * fout)) return DS_EINVAL;
    std::lock_guard<std::mutex> lk(h->host_mu);
    DeviceGuard g(h->device);
    if (!g.ok) { cudaGetLastError(); return DS_ECUDA; }
    cudaStream_t caller = reinterpret_cast<cudaStream_t>(stream);
    int64_t chunk = h->host_chunk > 0 ? h->host_chunk
                                      : std::max<int64_t>(1, kHostChunkBytes / std::max<int64_t>(fin, 1));
    chunk = std::min(chunk, n);
    if (!h->host_init) {
        for (auto& s : h->slots) {
            if (cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking) != cudaSuccess ||
                cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming) != cudaSuccess) {
                cudaGetLastError();
                free_host_state(h);
                return DS_ECUDA;
            }
        }
        if (cudaEventCreateWithFlags(&h->fork_ev, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            free_host_state(h);
            return DS_ECUDA;
        }
        h->host_init = true;
    }
    if (h->host_alloc_frames < chunk) {
        // grow the staging buffers stream-ordered on each slot's stream: the
        // old buffers are released after the slot's queued work, and no
        // device-wide synchronisation (cudaFree) stalls other streams
        // (allocations are 256-byte aligned, as the K-N1 bulk copies need)
        for (auto& s : h->slots) {
            if (s.d_in) cudaFreeAsync(s.d_in, s.stream);
            if (s.d_out) cudaFreeAsync(s.d_out, s.stream);
            s.d_in = s.d_out = nullptr;
        }
        h->host_alloc_frames = 0;
        for (auto& s : h->slots) {
            if (cudaMallocAsync(reinterpret_cast<void**>(&s.d_in), chunk * fin, s.stream) != cudaSuccess ||
                cudaMallocAsync(reinterpret_cast<void**>(&s.d_out), chunk * fout, s.stream) != cudaSuccess) {
                cudaGetLastError();
                free_host_state(h);
                return DS_ENOMEM;
            }
        }
        h->host_alloc_frames = chunk;
    }
    // fork: internal streams start after the work already queued on `stream`
    if (cudaEventRecord(h->fork_ev, caller) != cudaSuccess) { cudaGetLastError(); return DS_ECUDA; }
    for (auto& s : h->slots)
        if (cudaStreamWaitEvent(s.stream, h->fork_ev, 0) != cudaSuccess) { cudaGetLastError(); return DS_ECUDA; }
    // chunk c on slot c % 3: H2D -> kernel -> D2H in stream order; slots
    // overlap each other's copies (two copy engines) and compute.
    int64_t c = 0;
    for (int64_t f0 = 0; f0 < n; f0 += chunk, ++c) {
        const int64_t m = std::min(chunk, n - f0);
        HostSlot& s = h->slots[c % kHostSlots];
        if (live_rows_h2d(h, s.d_in, host_in + f0 * fin, m, s.stream) < 0) {
            cudaGetLastError();
            return DS_ECUDA;
        }
        int rc = run_device(h, s.d_in, m, s.d_out, s.stream);
        if (rc) return rc;
        if (cudaMemcpyAsync(host_out + f0 * fout, s.d_out, m * fout, cudaMemcpyDeviceToHost,
                            s.stream) != cudaSuccess) { cudaGetLastError(); return DS_ECUDA; }
    }
    // join: `stream` waits for every slot
    for (auto& s : h->slots) {
        if (cudaEventRecord(s.done, s.stream) != cudaSuccess ||
            cudaStreamWaitEvent(caller, s.done, 0) != cudaSuccess) { cudaGetLastError(); return DS_ECUDA; }
    }
    return DS_OK;
}

DS_API void ds_destroy(ds_handle* h) {
    if (!h) return;
    {
        std::lock_guard<std::mutex> lk(h->host_mu);
        DeviceGuard g(h->device);
        free_host_state(h);
        free_sched_state(h);
    }
    delete h;
}

DS_API int ds_last_error(void) { return g_last_error; }

DS_API const char* ds_strerror(int code) {
    switch (code) {
        case DS_OK: return "ok";
        case DS_EINVAL: return "invalid argument";
        case DS_ESHAPE: return "plane shape not divisible by the tiler paving (S:551)";
        case DS_EUNSUPPORTED: return "unsupported channels or filter spec";
        case DS_ECUDA: return "CUDA runtime error";
        case DS_ENOMEM: return "out of memory";
        default: return "unknown error";
    }
}

DS_API int ds_get_plan(const ds_handle* h, ds_plan_info* out) {
    if (!h || !out) return DS_EINVAL;
    *out = h->plan;
    return DS_OK;
}

DS_API int64_t ds_in_frame_bytes(const ds_handle* h) { return h ? h->plan.in_frame_bytes : -1; }
DS_API int64_t ds_out_frame_bytes(const ds_handle* h) { return h ? h->plan.out_frame_bytes : -1; }

DS_API int ds_plane_dims(const ds_handle* h, int plane, int32_t* in_w, int32_t* in_h,
                         int32_t* out_w, int32_t* out_h) {
    if (!h || plane < 0 || plane >= h->plan.n_planes) return DS_EINVAL;
    if (in_w) *in_w = h->plan.in_w[plane];
    if (in_h) *in_h = h->plan.in_h[plane];
    if (out_w) *out_w = h->plan.out_w[plane];
    if (out_h) *out_h = h->plan.out_h[plane];
    return DS_OK;
}

DS_API int ds_set_kernel(ds_handle* h, int32_t kernel) {
    if (!h) return DS_EINVAL;
    if (kernel != DS_KERNEL_AUTO && kernel != DS_KERNEL_FUSED && kernel != DS_KERNEL_GENERIC &&
        kernel != DS_KERNEL_FUSED_GENERAL)
        return DS_EINVAL;
    if (kernel == DS_KERNEL_FUSED && !h->plan.fused_eligible) return DS_EUNSUPPORTED;
    if (kernel == DS_KERNEL_FUSED_GENERAL && !h->plan.fused_general_eligible) return DS_EUNSUPPORTED;
    h->kernel_pref = kernel;
    return DS_OK;
}

DS_API int ds_last_kernel(const ds_handle* h) { return h ? h->last_kernel.load() : DS_EINVAL; }

DS_API int ds_set_tuning(ds_handle* h, int32_t stages, int32_t ctas_per_sm) {
    if (!h || stages < 2 || stages > 8 || ctas_per_sm < 0 || ctas_per_sm > 32) return DS_EINVAL;
    FusedCfg c = h->fused;
    c.stages = stages;
    c.ctas_per_sm = ctas_per_sm;
    DeviceGuard g(h->device);
    const int rc = prepare_cfg(c);
    if (rc) return rc;
    h->fused = c;
    h->fine = FusedCfg{};          // an explicit tuning applies to every call size
    h->onecta = FusedCfg{};
    h->tune_stages = stages;       // kept across ds_set_band_bytes / ds_set_general_stage_bytes
    h->tune_ctas = ctas_per_sm;
    return DS_OK;
}

// Re-plan the handle with new band / stage targets: the new plan and its
// configurations are committed only if all of them succeed (a failure leaves
// the handle exactly as it was), and an explicit ds_set_tuning is re-applied.
static int replan(ds_handle* h, int64_t band_target, int64_t general_target) {
    ds_plan_info pi;
    int rc = make_plan(h->W, h->H, h->channels, &h->spec, nullptr, &pi, band_target, general_target);
    if (rc) return rc;
    const ds_plan_info old_plan = h->plan;
    const FusedCfg old_fused = h->fused, old_fine = h->fine, old_onecta = h->onecta;
    const GeneralCfg old_general = h->general;
    const int64_t old_band = h->band_target, old_gen = h->general_target;
    h->plan = pi;
    h->band_target = band_target;
    h->general_target = general_target;
    const SpecCfg old_spec = h->spec_cfg;
    rc = configure_fused(h);
    if (!rc) rc = configure_general(h);
    if (!rc) rc = configure_spec(h);
    if (!rc && h->tune_stages > 0 && h->fused.valid) {
        FusedCfg c = h->fused;
        c.stages = h->tune_stages;
        c.ctas_per_sm = h->tune_ctas;
        DeviceGuard g(h->device);
        rc = prepare_cfg(c);
        if (!rc) {
            h->fused = c;
            h->fine = FusedCfg{};
            h->onecta = FusedCfg{};
        }
    }
    if (rc) {
        h->plan = old_plan;
        h->fused = old_fused;
        h->fine = old_fine;
        h->onecta = old_onecta;
        h->general = old_general;
        h->spec_cfg = old_spec;
        h->band_target = old_band;
        h->general_target = old_gen;
    }
    return rc;
}

DS_API int ds_set_band_bytes(ds_handle* h, int64_t target) {
    if (!h || target < 0) return DS_EINVAL;
    if (target == 0) target = default_band_target(h->plan.in_frame_bytes);
    return replan(h, target, h->general_target);
}

DS_API int ds_set_general_stage_bytes(ds_handle* h, int64_t target) {
    if (!h || target < 0) return DS_EINVAL;
    return replan(h, h->band_target, target);
}

DS_API int ds_set_run_bands(ds_handle* h, int32_t bands) {
    if (!h || bands < 0) return DS_EINVAL;
    h->run_bands = bands;
    return DS_OK;
}

DS_API int ds_set_debug_counter(ds_handle* h, uint32_t* counts) {
    if (!h) return DS_EINVAL;
    h->debug_unit_count = counts;
    return DS_OK;
}

DS_API int64_t ds_units(const ds_handle* h, int64_t n, int32_t kernel) {
    if (!h || n < 0) return -1;
    if (kernel == DS_KERNEL_FUSED) return h->plan.fused_eligible ? n * pick_cfg(h, n).plan.units_per_frame : -1;
    if (kernel == DS_KERNEL_FUSED_GENERAL) {
        if (h->general_variant != DS_GENERAL_RUNTIME && h->spec_cfg.valid) {
            int32_t L[DS_MAX_PLANES], upf = 0;
            spec_runs(h, n, L, &upf);
            return n * upf;
        }
        if (!h->general.valid) return -1;
        int32_t L[DS_MAX_PLANES];
        return n * general_runs(h, n, L);
    }
    return -1;
}

DS_API int ds_set_general_variant(ds_handle* h, int32_t variant) {
    if (!h || variant < DS_GENERAL_AUTO || variant > DS_GENERAL_COMPILED) return DS_EINVAL;
    if (variant == DS_GENERAL_COMPILED && !h->spec_cfg.valid) {
        // no built-in instance: compile K-N1s for this spec now (NVRTC)
        h->spec_jit_req = true;
        const int rc = configure_spec(h);
        if (rc) return rc;
        if (!h->spec_cfg.valid) return DS_EUNSUPPORTED;
    }
    if (variant == DS_GENERAL_RUNTIME && !h->general.valid) return DS_EUNSUPPORTED;
    h->general_variant = variant;
    return DS_OK;
}

DS_API int ds_last_variant(const ds_handle* h) { return h ? h->last_variant.load() : DS_EINVAL; }

DS_API int ds_launch_shape(const ds_handle* h, int64_t n, int32_t* grid, int32_t* block,
                           int32_t* smem) {
    if (!h || n < 0 || !h->plan.fused_eligible) return DS_EINVAL;
    DeviceGuard g(h->device);
    int gr, bl, sm;
    const FusedCfg& c = pick_cfg(h, n);
    const int rc = fused_grid(h, c, std::max<int64_t>(1, n * c.plan.units_per_frame), &gr, &bl, &sm);
    if (rc) return rc;
    if (grid) *grid = gr;
    if (block) *block = bl;
    if (smem) *smem = sm;
    return DS_OK;
}

DS_API int ds_launch_info(const ds_handle* h, int64_t n, int32_t kernel, ds_launch* out) {
    if (!h || n < 0 || !out) return DS_EINVAL;
    std::memset(out, 0, sizeof *out);
    out->kernel = kernel;
    if (kernel == DS_KERNEL_FUSED) {
        if (!h->plan.fused_eligible || !h->fused.valid) return DS_EUNSUPPORTED;
        const FusedCfg& c = pick_cfg(h, n);
        int gr, bl, sm;
        const int rc = fused_grid(h, c, std::max<int64_t>(1, n * c.plan.units_per_frame), &gr, &bl, &sm);
        if (rc) return rc;
        out->grid = gr; out->block = bl; out->smem_bytes = sm;
        out->stages = c.run_stages;
        out->ctas_per_sm = c.grid_per_sm;
        out->consumer_warps = c.ncw;
        out->units = n * c.plan.units_per_frame;
        out->unit_in_bytes_max = c.plan.unit_in_bytes_max;
        return DS_OK;
    }
    if (kernel == DS_KERNEL_FUSED_GENERAL && h->general_variant != DS_GENERAL_RUNTIME && h->spec_cfg.valid) {
        const SpecCfg& c = h->spec_cfg;
        int32_t L[DS_MAX_PLANES], upf = 0;
        spec_runs(h, n, L, &upf);
        const int64_t units = n * upf;
        out->grid = (int32_t)std::max<int64_t>(1, std::min<int64_t>(units, (int64_t)c.grid_per_sm * h->sm_count));
        out->block = c.threads; out->smem_bytes = c.smem;
        out->stages = c.stages;
        out->ctas_per_sm = c.grid_per_sm;
        out->consumer_warps = DS_SPEC_NW;
        out->units = units;
        out->unit_in_bytes_max = 0;             // no input staging: loads go to registers
        out->variant = c.jit ? 3 : 2;
        return DS_OK;
    }
    if (kernel == DS_KERNEL_FUSED_GENERAL) {
        const GeneralCfg& c = h->general;
        if (!h->plan.fused_general_eligible || !c.valid) return DS_EUNSUPPORTED;
        out->variant = 1;
        int32_t L[DS_MAX_PLANES];
        const int64_t units = n * general_runs(h, n, L);
        out->grid = (int32_t)std::max<int64_t>(1, std::min<int64_t>(units, (int64_t)c.grid_per_sm * h->sm_count));
        out->block = c.threads; out->smem_bytes = c.smem;
        out->stages = c.stages;
        out->ctas_per_sm = c.grid_per_sm;
        out->consumer_warps = c.ncw;
        out->units = units;
        out->unit_in_bytes_max = h->plan.general_stage_bytes_max;
        return DS_OK;
    }
    if (kernel == DS_KERNEL_GENERIC) {
        out->block = 256;
        const int64_t total_out = n * h->plan.out_frame_bytes;
        out->grid = (int32_t)std::max<int64_t>(1, std::min<int64_t>((total_out + 255) / 256, (int64_t)h->sm_count * 8));
        out->units = total_out;
        return DS_OK;
    }
    return DS_EINVAL;
}

DS_API int ds_generate(uint8_t* dev, int64_t n_bytes, uint64_t seed, int64_t start,
                       ds_stream_t stream) {
    if (n_bytes < 0 || start < 0 || (n_bytes > 0 && !dev)) return DS_EINVAL;
    if (n_bytes == 0) return DS_OK;
    int d = 0, sms = 0;
    if (cudaGetDevice(&d) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d) != cudaSuccess) {
        cudaGetLastError();
        return DS_ECUDA;
    }
    const int threads = 256;
    const int64_t blocks =
        std::min<int64_t>((n_bytes / 16 + threads) / threads, (int64_t)sms * 16);
    ds::ds_generate_kernel<<<(int)std::max<int64_t>(blocks, 1), threads, 0,
                             reinterpret_cast<cudaStream_t>(stream)>>>(
        dev, n_bytes, seed * 0x9E3779B97F4A7C15ull, start, aligned16(dev) ? 1 : 0);
    return cudaGetLastError() == cudaSuccess ? DS_OK : DS_ECUDA;
}

}  // extern "C"
