// ds_spec.cu -- host side of K-N1s (ds_spec.cuh): the fused band kernel with
// the filter spec compiled in.  Planning (strips, bands, strides), the
// built-in instances, eligibility and the launch.  Any spec without a
// built-in instance is compiled at run time (ds_spec_jit.cu).
// Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, SURVEY sec. n.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ds.h"
#include "ds_internal.h"
#include "ds_spec.cuh"
#include "ds_spec_builtin.cuh"

namespace dsi {

namespace {

bool stage_is(const ds_stage_spec& s, int P, int S, int Q, int D, int B, int O, int (*w)(int, int)) {
    if (s.pattern != P || s.paving != S || s.outputs != Q || s.divisor != D || s.bias != B || s.origin != O)
        return false;
    for (int j = 0; j < DS_MAX_OUTPUTS; ++j)
        for (int i = 0; i < DS_MAX_PATTERN; ++i)
            if (s.weight[j][i] != ((j < Q && i < P) ? w(j, i) : 0)) return false;
    return true;
}
template <class ST>
int wfn(int j, int i) { return ST::w(j, i); }
template <class ST>
bool stage_is(const ds_stage_spec& s) {
    return stage_is(s, ST::P, ST::S, ST::Q, ST::D, ST::B, ST::O, &wfn<ST>);
}

// words of an H chunk window (the HChunk<> constants, from the runtime spec):
// first and last word read from the chunk's first block, 16-byte blocks touched
void h_words(const ds_stage_spec& h, int ph, int* klo, int* khi) {
    int hi = 0;
    for (int j = 0; j < h.outputs; ++j)
        for (int i = 0; i < h.pattern; ++i)
            if (h.weight[j][i] != 0) hi = std::max(hi, i);
    *klo = ph / 4;
    *khi = (ph + 3 * h.paving + hi) / 4;
}
int64_t floor16(int64_t o) { return o >= 0 ? o / 16 : -((-o + 15) / 16); }

// Lanes of a row of nch chunks: segs 32-chunk warp segments (a power of two
// dividing NW), or, for rows of at most 16 chunks, 2^lgrpw rows per warp of
// 32 >> lgrpw chunk lanes each.  A warp's row step, (NW / segs) 2^lgrpw, stays
// below the plane height H (the row cursor wraps with one subtraction).
bool spec_lanes(int nch, int H, int* segs, int* lgrpw) {
    int s = 1;
    while (32 * s < nch) s *= 2;
    if (s > DS_SPEC_NW || H <= DS_SPEC_NW / s) return false;
    int lg = 0;
    if (s == 1)
        while (lg < 5 && (32 >> (lg + 1)) >= nch && (DS_SPEC_NW << (lg + 1)) < H) ++lg;
    *segs = s;
    *lgrpw = lg;
    return true;
}

// instance slots: row alignment 16, 8, 4, unaligned (1), and 16-byte rows 4 / 8 /
// 12 bytes past a boundary (17 / 18 / 19)
int al_index(int al) { return al == 16 ? 0 : al == 8 ? 1 : al == 4 ? 2 : al == 1 ? 3 : al - 13; }

}  // namespace

// The H origin of a plane reduced to (-W/2, W/2]: window bytes are taken mod W
// (S:251), so this is the same filter, and the windows of every chunk not
// crossing the row end start at this value's phase mod 16.
int64_t spec_h_origin(int64_t origin, int64_t W) {
    int64_t o = (origin % W + W) % W;
    if (o > W / 2) o -= W;
    return o;
}

// The window phase every plane shares (the instance's PH), or -1.
int spec_phase(const ds_filter_spec& sp, const ds_plan_info& pi) {
    int ph = -1;
    for (int p = 0; p < pi.n_planes; ++p) {
        const int q = (int)((spec_h_origin(sp.h.origin, pi.in_w[p]) % 16 + 16) % 16);
        if (ph >= 0 && q != ph) return -1;
        ph = q;
    }
    return ph;
}

// Alignment (16, 8 or 4; 0: none) of every row start of a frame-aligned call:
// frame size, plane offsets and row widths.
int spec_plan_align(const ds_plan_info& pi) {
    int64_t a = pi.in_frame_bytes;
    for (int p = 0; p < pi.n_planes; ++p) a |= pi.in_offset[p] | pi.in_w[p];
    return a % 16 == 0 ? 16 : a % 8 == 0 ? 8 : a % 4 == 0 ? 4 : 0;
}

// Built-in instances: (stage types, window phase, row alignment) -> kernel.
SpecFn spec_builtin(const ds_filter_spec& sp, int ph, int al) {
    auto pick = [al](auto k16, auto k8, auto k4, auto k1, auto k17, auto k18, auto k19) {
        switch (al) {
            case 16: return reinterpret_cast<SpecFn>(k16);
            case 8: return reinterpret_cast<SpecFn>(k8);
            case 4: return reinterpret_cast<SpecFn>(k4);
            case 17: return reinterpret_cast<SpecFn>(k17);
            case 18: return reinterpret_cast<SpecFn>(k18);
            case 19: return reinterpret_cast<SpecFn>(k19);
            default: return reinterpret_cast<SpecFn>(k1);
        }
    };
    constexpr int kHaloPh = (dss::HaloH::O % 16 + 16) % 16, kSpecPh = (dss::SpecH::O % 16 + 16) % 16;
    if (ph == kHaloPh && stage_is<dss::HaloH>(sp.h) && stage_is<dss::HaloV>(sp.v))
        return pick(&dss::ds_spec_kernel<dss::HaloH, dss::HaloV, kHaloPh, 16>,
                    &dss::ds_spec_kernel<dss::HaloH, dss::HaloV, kHaloPh, 8>,
                    &dss::ds_spec_kernel<dss::HaloH, dss::HaloV, kHaloPh, 4>,
                    &dss::ds_spec_kernel<dss::HaloH, dss::HaloV, kHaloPh, 1>,
                    &dss::ds_spec_kernel<dss::HaloH, dss::HaloV, kHaloPh, 17>,
                    &dss::ds_spec_kernel<dss::HaloH, dss::HaloV, kHaloPh, 18>,
                    &dss::ds_spec_kernel<dss::HaloH, dss::HaloV, kHaloPh, 19>);
    if (ph == kSpecPh && stage_is<dss::SpecH>(sp.h) && stage_is<dss::SpecV>(sp.v))
        return pick(&dss::ds_spec_kernel<dss::SpecH, dss::SpecV, kSpecPh, 16>,
                    &dss::ds_spec_kernel<dss::SpecH, dss::SpecV, kSpecPh, 8>,
                    &dss::ds_spec_kernel<dss::SpecH, dss::SpecV, kSpecPh, 4>,
                    &dss::ds_spec_kernel<dss::SpecH, dss::SpecV, kSpecPh, 1>,
                    &dss::ds_spec_kernel<dss::SpecH, dss::SpecV, kSpecPh, 17>,
                    &dss::ds_spec_kernel<dss::SpecH, dss::SpecV, kSpecPh, 18>,
                    &dss::ds_spec_kernel<dss::SpecH, dss::SpecV, kSpecPh, 19>);
    return nullptr;
}

// Geometry K-N1s can run, independent of pointers: H paving a multiple of 4
// (a chunk of 4 repetitions starts on a 16-byte block of its window), taps in
// s8 (dp4a), rows 4-byte aligned within the frame (W % 4 == 0 follows from
// W % Sh == 0), one window phase for all planes, at most DS_SPEC_MAXP planes.
bool spec_geometry_ok(const ds_filter_spec& sp, const ds_plan_info& pi) {
    if (sp.h.paving % 4 != 0 || pi.n_planes > DS_SPEC_MAXP) return false;
    for (const ds_stage_spec* s : {&sp.h, &sp.v})
        for (int j = 0; j < s->outputs; ++j)
            for (int i = 0; i < s->pattern; ++i)
                if (s->weight[j][i] < -128 || s->weight[j][i] > 127) return false;
    if (sp.h.pattern > 16 || sp.v.pattern > 16) return false;
    if (spec_plan_align(pi) == 0) return false;
    const int ph = spec_phase(sp, pi);
    if (ph < 0) return false;
    int klo, khi;
    h_words(sp.h, ph, &klo, &khi);
    const int kblk = (khi + 4) / 4;
    for (int p = 0; p < pi.n_planes; ++p) {
        const int W = pi.in_w[p];
        if (W < 64 || W / 16 < kblk) return false;        // a window fits in a row
        // at most 4 chunks per row may cross the row end (the wrap pass's table)
        const int np = W / sp.h.paving, nch = (np + 3) / 4;
        int segs, lgrpw;
        if (!spec_lanes(nch, pi.in_h[p], &segs, &lgrpw)) return false;
        const int64_t blk0 = floor16(spec_h_origin(sp.h.origin, W));
        int nwc = 0;
        for (int c = 0; c < nch; ++c) {
            const int64_t B = blk0 + (sp.h.paving / 4) * c;
            if (16 * B + 4 * klo < -W || 16 * B + 4 * (khi + 1) > 2 * W) return false;   // one wrap at most
            nwc += !(16 * B + 4 * klo >= 0 && 16 * B + 4 * (khi + 1) <= W);
        }
        if (nwc > 4) return false;
    }
    return true;
}

// Per-plane plan: bands of k V repetitions (the first band of a run stages
// R = Sv (k - 1) + Pv rows, later bands Sv k new rows, the V halo's rows
// carried over in the intermediate).  Scored per useful input row by the
// rounds of the H pass (8 warps over rows x 32-chunk segments), the V pass
// (256 threads over k x column quads) and a per-band barrier, under the
// shared-memory budget (two intermediate buffers) of 3 CTAs per SM.
bool spec_plane_plan(const ds_filter_spec& sp, int32_t W, int32_t H, int64_t budget, SpecPlaneCfg* out) {
    const int Sh = sp.h.paving, Qh = sp.h.outputs;
    const int Sv = sp.v.paving, Pv = sp.v.pattern;
    const int np = W / Sh, G = H / Sv;
    const int nch = (np + 3) / 4;
    int segs, lgrpw;
    if (!spec_lanes(nch, H, &segs, &lgrpw)) return false;
    const int rpw = 1 << lgrpw, cw = 32 >> lgrpw;
    const int64_t nq = ((int64_t)Qh * np + 3) / 4;
    // row stride: every chunk the row's lanes cover plus one scratch chunk (the
    // H pass's inactive lanes store there unconditionally), and every V quad
    const int64_t mp = round_up(std::max<int64_t>(4LL * Qh * ((int64_t)cw * segs + 1), 4 * nq), 16);
    const int ovl = std::max(0, Pv - Sv);
    double best = 1e300;
    bool found = false;
    for (int k = 1; k <= G; ++k) {
        if (G % k) continue;
        const int64_t R = (int64_t)Sv * (k - 1) + Pv;
        // + rpw - 1 rows: a warp's last pass may run past the band's rows on
        // its later row lanes; their (unread) results land there
        if (2 * (R + rpw - 1) * mp > budget) continue;
        const int64_t newrows = std::max<int64_t>(1, R - ovl);
        const int64_t per_pass = (int64_t)(DS_SPEC_NW / segs) * rpw;
        const double hr = (double)((newrows + per_pass - 1) / per_pass);
#if DS_SPEC_WS
        constexpr int ntv = DS_SPEC_NWV * 32;                  // the V warps
#else
        constexpr int ntv = DS_SPEC_NW * 32;
#endif
        const double vr = (double)((k * nq + ntv - 1) / ntv);
#if DS_SPEC_WS
        // H and V warps overlap: the slower group sets the pace
        const double cost = (std::max(90.0 * hr, 120.0 * vr) + 150.0) / ((double)Sv * k);
#else
        const double cost = (90.0 * hr + 120.0 * vr + 150.0) / ((double)Sv * k);
#endif
        if (cost < best * 0.999) {
            best = cost;
            found = true;
            out->k = k; out->nb = G / k; out->R = (int32_t)R; out->mp = (int32_t)mp;
            out->rows_alloc = (int32_t)(R + rpw - 1);
            out->strips = 1; out->sw = np; out->pitch = 0;
        }
    }
    return found;
}

// Configure K-N1s for the handle (h->spec_cfg.valid = false when it cannot
// run the geometry/spec, which is not an error).
int configure_spec(ds_handle* h) {
    SpecCfg c;
    const ds_plan_info& pi = h->plan;
    const ds_filter_spec& sp = h->spec;
    h->spec_cfg = c;
    if (!spec_geometry_ok(sp, pi)) return DS_OK;
    const int ph = spec_phase(sp, pi), al = spec_plan_align(pi);
    c.al = al;
    // built-in: an instance for the plan's row alignment and each lower one
    // (calls whose input pointer is less aligned than the plan), and the
    // funnel-shifting one for pointers that are not 4-byte aligned
    for (int a = al; a >= 4; a /= 2) c.fn_al[al_index(a)] = spec_builtin(sp, ph, a);
    c.fn_al[al_index(1)] = spec_builtin(sp, ph, 1);
    if (al == 16)
        for (int a = 17; a <= 19; ++a) c.fn_al[al_index(a)] = spec_builtin(sp, ph, a);
    SpecFn fn = c.fn_al[al_index(al)];
    c.jit = 0;
    if (!fn) {
        // no built-in instance: compile one at run time (NVRTC, ~0.3 s once per
        // spec and process); DS_SPEC_JIT=0 leaves such specs to the runtime-tap
        // kernel unless ds_set_general_variant(DS_GENERAL_COMPILED) asks for it
        const char* env = getenv("DS_SPEC_JIT");
        if (!h->spec_jit_req && env && env[0] == '0') return DS_OK;
        fn = spec_jit_kernel(h, ph, al);                               // nullptr when NVRTC is unavailable
        c.fn_al[al_index(al)] = fn;                                    // the plan's alignment only
        c.jit = 1;
    }
    if (!fn) return DS_OK;
#if DS_SPEC_WS                                           // 2 CTAs per SM
#ifndef DS_SPEC_BUDGET
#define DS_SPEC_BUDGET (100 * 1024)
#endif
#ifndef DS_SPEC_BUDGET_NARROW
#define DS_SPEC_BUDGET_NARROW (100 * 1024)
#endif
#endif
#ifndef DS_SPEC_BUDGET
#define DS_SPEC_BUDGET (54 * 1024)
#endif
#ifndef DS_SPEC_BUDGET_NARROW
#define DS_SPEC_BUDGET_NARROW (64 * 1024)
#endif
    // shared memory for the two intermediate buffers: 54 KB, or 64 KB when a
    // plane takes several rows per warp (short rows make a band of the larger
    // budget cheap; CIF / SD x 2000 halo: -5%; HD at 64 KB: +3%,
    // profiles/r02/k1s_budget_ab.txt).  3 CTAs per SM fit either way.
    bool narrow = false;
    for (int p = 0; p < pi.n_planes; ++p) {
        int segs, lgrpw;
        narrow |= spec_lanes((pi.in_w[p] / sp.h.paving + 3) / 4, pi.in_h[p], &segs, &lgrpw) && lgrpw > 0;
    }
    const int64_t budget = narrow ? DS_SPEC_BUDGET_NARROW : DS_SPEC_BUDGET;
    int64_t mmax = 0;
    for (int p = 0; p < pi.n_planes; ++p) {
        if (!spec_plane_plan(sp, pi.in_w[p], pi.in_h[p], budget, &c.plane[p])) return DS_OK;
        mmax = std::max<int64_t>(mmax, (int64_t)c.plane[p].rows_alloc * c.plane[p].mp);
    }
    c.stages = 0;
    c.stage_stride = 0;
    c.mid_stride = (int32_t)round_up(mmax, 128);
    c.threads = DS_SPEC_THREADS;
    c.smem = 2 * c.mid_stride;
    DeviceGuard g(h->device);
    int occ = 0;
    if (c.jit) {
        if (spec_jit_set_smem(fn, c.smem) || spec_jit_occupancy(fn, c.threads, c.smem, &occ) || occ < 1) return DS_OK;
    } else {
        for (SpecFn f : c.fn_al)
            if (f && cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          c.smem) != cudaSuccess) {
                cudaGetLastError();
                return DS_OK;
            }
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, reinterpret_cast<const void*>(fn), c.threads, c.smem) !=
                cudaSuccess ||
            occ < 1) {
            cudaGetLastError();
            return DS_OK;
        }
    }
    // CTAs per SM: up to 4 when a plane takes several rows per warp, else 3 --
    // wide rows make large bands, and a fourth CTA's prefetched band costs the
    // others theirs in L2 (HD halo: 0.239 ms at 4 CTAs, 0.213 at 3, with the
    // same 64-register build; QCIF / CIF x 2000: 4-7% faster at 4)
    c.grid_per_sm = std::min(occ, narrow ? 4 : 3);
    c.fn = fn;
    c.valid = true;
    h->spec_cfg = c;
    return DS_OK;
}

// Runs of bands for a launch over n frames (units per frame into *upf, run
// lengths into L): ds_set_run_bands forces them; otherwise see below.
void spec_runs(const ds_handle* h, int64_t n, int32_t* L, int32_t* upf) {
    const SpecCfg& c = h->spec_cfg;
    const ds_plan_info& pi = h->plan;
    const ds_filter_spec& sp = h->spec;
    if (h->run_bands > 0) {                       // ds_set_run_bands forces the run length
        int32_t u = 0;
        for (int p = 0; p < pi.n_planes; ++p) {
            L[p] = std::min<int32_t>(h->run_bands, c.plane[p].nb);
            u += (c.plane[p].nb + L[p] - 1) / L[p];
        }
        *upf = u;
        return;
    }
    // equal work per unit across planes: a band of plane p covers Sv k_p rows of
    // W_p bytes; runs are sized so the launch has ~4 units per CTA slot (longer runs
    // re-stage fewer halo rows and pay less per-unit setup, more units balance the
    // persistent schedule; 3 / 4 / 6 / 10 per slot measured 0.2320 / 0.2273 / 0.2287 /
    // 0.2384 ms on 300 HD halo frames)
    const int64_t slots = std::max<int64_t>(1, (int64_t)c.grid_per_sm * h->sm_count);
    double frame_work = 0;
    for (int p = 0; p < pi.n_planes; ++p) frame_work += (double)pi.in_w[p] * pi.in_h[p];
#ifndef DS_SPEC_UNITS_PER_SLOT
#define DS_SPEC_UNITS_PER_SLOT 4.0
#endif
    const double want_units = std::max<double>(1.0, DS_SPEC_UNITS_PER_SLOT * slots / std::max<int64_t>(n, 1));
    const double target = frame_work / want_units;                  // bytes of input per unit
    int32_t u = 0;
    for (int p = 0; p < pi.n_planes; ++p) {
        const double band_work = (double)sp.v.paving * c.plane[p].k * pi.in_w[p];
        const int32_t nb = c.plane[p].nb;
        int32_t l = (int32_t)std::max<double>(1.0, std::floor(target / band_work + 0.5));
        l = std::min(l, nb);
        const int32_t runs = (nb + l - 1) / l;
        L[p] = (nb + runs - 1) / runs;                                // even runs within the plane
        u += (nb + L[p] - 1) / L[p];
    }
    *upf = u;
}

// Instance for one call: the plan's row alignment lowered to the input
// pointer's (16, 8 or 4 bytes); nullptr when there is none (a pointer not
// 4-byte aligned, or a run-time compiled spec whose one instance needs more).
SpecFn spec_call_fn(const ds_handle* h, const uint8_t* in) {
    const SpecCfg& c = h->spec_cfg;
    if (!c.valid) return nullptr;
    const uintptr_t m16 = reinterpret_cast<uintptr_t>(in) & 15;
    if (c.al == 16 && m16 != 0 && (m16 & 3) == 0) {
        // 16-byte rows from a pointer 4, 8 or 12 bytes off: the word-shift
        // instance (16-byte block loads) when there is one
        if (SpecFn fs = c.fn_al[al_index(16 + (int)(m16 >> 2))]) return fs;
    }
    int a = c.al;
    while (a >= 4 && (reinterpret_cast<uintptr_t>(in) & (uintptr_t)(a - 1)) != 0) a /= 2;
    return c.fn_al[al_index(a >= 4 ? a : 1)];
}

bool spec_call_ok(const ds_handle* h, const uint8_t* in, const uint8_t* out) {
    (void)out;   // any output alignment: rows take 4-, 2- or 1-byte stores by their alignment
    return spec_call_fn(h, in) != nullptr;
}

int launch_spec(ds_handle* h, const uint8_t* in, int64_t n, uint8_t* out, cudaStream_t st) {
    const SpecCfg& c = h->spec_cfg;
    const ds_plan_info& pi = h->plan;
    const ds_filter_spec& sp = h->spec;
    // the kernel counts units in 32 bits: at most one unit per band per frame
    int64_t upf_max = 0;
    for (int q = 0; q < pi.n_planes; ++q) upf_max += c.plane[q].nb;
    const int64_t cap = std::max<int64_t>(1, (int64_t)INT32_MAX / std::max<int64_t>(upf_max, 1));
    if (n > cap) {
        for (int64_t off = 0; off < n; off += cap) {
            const int rc = launch_spec(h, in + off * pi.in_frame_bytes, std::min(cap, n - off),
                                       out + off * pi.out_frame_bytes, st);
            if (rc != DS_OK) return rc;
        }
        return DS_OK;
    }
    dss::SpecParams p;
    std::memset(&p, 0, sizeof p);
    p.in = in; p.out = out;
    p.unit_count = h->debug_unit_count;
    p.in_frame = pi.in_frame_bytes; p.out_frame = pi.out_frame_bytes;
    int32_t L[DS_MAX_PLANES] = {1, 1, 1}, upf = 0;
    spec_runs(h, n, L, &upf);
    p.upf = upf;
    p.n_units = n * upf;
    p.n_planes = pi.n_planes;
    p.mid_stride = c.mid_stride;
    p.ovl = std::max(0, sp.v.pattern - sp.v.paving);
    auto rcp = [](int32_t d) { return d > 1 ? (uint32_t)((0x100000000ULL + d - 1) / (uint64_t)d) : 0u; };
    int32_t start = 0;
    for (int q = 0; q < pi.n_planes; ++q) {
        const SpecPlaneCfg& g = c.plane[q];
        dss::SpecPlane& P = p.pl[q];
        P.in_off = pi.in_offset[q];
        P.out_off = pi.out_offset[q];
        P.W = pi.in_w[q];
        P.H = pi.in_h[q];
        P.Wout = pi.out_w[q];
        P.oh = (int32_t)spec_h_origin(sp.h.origin, P.W);
        P.ov = (int32_t)(((int64_t)sp.v.origin % P.H + P.H) % P.H);
        P.np = P.W / sp.h.paving;
        P.nch = (P.np + 3) / 4;
        if (!spec_lanes(P.nch, P.H, &P.segs, &P.lgrpw)) return DS_EUNSUPPORTED;   // configure_spec rules this out
        P.lgsegs = 0;
        while ((1 << P.lgsegs) < P.segs) ++P.lgsegs;
        P.nb16 = P.W / 16;
        P.blk0 = (int32_t)floor16(P.oh);
        // chunks whose window words are not all inside the row (wrap pass)
        int klo, khi;
        h_words(sp.h, (int)((P.oh % 16 + 16) % 16), &klo, &khi);
        P.nwc = 0;
        for (int c = 0; c < P.nch; ++c) {
            const int64_t B = P.blk0 + (sp.h.paving / 4) * c;
            if (!(16 * B + 4 * klo >= 0 && 16 * B + 4 * (khi + 1) <= P.W)) {
                if (P.nwc == 4) return DS_EUNSUPPORTED;         // configure_spec rules this out
                P.wch[P.nwc++] = c;
            }
        }
        P.k = g.k;
        P.nb = g.nb;
        P.L = L[q];
        P.nq = (sp.h.outputs * P.np + 3) / 4;
        P.nq_rcp = rcp(P.nq);
        P.mp = g.mp;
        P.unit_start = start;
        start += (P.nb + P.L - 1) / P.L;
    }
    p.in_mis = (int32_t)(reinterpret_cast<uintptr_t>(in) & 3);           // AL = 1 instances
    p.out_al4 = (reinterpret_cast<uintptr_t>(out) & 3) == 0 && pi.out_frame_bytes % 4 == 0;
    for (int q = 0; q < pi.n_planes; ++q)
        if (pi.out_offset[q] % 4 || pi.out_w[q] % 4) p.out_al4 = 0;
    if (p.n_units == 0) return DS_OK;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(p.n_units, (int64_t)c.grid_per_sm * h->sm_count));
    const SpecFn fn = spec_call_fn(h, in);
    if (!fn) return DS_EUNSUPPORTED;                                  // run_device checked spec_call_ok
    void* args[] = {&p};
    if (c.jit) return spec_jit_launch(fn, (unsigned)grid, (unsigned)c.threads, (unsigned)c.smem, st, args);
    if (cudaLaunchKernel(reinterpret_cast<const void*>(fn), dim3((unsigned)grid), dim3(c.threads), args,
                         (size_t)c.smem, st) != cudaSuccess) {
        cudaGetLastError();
        return DS_ECUDA;
    }
    return DS_OK;
}

}  // namespace dsi
