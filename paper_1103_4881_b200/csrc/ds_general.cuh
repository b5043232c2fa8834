// ds_general.cuh -- K-N1g: the fused band kernel for ANY separable stage spec
// (SURVEY f3): halos (pattern P > paving S) with toroidal wrap,
// origin != 0, other ratios, negative lobes, any divisor.
//
// Same persistent, warp-specialised TMA pipeline as K-N1.  A band is k V
// repetitions; they read input rows (o_v + S_v g + i) mod H for g in the
// band, i < P_v: R = S_v (k-1) + P_v consecutive rows modulo H, i.e. the band
// plus its halo (the bottom halo wraps to the plane's first rows).  A work
// unit is (frame, plane, column strip, run of L consecutive bands): with a V
// halo (P_v > S_v) each band after the first of a run copies the P_v - S_v
// intermediate rows it shares with the previous band (two mid buffers) and
// stages and H-filters only its S_v k new rows.
//
// Staging: whole rows at a pitch of round_up(W, 16) + 32 bytes -- the row,
// then a 32-byte pad holding its first bytes again (row[j mod W]), so an H
// window that wraps past the row end reads straight on into the pad.
// A plane too wide for the stage budget is split into column strips of S_w H
// repetitions (a multiple of 16): a unit then stages, per row, only its
// strip's input window (o_h + S_h a, width S_h (S_w - 1) + P_h, modulo W) as
// the 16-byte-aligned superset (two bulk copies when it wraps the row end)
// and stores its output rows strip-wise.  Unaligned planes are staged by the
// producer warp with plain loads.
//
// Consumers run the H task on every newly staged row into a u8 intermediate
// in shared memory -- column-fixed threads, one dp4a per 4 taps --
// then the V task from it (4x4 byte transposes + dp4a), stage the output band
// in shared memory and bulk-store it.  Divisions by runtime values are exact
// (truncation toward zero, then clamp): one multiply-high when the host
// proves the accumulator range allows it, else a reciprocal plus one
// correction step (g_out modes 0-2).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ds.h"
#include "ds_kernels.cuh"

// build-time tuning knob (tools/build_variant.sh): CTAs per SM the register
// budget is sized for
#ifndef DS_GEN_MINB
#define DS_GEN_MINB 2
#endif
#ifndef DS_GEN_NCW
#define DS_GEN_NCW 8              // consumer warps per CTA
#endif

namespace ds {

struct GenPlane {
    int64_t in_off, out_off;
    int32_t W, H, Wm;          // input row bytes, rows, output row bytes (= mid row bytes, whole rows)
    int32_t pitch;             // staged row stride: round_up(W, 16) + 32 (row, then wrap pad),
                               // or a strip window's stride (strips > 1)
    int32_t k;                 // V repetitions per band
    int32_t R;                 // staged rows of a run's first band = Sv (k-1) + Pv
    int32_t np;                // H repetitions per row = W / Sh
    uint32_t np_rcp;           // ceil(2^32 / np) (np > 1)
    uint32_t wm_rcp;           // ceil(2^32 / Wm) (Wm > 1)
    uint32_t quads_rcp;        // ceil(2^32 / (Wm / 4)) (Wm / 4 > 1)
    int32_t oh;                // H origin reduced mod W (>= 0)
    int32_t ov;                // V origin reduced mod H (>= 0)
    int32_t unit_start;        // first unit (run) of this plane within a frame
    int32_t nb;                // bands in the plane: (H / Sv) / k
    int32_t hgroups;           // H pass row groups: NC / np when np <= NC, else 1
    int32_t L;                 // bands per run (unit); consecutive bands reuse the halo's mid rows
    int32_t unit_out;          // Qv * k * Wm (output bytes of one band)
    int32_t bulk_store;
    int32_t coop;              // 1: rows staged by the producer warp with plain loads
    // column strips (strips > 1): strip j covers H repetitions [j sw, min((j+1) sw, np))
    int32_t strips, sw;        // strip count, repetitions per strip (last: np - (strips-1) sw)
    int32_t runs;              // runs of bands per strip: ceil(nb / L)
    int32_t np_last, hgroups_last;
    uint32_t np_rcp_last, quads_rcp_last, wm_rcp_last, sw_rcp, runs_rcp;
    int32_t bulk_rows;         // strips: output row segments may be bulk-stored (16-byte aligned)
};

// The part of a plane one unit covers: the whole width (strips == 1, staged
// rows = row + wrap pad) or one column strip (staged rows = the strip's input
// window from its 16-aligned superset).
struct GenView {
    int32_t np, wm, hgroups;   // H repetitions, mid/output bytes per row, H-pass row groups
    uint32_t np_rcp, wm_rcp, quads_rcp;
    int32_t col0;              // first output column of the unit (Qh * first repetition)
    int32_t cbase, cwrap;      // window start of repetition t: cbase + Sh t, minus cwrap once if >= cwrap
    int32_t unit_out;          // output bytes of one band: Qv k wm
    int32_t strip, run;
};

struct GenStage {
    int32_t P, S, Q, bias;
    uint32_t D, D_rcp;         // divisor and floor(2^32 / D) (D = 1: 0xffffffff)
    int32_t s8;                // 1: every weight fits in s8 -> dp4a fast path
    // FASTDIV: clamp(trunc(acc / D)) = min(umulhi(max(acc + fbias - bias, lo), M), 255)
    // with M = ceil(2^32 / D), exact while max_acc * (M D - 2^32) < 2^32 (host-checked);
    // D = 1: M = 2^32 - 1, accumulator biased by +1 and lo = 1
    int32_t fbias;             // accumulator start on the FASTDIV path (bias, or bias + 1 for D = 1)
    uint32_t M, lo;
    int32_t exact;             // FASTDIV and 0 <= acc < 256 D for every window: no clamps needed
    int32_t w[DS_MAX_OUTPUTS][DS_MAX_PATTERN];
    uint32_t wp[DS_MAX_OUTPUTS][DS_MAX_PATTERN / 4];   // s8-packed weights, 4 taps per word
};

struct GeneralParams {
    const uint8_t* in;
    uint8_t* out;
    uint32_t* unit_count;      // debug: +1 per unit processed, else null
    int64_t in_frame, out_frame, n_units;
    int32_t upf, n_planes, stages, stage_stride, mid_stride, out_stride;
    int32_t ovl;               // Pv - Sv > 0: mid rows a band shares with the next
    int32_t mid_alt;           // byte offset of the second mid buffer (0: one buffer)
    GenPlane pl[DS_MAX_PLANES];
    GenStage h, v;
};

// clamp_0^255(trunc(acc / D)), branch-free: a non-positive accumulator
// truncates to a non-positive quotient, which clamps to 0 -- so divide
// max(acc, 0) instead of branching on the sign.  floor(a / D) for
// 0 <= a < 2^32: q0 = umulhi(a, floor(2^32 / D)) is q or q - 1, one
// correction step makes it exact.
__device__ __forceinline__ uint32_t g_stage_out(int32_t acc, uint32_t D, uint32_t rcp) {
    const uint32_t a = (uint32_t)max(acc, 0);
    uint32_t q = __umulhi(a, rcp);
    q += (a - q * D >= D) ? 1u : 0u;
    return min(q, 255u);
}
// Division modes (host-chosen, both stages): 0 reciprocal + correction,
// 1 FASTDIV with clamps, 2 FASTDIV where the host proved lo <= acc and
// acc / D <= 255 for every window, so both clamps are dead: one IMAD.HI.
template <int FAST>
__device__ __forceinline__ uint32_t g_out(const GenStage& g, int32_t acc) {
    if (FAST == 2) return __umulhi((uint32_t)acc, g.M);
    if (FAST == 1) return min(__umulhi((uint32_t)max(acc, (int32_t)g.lo), g.M), 255u);
    return g_stage_out(acc, g.D, g.D_rcp);
}
template <int FAST>
__device__ __forceinline__ int32_t g_bias(const GenStage& g) {
    return FAST ? g.fbias : g.bias;
}
// d = c + sum_i a.u8[i] * b.s8[i]
__device__ __forceinline__ int32_t dp4a_us(uint32_t a, uint32_t b, int32_t c) {
    int32_t d;
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
// shared-window accesses on 32-bit shared addresses (no generic->shared
// conversion per access)
__device__ __forceinline__ uint32_t lds32s(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds8s(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts8s(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts32s(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ int32_t g_div_small(int32_t t, int32_t d, uint32_t rcp) {
    return d == 1 ? t : (int32_t)__umulhi((uint32_t)t, rcp);
}

// Unit -> (strip, run) and the strip's geometry.  a = first repetition of
// the strip, cs = its window start (o_h + S_h a) mod W; staged rows hold the
// window from the 16-aligned superset start x0 = cs & ~15, so repetition t of
// the strip starts at byte (cs - x0) + S_h t of its staged row.
__device__ __forceinline__ GenView g_view(const GenPlane& P, int Sh, int Qh, int Qv, int local) {
    GenView v;
    if (P.strips == 1) {
        v.np = P.np; v.wm = P.Wm; v.hgroups = P.hgroups;
        v.np_rcp = P.np_rcp; v.wm_rcp = P.wm_rcp; v.quads_rcp = P.quads_rcp;
        v.col0 = 0; v.cbase = P.oh; v.cwrap = P.W;
        v.unit_out = P.unit_out;
        v.strip = 0; v.run = local;
        return v;
    }
    v.strip = (int)__umulhi((uint32_t)local, P.runs_rcp);
    if (P.runs == 1) v.strip = local;
    v.run = local - v.strip * P.runs;
    const bool last = v.strip == P.strips - 1;
    v.np = last ? P.np_last : P.sw;
    v.wm = Qh * v.np;
    v.hgroups = last ? P.hgroups_last : P.hgroups;
    v.np_rcp = last ? P.np_rcp_last : P.np_rcp;
    v.wm_rcp = last ? P.wm_rcp_last : P.wm_rcp;
    v.quads_rcp = last ? P.quads_rcp_last : P.quads_rcp;
    const int a = v.strip * P.sw;
    v.col0 = Qh * a;
    const int64_t cs = ((int64_t)P.oh + (int64_t)Sh * a) % P.W;
    v.cbase = (int)(cs & 15);             // TMA superset phase (coop rows: staged from cs, see producer)
    if (P.coop) v.cbase = 0;
    v.cwrap = 0x7fffffff;
    v.unit_out = Qv * P.k * v.wm;
    return v;
}

// ---- H pass over one staged unit: item = (staged row r, H repetition r1),
// Q outputs into mid row r at 3 r1 ...  The window starts at
// c0 = (o_h + S_h r1) mod W < W and runs at most 19 bytes on, inside the row
// and its wrap pad: 5 aligned words byte-shifted into a 16-byte window (taps
// past P are zero in the packed weights), one dp4a per 4 taps.
template <int Q, int FAST>
__device__ __forceinline__ void g_h_dot(const GenStage& g, const uint32_t (&x)[4], uint32_t (&o)[Q]) {
#pragma unroll
    for (int j = 0; j < Q; ++j) {
        int32_t acc = dp4a_us(x[0], g.wp[j][0], g_bias<FAST>(g));
        acc = dp4a_us(x[1], g.wp[j][1], acc);
        acc = dp4a_us(x[2], g.wp[j][2], acc);
        acc = dp4a_us(x[3], g.wp[j][3], acc);
        o[j] = g_out<FAST>(g, acc);
    }
}
// One H item at window words wb (byte shift in sel) -> Q bytes at mo.
template <int Q, int FAST>
__device__ __forceinline__ void g_h_win(uint32_t wb, uint32_t sel, uint32_t (&x)[4]) {
    const uint32_t w0 = lds32s(wb), w1 = lds32s(wb + 4), w2 = lds32s(wb + 8), w3 = lds32s(wb + 12),
                   w4 = lds32s(wb + 16);
    x[0] = __byte_perm(w0, w1, sel);
    x[1] = __byte_perm(w1, w2, sel);
    x[2] = __byte_perm(w2, w3, sel);
    x[3] = __byte_perm(w3, w4, sel);
}
// H pass, column-fixed: a thread keeps one H repetition r1 (its window start
// c0, byte shift and mid column never change) and walks the staged rows, three
// rows per step (loads of all first: three independent chains; -0.5% halo,
// -1.2% SPEC taps against two), then two, then one.  With
// np <= NC the threads form G = NC / np row groups (thread -> (group, r1));
// with np > NC a thread takes columns tid, tid + NC, ... for every row.
template <int Q, int FAST, int NC>
__device__ __forceinline__ void g_h_pass(const GenStage& g, const GenPlane& P, const GenView& V, uint32_t st,
                                         uint32_t mid, int rows, int tid) {
    const int np = V.np;
    int r1 = tid, r = 0, G = 1;
    if (np <= NC) {
        G = V.hgroups;                                // NC / np
        r = g_div_small(tid, np, V.np_rcp);           // row group
        if (r >= G) return;                           // idle: NC % np threads
        r1 = tid - r * np;
    }
    for (; r1 < np; r1 += NC) {
        int c0 = V.cbase + g.S * r1;
        if (c0 >= V.cwrap) c0 -= V.cwrap;             // whole rows: oh < W and Sh*r1 < W
        const uint32_t sel = 0x3210u + 0x1111u * (uint32_t)(c0 & 3);
        const uint32_t wstep = G * P.pitch, mstep = G * V.wm;
        uint32_t wb = st + r * P.pitch + (c0 & ~3);
        uint32_t mo = mid + r * V.wm + Q * r1;
        int rr = r;
        for (; rr + 2 * G < rows; rr += 3 * G) {          // three rows per step, then two, then one
            uint32_t xa[4], xb[4], xc[4], oa[Q], ob[Q], oc[Q];
            g_h_win<Q, FAST>(wb, sel, xa);
            g_h_win<Q, FAST>(wb + wstep, sel, xb);
            g_h_win<Q, FAST>(wb + 2 * wstep, sel, xc);
            g_h_dot<Q, FAST>(g, xa, oa);
            g_h_dot<Q, FAST>(g, xb, ob);
            g_h_dot<Q, FAST>(g, xc, oc);
#pragma unroll
            for (int j = 0; j < Q; ++j) {
                sts8s(mo + j, oa[j]);
                sts8s(mo + mstep + j, ob[j]);
                sts8s(mo + 2 * mstep + j, oc[j]);
            }
            wb += 3 * wstep;
            mo += 3 * mstep;
        }
        for (; rr + G < rows; rr += 2 * G) {
            uint32_t xa[4], xb[4], oa[Q], ob[Q];
            g_h_win<Q, FAST>(wb, sel, xa);
            g_h_win<Q, FAST>(wb + wstep, sel, xb);
            g_h_dot<Q, FAST>(g, xa, oa);
            g_h_dot<Q, FAST>(g, xb, ob);
#pragma unroll
            for (int j = 0; j < Q; ++j) {
                sts8s(mo + j, oa[j]);
                sts8s(mo + mstep + j, ob[j]);
            }
            wb += 2 * wstep;
            mo += 2 * mstep;
        }
        if (rr < rows) {
            uint32_t xa[4], oa[Q];
            g_h_win<Q, FAST>(wb, sel, xa);
            g_h_dot<Q, FAST>(g, xa, oa);
#pragma unroll
            for (int j = 0; j < Q; ++j) sts8s(mo + j, oa[j]);
        }
        if (np <= NC) break;
    }
}
// Taps outside s8: byte loop (same item space, same window bounds)
template <int FAST, int NC>
__device__ __forceinline__ void g_h_pass_bytes(const GenStage& g, const int32_t (*w)[DS_MAX_PATTERN],
                                               const GenPlane& P, const GenView& V, uint32_t st, uint32_t mid,
                                               int rows, int tid) {
    const int np = V.np, items = rows * np;
    for (int it = tid; it < items; it += NC) {
        const int r = g_div_small(it, np, V.np_rcp);
        const int r1 = it - r * np;
        int c0 = V.cbase + g.S * r1;
        if (c0 >= V.cwrap) c0 -= V.cwrap;
        const uint32_t rowp = st + r * P.pitch + c0;
        const uint32_t mo = mid + r * V.wm + g.Q * r1;
        for (int j = 0; j < g.Q; ++j) {
            int32_t acc = g_bias<FAST>(g);
            for (int i = 0; i < g.P; ++i) acc += w[j][i] * (int32_t)lds8s(rowp + i);
            sts8s(mo + j, g_out<FAST>(g, acc));
        }
    }
}

// V outputs k0 .. k0+Q-1 of one 4-column group: 4x4 byte transposes turn 4
// mid rows x 4 columns into 4 column words, one dp4a per 4 taps.
template <int Q, int FAST>
__device__ __forceinline__ void g_v_quad(const GenStage& g, int k0, uint32_t mb, int Wm, uint32_t ob0) {
    int32_t acc[Q][4];
#pragma unroll
    for (int kk = 0; kk < Q; ++kk)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[kk][e] = g_bias<FAST>(g);
    const int nb = (g.P + 3) >> 2;                  // <= DS_MAX_PATTERN / 4
#pragma unroll
    for (int b4 = 0; b4 < DS_MAX_PATTERN / 4; ++b4) {
        if (b4 >= nb) break;
        const uint32_t rb = mb + 4 * b4 * Wm;
        const uint32_t r0 = lds32s(rb), r1 = lds32s(rb + Wm), r2 = lds32s(rb + 2 * Wm), r3 = lds32s(rb + 3 * Wm);
        const uint32_t ta = __byte_perm(r0, r1, 0x5140), tb = __byte_perm(r2, r3, 0x5140);
        const uint32_t tc = __byte_perm(r0, r1, 0x7362), td = __byte_perm(r2, r3, 0x7362);
        const uint32_t c0 = __byte_perm(ta, tb, 0x5410), c1 = __byte_perm(ta, tb, 0x7632),
                       c2 = __byte_perm(tc, td, 0x5410), c3 = __byte_perm(tc, td, 0x7632);
#pragma unroll
        for (int kk = 0; kk < Q; ++kk) {
            const uint32_t wq = g.wp[k0 + kk][b4];
            acc[kk][0] = dp4a_us(c0, wq, acc[kk][0]);
            acc[kk][1] = dp4a_us(c1, wq, acc[kk][1]);
            acc[kk][2] = dp4a_us(c2, wq, acc[kk][2]);
            acc[kk][3] = dp4a_us(c3, wq, acc[kk][3]);
        }
    }
#pragma unroll
    for (int kk = 0; kk < Q; ++kk) {
        const uint32_t o = g_out<FAST>(g, acc[kk][0]) | (g_out<FAST>(g, acc[kk][1]) << 8) |
                           (g_out<FAST>(g, acc[kk][2]) << 16) | (g_out<FAST>(g, acc[kk][3]) << 24);
        sts32s(ob0 + (k0 + kk) * Wm, o);
    }
}
// ---- V pass (Wm % 4 == 0, s8 taps): item = (V repetition gi, 4 mid columns);
// outputs in groups of at most 4 (QA, then QB) to bound live accumulators.
template <int QA, int QB, int FAST, int NC>
__device__ __forceinline__ void g_v_pass(const GenStage& g, const GenPlane& P, const GenView& V, uint32_t mid,
                                         uint32_t ob, int tid) {
    const int Wm = V.wm, quads = Wm >> 2, items = P.k * quads;
    for (int it = tid; it < items; it += NC) {
        const int gi = g_div_small(it, quads, V.quads_rcp);
        const int q = it - gi * quads;
        const uint32_t mb = mid + g.S * gi * Wm + 4 * q;
        const uint32_t ob0 = ob + (QA + QB) * gi * Wm + 4 * q;
        g_v_quad<QA, FAST>(g, 0, mb, Wm, ob0);
        if (QB > 0) g_v_quad<(QB > 0 ? QB : 1), FAST>(g, QA, mb, Wm, ob0);
    }
}
// V pass, general: item = output byte of the band
template <int FAST, int NC>
__device__ __forceinline__ void g_v_pass_bytes(const GenStage& g, const int32_t (*w)[DS_MAX_PATTERN],
                                               const GenPlane& P, const GenView& V, uint32_t mid, uint32_t ob,
                                               int tid) {
    const int Wm = V.wm;
    for (int it = tid; it < V.unit_out; it += NC) {
        const int orow = g_div_small(it, Wm, V.wm_rcp);
        const int c = it - orow * Wm;
        const int gi = orow / g.Q, kk = orow - gi * g.Q;
        const uint32_t mcol = mid + g.S * gi * Wm + c;
        int32_t acc = g_bias<FAST>(g);
        for (int i = 0; i < g.P; ++i) acc += w[kk][i] * (int32_t)lds8s(mcol + i * Wm);
        sts8s(ob + it, g_out<FAST>(g, acc));
    }
}

// Producer-warp staging of the `rows` rows (row0 + i) mod H of a plane the
// TMA cannot copy (unaligned rows or pointer): each staged row is the W row
// bytes, then the 32-byte wrap pad row[j mod W].  Items (row, word) are walked
// with incremental indices (a band of R > H rows wraps more than once: row
// indices reduce by a loop) and loaded kCoopBatch per lane before their stores:
// the shared destination and global source may alias as far as the compiler
// knows, so a plain load-store loop serialises on DRAM latency (SD/QCIF chroma
// rows are 22-90 words: one round trip per word per row).
constexpr int kCoopBatch = 8;
__device__ __forceinline__ void cp_async_ca(uint32_t dst, const void* src, int bytes) {
    if (bytes == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void g_coop_rows(uint8_t* dst, int pitch, const uint8_t* plane, int row0, int rows,
                                            int H, int W, int lane) {
    const int G = ((((uintptr_t)plane | (uintptr_t)W) & 7) == 0) ? 8
                  : ((((uintptr_t)plane | (uintptr_t)W) & 3) == 0) ? 4 : 0;
    if (G) {
        // 4- or 8-byte aligned rows: cp.async (no register staging), every copy
        // of the band in flight at once, one wait.  A row is W / G chunks, then
        // (W >= 32) the 32-byte pad as the row's first 32 / G chunks.
        const int nr = W / G, n = nr + (W >= 32 ? 32 / G : 0);
        const int total = rows * n;
        const uint32_t d0 = (uint32_t)__cvta_generic_to_shared(dst);
        int r = lane / n, x = lane - (lane / n) * n;
        for (int it = lane; it < total; it += 32) {
            int rr = row0 + r;
            while (rr >= H) rr -= H;
            const uint8_t* src = plane + (int64_t)rr * W + (int64_t)(x < nr ? x : x - nr) * G;
            cp_async_ca(d0 + (uint32_t)(r * pitch + x * G), src, G);
            x += 32;
            while (x >= n) { x -= n; ++r; }
        }
        if (W < 32) {                                // pad of a short row: row[j mod W]
            const int pc = lane % W;
            for (int i = 0; i < rows; ++i) {
                int rr = row0 + i;
                while (rr >= H) rr -= H;
                dst[(size_t)i * pitch + W + lane] = __ldg(plane + (int64_t)rr * W + pc);
            }
        }
        cp_async_wait_all();
        return;
    }
    if ((W & 3) == 0) {
        // misaligned plane, W % 4 == 0: every row has the same misalignment m,
        // and each staged word k (row bytes 4k..4k+3; pad words: row bytes
        // 4p..4p+3) is two aligned source words funnelled by m bytes.  The
        // second word holds a valid row byte, so it stays inside the allocation.
        const uint32_t m = (uint32_t)((uintptr_t)plane & 3);
        const uint32_t sel = 0x3210u + 0x1111u * m;
        const int nr = W >> 2, n = nr + (W >= 32 ? 8 : 0);
        const int total = rows * n;
        int r = lane / n, x = lane - (lane / n) * n;
        for (int it0 = 0; it0 < total; it0 += 32 * kCoopBatch) {
            uint32_t lo[kCoopBatch], hi[kCoopBatch];
            int dr[kCoopBatch], dx[kCoopBatch];
#pragma unroll
            for (int j = 0; j < kCoopBatch; ++j) {
                dr[j] = r;
                dx[j] = x;
                if (it0 + 32 * j + lane < total) {
                    int rr = row0 + r;
                    while (rr >= H) rr -= H;
                    const uint32_t* a = reinterpret_cast<const uint32_t*>(
                        plane + (int64_t)rr * W + 4 * (int64_t)(x < nr ? x : x - nr) - m);
                    lo[j] = __ldg(a);
                    hi[j] = __ldg(a + 1);
                }
                x += 32;
                while (x >= n) { x -= n; ++r; }
            }
#pragma unroll
            for (int j = 0; j < kCoopBatch; ++j)
                if (it0 + 32 * j + lane < total)
                    reinterpret_cast<uint32_t*>(dst + (size_t)dr[j] * pitch)[dx[j]] = __byte_perm(lo[j], hi[j], sel);
        }
        if (W < 32) {
            const int pc = lane % W;
            for (int i = 0; i < rows; ++i) {
                int rr = row0 + i;
                while (rr >= H) rr -= H;
                dst[(size_t)i * pitch + W + lane] = __ldg(plane + (int64_t)rr * W + pc);
            }
        }
        return;
    }
    const bool words = (((uintptr_t)plane | (uintptr_t)W) & 3) == 0;
    const int n = words ? W >> 2 : W;               // items per row
    const int total = rows * n;
    int r = lane / n, x = lane - (lane / n) * n;    // item lane
    for (int it0 = 0; it0 < total; it0 += 32 * kCoopBatch) {
        uint32_t v[kCoopBatch];
        int dr[kCoopBatch], dx[kCoopBatch];
#pragma unroll
        for (int j = 0; j < kCoopBatch; ++j) {
            dr[j] = r;
            dx[j] = x;
            if (it0 + 32 * j + lane < total) {
                int rr = row0 + r;
                while (rr >= H) rr -= H;
                const uint8_t* src = plane + (int64_t)rr * W;
                v[j] = words ? __ldg(reinterpret_cast<const uint32_t*>(src) + x) : (uint32_t)__ldg(src + x);
            }
            x += 32;
            while (x >= n) { x -= n; ++r; }
        }
#pragma unroll
        for (int j = 0; j < kCoopBatch; ++j) {
            if (it0 + 32 * j + lane < total) {
                uint8_t* d = dst + (size_t)dr[j] * pitch;
                if (words) reinterpret_cast<uint32_t*>(d)[dx[j]] = v[j];
                else d[dx[j]] = (uint8_t)v[j];
            }
        }
    }
    const int pc = lane < W ? lane : lane % W;      // pad column j -> row[j mod W]
    for (int i0 = 0; i0 < rows; i0 += kCoopBatch) {
        uint32_t v[kCoopBatch];
#pragma unroll
        for (int j = 0; j < kCoopBatch; ++j) {
            if (i0 + j < rows) {
                int rr = row0 + i0 + j;
                while (rr >= H) rr -= H;
                v[j] = __ldg(plane + (int64_t)rr * W + pc);
            }
        }
#pragma unroll
        for (int j = 0; j < kCoopBatch; ++j)
            if (i0 + j < rows) dst[(size_t)(i0 + j) * pitch + W + lane] = (uint8_t)v[j];
    }
}

// Producer-warp staging of one strip window row (plain loads): bytes
// row[(cs + j) mod W] for j < len.
// Strip windows of `rows` rows (row0 + i) mod H for planes the TMA cannot copy:
// staged word q of a row is window bytes 4q..4q+3, i.e. row[(cs + 4q + t) mod W]:
// two aligned source words funnelled by that address's misalignment (batched
// kCoopBatch per lane before the stores), or bytes for the one word per row
// that straddles the row end.  Writes up to 3 bytes past len (the pitch has
// room: >= len + 35).
__device__ __forceinline__ void g_coop_windows(uint8_t* dst, int pitch, const uint8_t* plane, int row0, int rows,
                                               int H, int W, int cs, int len, int lane) {
    const int n = (len + 3) >> 2;
    const int total = rows * n;
    int r = lane / n, x = lane - (lane / n) * n;
    for (int it0 = 0; it0 < total; it0 += 32 * kCoopBatch) {
        uint32_t v[kCoopBatch];
        int dr[kCoopBatch], dx[kCoopBatch];
#pragma unroll
        for (int j = 0; j < kCoopBatch; ++j) {
            dr[j] = r;
            dx[j] = x;
            if (it0 + 32 * j + lane < total) {
                int rr = row0 + r;
                while (rr >= H) rr -= H;
                const uint8_t* row = plane + (int64_t)rr * W;
                int c = cs + 4 * x;
                while (c >= W) c -= W;
                if (c + 3 < W) {
                    const uintptr_t a = (uintptr_t)(row + c);
                    const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
                    v[j] = __byte_perm(__ldg(w), __ldg(w + 1), 0x3210u + 0x1111u * (uint32_t)(a & 3));
                } else {
                    uint32_t b = 0;
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const int ct = c + t >= W ? c + t - W : c + t;   // c < W, so one wrap at most
                        b |= (uint32_t)__ldg(row + ct) << (8 * t);
                    }
                    v[j] = b;
                }
            }
            x += 32;
            while (x >= n) { x -= n; ++r; }
        }
#pragma unroll
        for (int j = 0; j < kCoopBatch; ++j)
            if (it0 + 32 * j + lane < total)
                reinterpret_cast<uint32_t*>(dst + (size_t)dr[j] * pitch)[dx[j]] = v[j];
    }
}

// rows of this plane go by cp.async (4- or 8-byte aligned pointer and W)
__device__ __forceinline__ bool g_coop_async(const uint8_t* plane, int W) {
    return (((uintptr_t)plane | (uintptr_t)W) & 3) == 0;
}
template <int NT>
__device__ __forceinline__ void gc_pads_nt(uint8_t* dst, int pitch, const uint8_t* plane, int row0, int rows,
                                            int H, int W, int t) {
    const int total = rows * 32;
    for (int it0 = 0; it0 < total; it0 += NT * kCoopBatch) {
        uint32_t v[kCoopBatch];
#pragma unroll
        for (int j = 0; j < kCoopBatch; ++j) {
            const int it = it0 + NT * j + t;
            if (it < total) {
                int rr = row0 + (it >> 5);
                while (rr >= H) rr -= H;
                const int jc = it & 31;
                v[j] = __ldg(plane + (int64_t)rr * W + (jc < W ? jc : jc % W));
            }
        }
#pragma unroll
        for (int j = 0; j < kCoopBatch; ++j) {
            const int it = it0 + NT * j + t;
            if (it < total) dst[(size_t)(it >> 5) * pitch + W + (it & 31)] = (uint8_t)v[j];
        }
    }
}

template <int NT>
__device__ __forceinline__ void gc_rows_nt(uint8_t* dst, int pitch, const uint8_t* plane, int row0, int rows,
                                            int H, int W, int t) {
    const int G = ((((uintptr_t)plane | (uintptr_t)W) & 7) == 0) ? 8
                  : ((((uintptr_t)plane | (uintptr_t)W) & 3) == 0) ? 4 : 0;
    if (G) {
        // 4- or 8-byte aligned rows: cp.async (no register staging), every copy
        // of the band in flight at once, one wait.  A row is W / G chunks, then
        // (W >= 32) the 32-byte pad as the row's first 32 / G chunks.
        const int nr = W / G, n = nr + (W >= 32 ? 32 / G : 0);
        const int total = rows * n;
        const uint32_t d0 = (uint32_t)__cvta_generic_to_shared(dst);
        int r = t / n, x = t - (t / n) * n;
        for (int it = t; it < total; it += NT) {
            int rr = row0 + r;
            while (rr >= H) rr -= H;
            const uint8_t* src = plane + (int64_t)rr * W + (int64_t)(x < nr ? x : x - nr) * G;
            cp_async_ca(d0 + (uint32_t)(r * pitch + x * G), src, G);
            x += NT;
            if (NT <= 32) { while (x >= n) { x -= n; ++r; } } else if (x >= n) { const int q = x / n; r += q; x -= q * n; }
        }
        if (W < 32) gc_pads_nt<NT>(dst, pitch, plane, row0, rows, H, W, t);   // short rows: row[j mod W]
        cp_async_wait_all();
        return;
    }
    if ((W & 3) == 0) {
        // misaligned plane, W % 4 == 0: every row has the same misalignment m,
        // and each staged word k (row bytes 4k..4k+3; pad words: row bytes
        // 4p..4p+3) is two aligned source words funnelled by m bytes.  The
        // second word holds a valid row byte, so it stays inside the allocation.
        const uint32_t m = (uint32_t)((uintptr_t)plane & 3);
        const uint32_t sel = 0x3210u + 0x1111u * m;
        const int nr = W >> 2, n = nr + (W >= 32 ? 8 : 0);
        const int total = rows * n;
        int r = t / n, x = t - (t / n) * n;
        for (int it0 = 0; it0 < total; it0 += NT * kCoopBatch) {
            uint32_t lo[kCoopBatch], hi[kCoopBatch];
            int dr[kCoopBatch], dx[kCoopBatch];
#pragma unroll
            for (int j = 0; j < kCoopBatch; ++j) {
                dr[j] = r;
                dx[j] = x;
                if (it0 + NT * j + t < total) {
                    int rr = row0 + r;
                    while (rr >= H) rr -= H;
                    const uint32_t* a = reinterpret_cast<const uint32_t*>(
                        plane + (int64_t)rr * W + 4 * (int64_t)(x < nr ? x : x - nr) - m);
                    lo[j] = __ldg(a);
                    hi[j] = __ldg(a + 1);
                }
                x += NT;
                if (NT <= 32) { while (x >= n) { x -= n; ++r; } } else if (x >= n) { const int q = x / n; r += q; x -= q * n; }
            }
#pragma unroll
            for (int j = 0; j < kCoopBatch; ++j)
                if (it0 + NT * j + t < total)
                    reinterpret_cast<uint32_t*>(dst + (size_t)dr[j] * pitch)[dx[j]] = __byte_perm(lo[j], hi[j], sel);
        }
        if (W < 32) gc_pads_nt<NT>(dst, pitch, plane, row0, rows, H, W, t);
        return;
    }
    const bool words = (((uintptr_t)plane | (uintptr_t)W) & 3) == 0;
    const int n = words ? W >> 2 : W;               // items per row
    const int total = rows * n;
    int r = t / n, x = t - (t / n) * n;    // item t
    for (int it0 = 0; it0 < total; it0 += NT * kCoopBatch) {
        uint32_t v[kCoopBatch];
        int dr[kCoopBatch], dx[kCoopBatch];
#pragma unroll
        for (int j = 0; j < kCoopBatch; ++j) {
            dr[j] = r;
            dx[j] = x;
            if (it0 + NT * j + t < total) {
                int rr = row0 + r;
                while (rr >= H) rr -= H;
                const uint8_t* src = plane + (int64_t)rr * W;
                v[j] = words ? __ldg(reinterpret_cast<const uint32_t*>(src) + x) : (uint32_t)__ldg(src + x);
            }
            x += NT;
            if (NT <= 32) { while (x >= n) { x -= n; ++r; } } else if (x >= n) { const int q = x / n; r += q; x -= q * n; }
        }
#pragma unroll
        for (int j = 0; j < kCoopBatch; ++j) {
            if (it0 + NT * j + t < total) {
                uint8_t* d = dst + (size_t)dr[j] * pitch;
                if (words) reinterpret_cast<uint32_t*>(d)[dx[j]] = v[j];
                else d[dx[j]] = (uint8_t)v[j];
            }
        }
    }
    gc_pads_nt<NT>(dst, pitch, plane, row0, rows, H, W, t);
}

template <int NT>
__device__ __forceinline__ void gc_windows_nt(uint8_t* dst, int pitch, const uint8_t* plane, int row0, int rows,
                                               int H, int W, int cs, int len, int t) {
    const int n = (len + 3) >> 2;
    const int total = rows * n;
    int r = t / n, x = t - (t / n) * n;
    for (int it0 = 0; it0 < total; it0 += NT * kCoopBatch) {
        uint32_t v[kCoopBatch];
        int dr[kCoopBatch], dx[kCoopBatch];
#pragma unroll
        for (int j = 0; j < kCoopBatch; ++j) {
            dr[j] = r;
            dx[j] = x;
            if (it0 + NT * j + t < total) {
                int rr = row0 + r;
                while (rr >= H) rr -= H;
                const uint8_t* row = plane + (int64_t)rr * W;
                int c = cs + 4 * x;
                while (c >= W) c -= W;
                if (c + 3 < W) {
                    const uintptr_t a = (uintptr_t)(row + c);
                    const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
                    v[j] = __byte_perm(__ldg(w), __ldg(w + 1), 0x3210u + 0x1111u * (uint32_t)(a & 3));
                } else {
                    uint32_t b = 0;
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const int ct = c + t >= W ? c + t - W : c + t;   // c < W, so one wrap at most
                        b |= (uint32_t)__ldg(row + ct) << (8 * t);
                    }
                    v[j] = b;
                }
            }
            x += NT;
            if (NT <= 32) { while (x >= n) { x -= n; ++r; } } else if (x >= n) { const int q = x / n; r += q; x -= q * n; }
        }
#pragma unroll
        for (int j = 0; j < kCoopBatch; ++j)
            if (it0 + NT * j + t < total)
                reinterpret_cast<uint32_t*>(dst + (size_t)dr[j] * pitch)[dx[j]] = v[j];
    }
}

// Consumer-side staging (CS instantiations only; out of line): strip windows
// (cs >= 0) or whole rows, over NT threads.  gc_*_nt are g_coop_* over NT
// threads instead of one warp.
template <int NT>
__device__ __noinline__ void g_coop_stage_consumers(uint8_t* dst, int pitch, const uint8_t* plane, int row0,
                                                    int rows, int H, int W, int cs, int len, int t) {
    if (cs >= 0) gc_windows_nt<NT>(dst, pitch, plane, row0, rows, H, W, cs, len, t);
    else gc_rows_nt<NT>(dst, pitch, plane, row0, rows, H, W, t);
}


struct GenCursor {
    int64_t u, f;
    int32_t local, gdiv, gmod, upf;
    __device__ __forceinline__ void init(const GeneralParams& p) {
        u = blockIdx.x;
        upf = p.upf;
        f = (int64_t)(blockIdx.x / (uint32_t)upf);
        local = (int32_t)(blockIdx.x - (uint32_t)f * (uint32_t)upf);
        gdiv = (int32_t)(gridDim.x / (uint32_t)upf);
        gmod = (int32_t)(gridDim.x - (uint32_t)gdiv * (uint32_t)upf);
    }
    __device__ __forceinline__ void next() {
        u += gridDim.x;
        f += gdiv;
        local += gmod;
        if (local >= upf) { local -= upf; ++f; }
    }
    __device__ __forceinline__ int plane(const GeneralParams& p) const {
        return (p.n_planes > 2 && local >= p.pl[2].unit_start)   ? 2
               : (p.n_planes > 1 && local >= p.pl[1].unit_start) ? 1
                                                                 : 0;
    }
};

// 2 CTAs x (8 consumer + 1 producer) warps per SM: the register file is
// split across 4 SMSPs, so 18 warps need <= 102 registers each.

// CS: some plane's rows are staged by the consumers (misaligned words, strip
// windows of planes the TMA cannot copy: 8x the producer warp's loads in
// flight); a separate instantiation, so the CS = false kernel is unchanged.
template <int FAST, bool CS>
__global__ void __launch_bounds__((DS_GEN_NCW + 1) * 32, DS_GEN_MINB)
    ds_fused_general_kernel(const __grid_constant__ GeneralParams p) {
    constexpr int NCW = DS_GEN_NCW;
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int NC = NCW * 32;
    const int S = p.stages;
    uint8_t* ring = smem;
    uint8_t* mid = smem + (size_t)S * p.stage_stride;
    uint8_t* outs = mid + p.mid_stride + p.mid_alt;
    uint64_t* full = reinterpret_cast<uint64_t*>(outs + (size_t)2 * p.out_stride);
    uint64_t* empty = full + S;
    uint64_t* outb = empty + S;                     // the band's V writes are complete (NCW arrivals)
    __shared__ int32_t wh[DS_MAX_OUTPUTS][DS_MAX_PATTERN], wv[DS_MAX_OUTPUTS][DS_MAX_PATTERN];

    const int tid = threadIdx.x;
    for (int i = tid; i < DS_MAX_OUTPUTS * DS_MAX_PATTERN; i += blockDim.x) {
        wh[i / DS_MAX_PATTERN][i % DS_MAX_PATTERN] = p.h.w[i / DS_MAX_PATTERN][i % DS_MAX_PATTERN];
        wv[i / DS_MAX_PATTERN][i % DS_MAX_PATTERN] = p.v.w[i / DS_MAX_PATTERN][i % DS_MAX_PATTERN];
    }
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        mbar_init(outb, NCW);
        fence_barrier_init();
    }
    __syncthreads();

    const int warp = tid >> 5, lane = tid & 31;
    GenCursor cur;
    cur.init(p);
    int s = 0;
    uint32_t phase = 0;
    if (warp == NCW) {
        // ---------------- producer warp: band + halo rows into the ring, one
        // staged row (pitch P.pitch) per input row (o_v + S_v k band + i) mod H.
        // Bulk-copy planes: lane 0 posts the byte count, then every lane issues
        // the TMA copies of its rows (row, then its first 32 bytes as the pad).
        // Other planes: all 32 lanes copy with plain loads and lane 0 arrives
        // on full[s] without a transaction count.
        const uint64_t pol = policy_evict_first();
        bool first_round = true;
        for (; cur.u < p.n_units; cur.next()) {
            const GenPlane& P = p.pl[cur.plane(p)];
            const GenView V = g_view(P, p.h.S, p.h.Q, p.v.Q, cur.local - P.unit_start);
            const int b0 = V.run * P.L, b1 = min(b0 + P.L, P.nb);
            const uint8_t* plane = p.in + cur.f * p.in_frame + P.in_off;
            // strips: the window [cs, cs + lw) mod W, staged from x0 = cs & ~15
            int cs = 0, lw = 0, x0 = 0, seg0 = 0, seg1 = 0;
            if (P.strips > 1) {
                cs = (int)(((int64_t)P.oh + (int64_t)p.h.S * V.strip * P.sw) % P.W);
                lw = p.h.S * (V.np - 1) + p.h.P;
                x0 = cs & ~15;
                const int x1 = (cs + lw + 15) & ~15;
                seg0 = min(x1, P.W) - x0;
                seg1 = x1 > P.W ? x1 - P.W : 0;
            }
            for (int band = b0; band < b1; ++band) {
                if (!first_round) mbar_wait_sleep(&empty[s], phase ^ 1);
                uint8_t* dst = ring + (size_t)s * p.stage_stride;
                // first band of a run: all R rows; later bands: the Sv k rows
                // past the ovl rows whose mid the previous band produced
                const int reuse = band > b0 ? p.ovl : 0;
                const int rows = P.R - reuse;
                const int row0 = (int)(((int64_t)P.ov + (int64_t)p.v.S * P.k * band + reuse) % P.H);
                if (P.strips > 1) {
                    if (!P.coop) {
                        if (lane == 0) mbar_arrive_expect_tx(&full[s], (uint32_t)rows * (uint32_t)(seg0 + seg1));
                        __syncwarp();
                        for (int i = lane; i < rows; i += 32) {
                            const uint8_t* src = plane + (int64_t)((row0 + i) % P.H) * P.W;
                            uint8_t* d = dst + (size_t)i * P.pitch;
                            bulk_g2s(d, src + x0, (uint32_t)seg0, &full[s], pol);
                            if (seg1) bulk_g2s(d + seg0, src, (uint32_t)seg1, &full[s], pol);
                        }
                    } else {
                        if (!CS) g_coop_windows(dst, P.pitch, plane, row0, rows, P.H, P.W, cs, lw, lane);
                        __syncwarp();                   // CS: the consumers stage it
                        if (lane == 0) mbar_arrive(&full[s]);
                    }
                } else if (!P.coop) {
                    if (lane == 0) mbar_arrive_expect_tx(&full[s], (uint32_t)rows * (uint32_t)(P.W + 32));
                    __syncwarp();
                    for (int i = lane; i < rows; i += 32) {
                        const uint8_t* src = plane + (int64_t)((row0 + i) % P.H) * P.W;
                        uint8_t* d = dst + (size_t)i * P.pitch;
                        bulk_g2s(d, src, (uint32_t)P.W, &full[s], pol);
                        bulk_g2s(d + P.W, src, 32u, &full[s], pol);
                    }
                } else {
                    // CS: rows cp.async cannot take are staged by the consumers
                    if (!CS || g_coop_async(plane, P.W)) g_coop_rows(dst, P.pitch, plane, row0, rows, P.H, P.W, lane);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&full[s]);      // release: generic smem writes
                }
                if (++s == S) { s = 0; phase ^= 1; first_round = false; }
            }
        }
        return;
    }

    int oslot = 0;
    uint32_t mpar = 0;                              // which mid buffer the next band writes
    uint32_t opar = 0;                              // outb phase
    for (; cur.u < p.n_units; cur.next()) {
        const GenPlane& P = p.pl[cur.plane(p)];
        const GenView V = g_view(P, p.h.S, p.h.Q, p.v.Q, cur.local - P.unit_start);
        const int b0 = V.run * P.L, b1 = min(b0 + P.L, P.nb);
        if (p.unit_count != nullptr && tid == 0) atomicAdd(p.unit_count + cur.u, 1u);
        for (int band = b0; band < b1; ++band) {
            const uint32_t st = smem_u32(ring) + s * p.stage_stride;
            uint8_t* ob = outs + (size_t)oslot * p.out_stride;
            const uint32_t ob_s = smem_u32(ob);
            const uint32_t mid_s = smem_u32(mid) + mpar * p.mid_alt;
            const int reuse = band > b0 ? p.ovl : 0;
            if (reuse) {
                // the previous band's mid rows [Sv k, R) are this band's rows
                // [0, ovl) (its buffer is not written again before two more barriers)
                const uint32_t src = smem_u32(mid) + (mpar ^ 1) * p.mid_alt + p.v.S * P.k * V.wm;
                const int nbytes = reuse * V.wm;
                if ((V.wm & 3) == 0)
                    for (int x = 4 * tid; x < nbytes; x += 4 * NC) sts32s(mid_s + x, lds32s(src + x));
                else
                    for (int x = tid; x < nbytes; x += NC) sts8s(mid_s + x, lds8s(src + x));
            }
            const int rows = P.R - reuse;
            const uint32_t mid_h = mid_s + reuse * V.wm;
            mbar_wait(&full[s], phase);
            if (CS && P.coop) {
                const uint8_t* plane = p.in + cur.f * p.in_frame + P.in_off;
                if (P.strips > 1 || !g_coop_async(plane, P.W)) {
                    const int row0 = (int)(((int64_t)P.ov + (int64_t)p.v.S * P.k * band + reuse) % P.H);
                    const int cs = P.strips > 1 ? (int)(((int64_t)P.oh + (int64_t)p.h.S * V.strip * P.sw) % P.W) : -1;
                    g_coop_stage_consumers<NC>(ring + (size_t)s * p.stage_stride, P.pitch, plane, row0, rows, P.H,
                                               P.W, cs, p.h.S * (V.np - 1) + p.h.P, tid);
                    named_bar_sync(1, NC);
                }
            }

            // ---- H task on every newly staged row -> mid (u8)
            if (p.h.s8) {
                switch (p.h.Q) {
                    case 1: g_h_pass<1, FAST, NC>(p.h, P, V, st, mid_h, rows, tid); break;
                    case 2: g_h_pass<2, FAST, NC>(p.h, P, V, st, mid_h, rows, tid); break;
                    case 3: g_h_pass<3, FAST, NC>(p.h, P, V, st, mid_h, rows, tid); break;
                    case 4: g_h_pass<4, FAST, NC>(p.h, P, V, st, mid_h, rows, tid); break;
                    case 5: g_h_pass<5, FAST, NC>(p.h, P, V, st, mid_h, rows, tid); break;
                    case 6: g_h_pass<6, FAST, NC>(p.h, P, V, st, mid_h, rows, tid); break;
                    case 7: g_h_pass<7, FAST, NC>(p.h, P, V, st, mid_h, rows, tid); break;
                    default: g_h_pass<8, FAST, NC>(p.h, P, V, st, mid_h, rows, tid); break;
                }
            } else {
                g_h_pass_bytes<FAST, NC>(p.h, wh, P, V, st, mid_h, rows, tid);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);     // ring slot no longer read
            named_bar_sync(1, NC);                      // mid complete

            // ---- V task from mid -> output band
            if (p.v.s8 && (V.wm & 3) == 0) {
                switch (p.v.Q) {
                    case 1: g_v_pass<1, 0, FAST, NC>(p.v, P, V, mid_s, ob_s, tid); break;
                    case 2: g_v_pass<2, 0, FAST, NC>(p.v, P, V, mid_s, ob_s, tid); break;
                    case 3: g_v_pass<3, 0, FAST, NC>(p.v, P, V, mid_s, ob_s, tid); break;
                    case 4: g_v_pass<4, 0, FAST, NC>(p.v, P, V, mid_s, ob_s, tid); break;
                    case 5: g_v_pass<4, 1, FAST, NC>(p.v, P, V, mid_s, ob_s, tid); break;
                    case 6: g_v_pass<4, 2, FAST, NC>(p.v, P, V, mid_s, ob_s, tid); break;
                    case 7: g_v_pass<4, 3, FAST, NC>(p.v, P, V, mid_s, ob_s, tid); break;
                    default: g_v_pass<4, 4, FAST, NC>(p.v, P, V, mid_s, ob_s, tid); break;
                }
            } else {
                g_v_pass_bytes<FAST, NC>(p.v, wv, P, V, mid_s, ob_s, tid);
            }
            if (P.strips == 1) {
                uint8_t* dst = p.out + cur.f * p.out_frame + P.out_off + (int64_t)band * P.unit_out;
                if (P.bulk_store && p.mid_alt) {
                    // Only the storing thread waits for the band's V writes; the other
                    // warps go on to the next band's H pass.  That writes the other mid
                    // buffer (two mid buffers: mid_alt), and this band's mid and out slot
                    // are rewritten only after the next band's mid barrier, which thread 0
                    // reaches after bulk_wait_read (the other out slot is free).
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(outb);
                    if (tid == 0) {
                        mbar_wait(outb, opar);
                        bulk_s2g(dst, ob, (uint32_t)P.unit_out);
                        bulk_commit();
                        bulk_wait_read<1>();
                    }
                    opar ^= 1;
                } else if (P.bulk_store) {
                    fence_proxy_async_smem();
                    named_bar_sync(1, NC);              // output band complete; mid free
                    if (tid == 0) {
                        bulk_s2g(dst, ob, (uint32_t)P.unit_out);
                        bulk_commit();
                        bulk_wait_read<1>();            // the other out slot is free
                    }
                } else {
                    named_bar_sync(1, NC);
                    for (int x = tid; x < P.unit_out; x += NC) dst[x] = ob[x];
                }
            } else {
                // strip: Qv k output rows of V.wm bytes at column col0 of the plane
                const int orows = p.v.Q * P.k;
                uint8_t* dst = p.out + cur.f * p.out_frame + P.out_off + (int64_t)band * orows * P.Wm + V.col0;
                if (P.bulk_rows && (V.wm & 15) == 0 && p.mid_alt) {
                    fence_proxy_async_smem();           // as above: only the storing thread waits
                    __syncwarp();
                    if (lane == 0) mbar_arrive(outb);
                    if (tid == 0) {
                        mbar_wait(outb, opar);
                        for (int r = 0; r < orows; ++r)
                            bulk_s2g(dst + (int64_t)r * P.Wm, ob + (size_t)r * V.wm, (uint32_t)V.wm);
                        bulk_commit();
                        bulk_wait_read<1>();
                    }
                    opar ^= 1;
                } else if (P.bulk_rows && (V.wm & 15) == 0) {
                    fence_proxy_async_smem();
                    named_bar_sync(1, NC);
                    if (tid == 0) {
                        for (int r = 0; r < orows; ++r)
                            bulk_s2g(dst + (int64_t)r * P.Wm, ob + (size_t)r * V.wm, (uint32_t)V.wm);
                        bulk_commit();
                        bulk_wait_read<1>();
                    }
                } else {
                    named_bar_sync(1, NC);
                    for (int x = tid; x < V.unit_out; x += NC) {
                        const int r = g_div_small(x, V.wm, V.wm_rcp);
                        dst[(int64_t)r * P.Wm + (x - r * V.wm)] = ob[x];
                    }
                }
            }
            if (++s == S) { s = 0; phase ^= 1; }
            oslot ^= 1;
            mpar ^= (p.mid_alt != 0);
        }
    }
    if (tid == 0) bulk_wait_all();
}

}  // namespace ds
