// ds_kernels.cuh -- sm_100a kernels of the arxiv 1103.4881 downscaler.
//
// Citation key: P:n = PAPER.md line n, S:n = SPEC.md line n, SURVEY sec. n.
//
//   K-N1 ds_fused_band_kernel   persistent, warp-specialised: one producer
//        lane streams whole-width row bands (the input patterns of a group
//        of vertical repetitions, minus the dead row) HBM -> shared memory
//        with 1-D TMA bulk copies (cp.async.bulk + mbarrier ring); consumer
//        warps run the horizontal task (taps S:530) and the vertical
//        task (taps S:540) on-chip with the u8 intermediate in
//        registers, stage the output band in shared memory and
//        write it back with one TMA bulk store.  Planes whose rows are not
//        16-byte multiples ("narrow") or short ("whole-band") stage the whole
//        band, dead rows included, in one copy; each plan shape gets its own
//        instantiation (MODES) so unused consumer loops are not compiled in.
//        No tensor cores: this is a memory-bound stencil.
//   K-N2 ds_generic_kernel      one thread per output pixel, any stage spec
//        (halos P > S, origin != 0, any taps), any alignment; follows the
//        tiler definition e = (o + S r + f) mod n directly.
//   K-N4 ds_generate_kernel     counter-hash synthetic frames (test/bench).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ds.h"
#include "ds_pipeline.cuh"

namespace ds {

// ------------------------------------------------------------- parameters --
struct FusedPlane {
    int64_t in_off, out_off;   // plane offsets inside one frame (bytes)
    int32_t W, Wout;           // input / output row bytes
    int32_t k;                 // 9-row groups per unit (band)
    int32_t chunks;            // 16-byte column chunks per row = W / 16
    int32_t tasks;             // 2 * k * chunks  (one task = 16 B x 4 slot rows)
    int32_t unit_start;        // first per-frame unit index of this plane
    int32_t unit_in;           // bytes staged per unit = 8 * k * W
    int32_t unit_out;          // bytes produced per unit = 4 * k * Wout
    int32_t bulk_store;        // 1: TMA bulk store legal (16 B aligned)
    uint32_t chunks_rcp;       // ceil(2^32 / chunks) (chunks > 1): t / chunks = umulhi(t, rcp)
    int32_t narrow;            // 1: W % 16 == 8 -- the whole band (dead rows included) is
                               // bulk-copied from a 16-aligned superset; rows are 8-aligned
                               // in smem, the last chunk of a row holds one packet
    int32_t whole;             // 1: W % 16 == 0 but short rows -- the whole band (dead rows
                               // included) is one bulk copy: 9x fewer, larger TMA ops
};

struct FusedParams {
    const uint8_t* in;
    uint8_t* out;
    uint32_t* unit_count;      // debug (ds_set_debug_counter): +1 per unit processed, else null
    int64_t in_frame, out_frame;
    int64_t n_units;           // n_frames * units_per_frame
    int32_t upf;               // units per frame
    int32_t n_planes;
    int32_t stages;            // ring depth
    int32_t stage_stride;      // bytes per ring slot (>= max unit_in, 128-aligned)
    int32_t out_stride;        // bytes per output slot (>= max unit_out, 128-aligned)
    int32_t reserved_;         // keeps pl[] 8-byte aligned
    FusedPlane pl[DS_MAX_PLANES];
};

struct GenericParams {
    const uint8_t* in;
    uint8_t* out;
    int64_t in_frame, out_frame, total_out;
    int64_t in_off[DS_MAX_PLANES], out_off[DS_MAX_PLANES];
    int32_t W[DS_MAX_PLANES], H[DS_MAX_PLANES], Wout[DS_MAX_PLANES];
    int32_t n_planes;
    ds_stage_spec h, v;
};

constexpr int kOutSlots = 3;   // output staging ring (one barrier per unit)

// ------------------------------------------------------- filter arithmetic --
// floor(x / 6) for 0 <= x < 2^31: umulhi(x, ceil(2^32 / 6)).
__device__ __forceinline__ uint32_t div6(uint32_t x) { return __umulhi(x, 0x2AAAAAABu); }

// Horizontal task on one 16-byte row chunk = two 8-pixel packets
// (S:527-531): out0 = (p0 + 5 p1 + 3)/6, out1 = (3 p3 + 3 p4 + 3)/6 =
// (p3 + p4 + 1) >> 1, out2 = (5 p6 + p7 + 3)/6; p2 and p5 have zero weight.
// The six u8 mid values are returned packed in 16-bit lanes:
//   q0 = A0 | A1 << 16,  q1 = A2 | B0 << 16,  q2 = B1 | B2 << 16.
__device__ __forceinline__ void h_chunk(uint4 v, uint32_t& q0, uint32_t& q1, uint32_t& q2) {
    const uint32_t tA = __byte_perm(v.x, v.y, 0x7643);   // [p3 p4 p6 p7] of packet A
    const uint32_t tB = __byte_perm(v.z, v.w, 0x7643);
    const uint32_t a0 = div6(__dp4a(v.x, 0x0501u, 3u));
    const uint32_t a1 = __dp4a(tA, 0x0101u, 1u) >> 1;
    const uint32_t a2 = div6(__dp4a(tA, 0x01050000u, 3u));
    const uint32_t b0 = div6(__dp4a(v.z, 0x0501u, 3u));
    const uint32_t b1 = __dp4a(tB, 0x0101u, 1u) >> 1;
    const uint32_t b2 = div6(__dp4a(tB, 0x01050000u, 3u));
    q0 = __byte_perm(a0, a1, 0x5410);
    q1 = __byte_perm(a2, b0, 0x5410);
    q2 = __byte_perm(b1, b2, 0x5410);
}

// Vertical task output row: (wa*m_a + wb*m_b + 4) >> 3 on two
// 16-bit lanes at once.  Scaling by 32 puts the quotient in byte 1 of each
// lane: 32*(wa*m_a + wb*m_b + 4) <= 32*2044 < 2^16, so lanes never carry.
template <uint32_t WA, uint32_t WB>
__device__ __forceinline__ uint32_t v_pair(uint32_t qa, uint32_t qb) {
    return qa * (32u * WA) + qb * (32u * WB) + 0x00800080u;
}

// One consumer task: 4 slot rows x 16 bytes -> H task -> two V output rows of
// 6 bytes (lo = bytes 0..3, hi = bytes 4..5).  V taps: half 0 ->
// out0 rows (0,1) w (3,5), out1 rows (2,3) w (1,7); half 1 -> out2 rows
// (5,6) w (7,1), out3 rows (7,8) w (5,3).
__device__ __forceinline__ void k1_task(const uint4 (&r)[4], int half, uint32_t (&lo)[2],
                                        uint32_t (&hi)[2]) {
    uint32_t q[4][3];
#pragma unroll
    for (int j = 0; j < 4; ++j) h_chunk(r[j], q[j][0], q[j][1], q[j][2]);
    const uint32_t wa0 = half ? 32u * 7 : 32u * 3, wb0 = half ? 32u * 1 : 32u * 5;
    const uint32_t wa1 = half ? 32u * 5 : 32u * 1, wb1 = half ? 32u * 3 : 32u * 7;
    uint32_t o[2][3];
#pragma unroll
    for (int e = 0; e < 3; ++e) {
        o[0][e] = q[0][e] * wa0 + q[1][e] * wb0 + 0x00800080u;
        o[1][e] = q[2][e] * wa1 + q[3][e] * wb1 + 0x00800080u;
    }
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
        lo[kk] = __byte_perm(o[kk][0], o[kk][1], 0x7531);
        hi[kk] = __byte_perm(o[kk][2], 0u, 0x4431);
    }
}

// Store a task's two 6-byte output pieces (rows orow and orow + Wout, bytes
// 6c .. 6c+5; the output slot is 16-byte aligned).  Even chunks
// start on a word (word, then half-word), odd chunks on a half-word (half-word,
// then word): one 4-byte and one 2-byte store per row with per-lane addresses
// and data instead of three 2-byte stores.  Measured 0.5-1% slower than the
// three 2-byte stores on HD/4K (same-call A/B, profiles/r02/k1_store6_ab.txt),
// so DS_K1_STORE6 defaults to 0.
#ifndef DS_K1_STORE6
#define DS_K1_STORE6 0
#endif
__device__ __forceinline__ void k1_store6(uint8_t* orow, int Wout, int c, const uint32_t (&lo)[2],
                                          const uint32_t (&hi)[2]) {
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
        uint8_t* d = orow + (size_t)kk * Wout;
#if DS_K1_STORE6
        if ((Wout & 3) != 0) {                       // rows not word-aligned (e.g. 66-byte CIF chroma)
            sts16(d, lo[kk]);
            sts16(d + 2, lo[kk] >> 16);
            sts16(d + 4, hi[kk]);
            continue;
        }
        const bool odd = c & 1;
        const uint32_t w = odd ? __byte_perm(lo[kk], hi[kk], 0x5432) : lo[kk];   // bytes 2..5 : 0..3
        const uint32_t h = odd ? lo[kk] : hi[kk];                                 // bytes 0..1 : 4..5
        uint8_t* dw = d + (odd ? 2 : 0);
        uint8_t* dh = d + (odd ? 0 : 4);
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(smem_u32(dw)), "r"(w) : "memory");
        sts16(dh, h);
#else
        sts16(d, lo[kk]);
        sts16(d + 2, lo[kk] >> 16);
        sts16(d + 4, hi[kk]);
#endif
    }
}

// ------------------------------------------------------------------- K-N1 --
// Work unit = (frame, plane, band of k 9-row groups), full plane width.
// Ring slot layout: for group g, rows 8g..8g+3 hold input rows 9g+0..3 and
// rows 8g+4..8g+7 hold input rows 9g+5..8 (row 9g+4 has zero V weight,
// S:540, and is never read from HBM).
//
// Consumer task = (half-group hg, 16-byte column chunk c): the 4 slot rows
// 8(hg>>1) + 4(hg&1) .. +3, i.e. the two V outputs 4g+2(hg&1) and +1 of the
// six columns 6c..6c+5.  Consecutive lanes take consecutive chunks (conflict
// -free LDS.128).  No runtime integer division anywhere in the unit loop:
// unit -> (frame, plane, band) and ring/phase counters advance
// incrementally, task -> (hg, c) uses a precomputed reciprocal.

// Per-CTA walk over its units u = blockIdx.x + i * gridDim.x.
struct UnitCursor {
    int64_t u, f;
    int32_t local;
    int32_t gdiv, gmod, upf;
    __device__ __forceinline__ void init(const FusedParams& p) {
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
    __device__ __forceinline__ int plane(const FusedParams& p) const {
        return (p.n_planes > 2 && local >= p.pl[2].unit_start)   ? 2
               : (p.n_planes > 1 && local >= p.pl[1].unit_start) ? 1
                                                                 : 0;
    }
};

// ---- K-N1 consumer loops over one unit's tasks (task t = half-group
// t / chunks, 16-byte chunk t % chunks).
// Wide planes: the slot holds the 8 live rows of each group; half-group hg
// reads slot rows 4 hg .. 4 hg + 3.
template <int NC>
__device__ __forceinline__ void k1_loop_wide(const uint8_t* st, uint8_t* ob, int W, int Wout, int chunks,
                                             int tasks, uint32_t rcp, int tid) {
    for (int t = tid; t < tasks; t += NC) {
        const int hg = chunks == 1 ? t : (int)__umulhi((uint32_t)t, rcp);   // t / chunks
        const int c = t - hg * chunks;
        const uint8_t* base = st + (size_t)4 * hg * W + 16 * c;
        uint4 r[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) r[j] = lds128(base + (size_t)j * W);
        uint32_t lo[2], hi[2];
        k1_task(r, hg & 1, lo, hi);
        uint8_t* orow = ob + (size_t)2 * hg * Wout + 6 * c;
        k1_store6(orow, Wout, c, lo, hi);
    }
}
// Whole band staged (short aligned rows): half-group hg reads slot rows
// 9 (hg / 2) + 5 (hg % 2) + 0..3.
template <int NC>
__device__ __forceinline__ void k1_loop_whole(const uint8_t* st, uint8_t* ob, int W, int Wout, int chunks,
                                              int tasks, uint32_t rcp, int tid) {
    for (int t = tid; t < tasks; t += NC) {
        const int hg = chunks == 1 ? t : (int)__umulhi((uint32_t)t, rcp);   // t / chunks
        const int c = t - hg * chunks;
        const int half = hg & 1;
        const uint8_t* base = st + (size_t)(9 * (hg >> 1) + 5 * half) * W + 16 * c;
        uint4 r[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) r[j] = lds128(base + (size_t)j * W);
        uint32_t lo[2], hi[2];
        k1_task(r, half, lo, hi);
        uint8_t* orow = ob + (size_t)2 * hg * Wout + 6 * c;
        k1_store6(orow, Wout, c, lo, hi);
    }
}
// Narrow plane (W % 16 == 8): st points at the band's first byte inside the
// slot (phase applied); rows are 8-byte aligned; the last chunk of a row holds
// one packet; output rows are odd -> byte stores.
template <int NC>
__device__ __forceinline__ void k1_loop_narrow(const uint8_t* st, uint8_t* ob, int W, int Wout, int chunks,
                                               int tasks, uint32_t rcp, int tid) {
    for (int t = tid; t < tasks; t += NC) {
        const int hg = chunks == 1 ? t : (int)__umulhi((uint32_t)t, rcp);   // t / chunks
        const int c = t - hg * chunks;
        const int half = hg & 1;
        const uint8_t* base = st + (size_t)(9 * (hg >> 1) + 5 * half) * W + 16 * c;
        uint4 r[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint2 a = lds64(base + (size_t)j * W), b = lds64(base + (size_t)j * W + 8);
            r[j] = make_uint4(a.x, a.y, b.x, b.y);
        }
        uint32_t lo[2], hi[2];
        k1_task(r, half, lo, hi);
        uint8_t* orow = ob + (size_t)2 * hg * Wout + 6 * c;
        const bool two = c + 1 < chunks;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
            uint8_t* d = orow + (size_t)kk * Wout;
            sts8(d, lo[kk]);
            sts8(d + 1, lo[kk] >> 8);
            sts8(d + 2, lo[kk] >> 16);
            if (two) {
                sts8(d + 3, lo[kk] >> 24);
                sts8(d + 4, hi[kk]);
                sts8(d + 5, hi[kk] >> 8);
            }
        }
    }
}
// MODES: bit 0 wide planes (8 live rows per group staged), bit 1 whole-band
// planes (short aligned rows), bit 2 narrow planes (W % 16 == 8).  Each
// instantiation compiles only the consumer loops its plan needs: a loop that
// is present but unused measurably slows the others (a per-unit branch in
// front of the HD loop cost 7.7%; out-of-line loops cost SD 14%).
template <int NCW, int MODES>
__global__ void __launch_bounds__((NCW + 1) * 32)
    ds_fused_band_kernel(const __grid_constant__ FusedParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int NC = NCW * 32;
    const int S = p.stages;
    uint8_t* ring = smem;
    uint8_t* outs = smem + (size_t)S * p.stage_stride;
    uint64_t* full = reinterpret_cast<uint64_t*>(outs + (size_t)kOutSlots * p.out_stride);
    uint64_t* empty = full + S;

    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        fence_barrier_init();
    }
    __syncthreads();

    const int warp = tid >> 5, lane = tid & 31;
    UnitCursor cur;
    cur.init(p);
    int s = 0;
    uint32_t phase = 0;
    if (warp == NCW) {
        // ---------------- producer: one lane streams bands into the ring --
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            bool first_round = true;
            for (; cur.u < p.n_units; cur.next()) {
                if (!first_round) mbar_wait(&empty[s], phase ^ 1);
                const FusedPlane& P = p.pl[cur.plane(p)];
                const int band = cur.local - P.unit_start;
                const uint8_t* src =
                    p.in + cur.f * p.in_frame + P.in_off + (int64_t)band * 9 * P.k * P.W;
                uint8_t* dst = ring + (size_t)s * p.stage_stride;
                if ((MODES & 4) && P.narrow) {
                    // one copy of the whole band from its 16-aligned superset: the
                    // start is at most 8 bytes into the previous band (never before
                    // the buffer: frames are 16-aligned), the end at most 15 bytes
                    // past the band (never past the buffer, whose end is aligned)
                    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
                    const uintptr_t a0 = a & ~uintptr_t(15);
                    const uintptr_t a1 = (a + (uintptr_t)9 * P.k * P.W + 15) & ~uintptr_t(15);
                    mbar_arrive_expect_tx(&full[s], (uint32_t)(a1 - a0));
                    bulk_g2s(dst, reinterpret_cast<const uint8_t*>(a0), (uint32_t)(a1 - a0), &full[s], pol);
                } else if ((MODES & 2) && P.whole) {
                    mbar_arrive_expect_tx(&full[s], (uint32_t)P.unit_in);
                    bulk_g2s(dst, src, (uint32_t)P.unit_in, &full[s], pol);      // rows 0..9k-1
                } else {
                mbar_arrive_expect_tx(&full[s], (uint32_t)P.unit_in);
                // live rows of the band: 0..3 | 5..12 | 14..21 | ... | 9k-4..9k-1.
                // Rows 5..8 of group g and 0..3 of group g+1 are contiguous both in
                // HBM and in the slot, so a band of k groups takes k + 1 copies
                // (measured +1.5% on HD 4:2:0 over two copies per group).
                const uint32_t half = 4u * (uint32_t)P.W;
                bulk_g2s(dst, src, half, &full[s], pol);                                  // g0 rows 0..3
                for (int g = 0; g + 1 < P.k; ++g)
                    bulk_g2s(dst + (size_t)(8 * g + 4) * P.W, src + (int64_t)(9 * g + 5) * P.W,
                             2u * half, &full[s], pol);                                   // rows 5..8 | 0..3
                bulk_g2s(dst + (size_t)(8 * P.k - 4) * P.W, src + (int64_t)(9 * P.k - 4) * P.W, half,
                         &full[s], pol);                                                  // last rows 5..8
                }
                if (++s == S) { s = 0; phase ^= 1; first_round = false; }
            }
        }
        return;
    }

    // ---------------- consumers ---------------------------------------------
    int oslot = 0;
    for (; cur.u < p.n_units; cur.next()) {
        const FusedPlane& P = p.pl[cur.plane(p)];
        const int band = cur.local - P.unit_start;
        const uint8_t* st = ring + (size_t)s * p.stage_stride;
        uint8_t* ob = outs + (size_t)oslot * p.out_stride;
        const int W = P.W, Wout = P.Wout, chunks = P.chunks, tasks = P.tasks;
        const uint32_t rcp = P.chunks_rcp;

        mbar_wait(&full[s], phase);

        if ((MODES & 2) && P.whole) {
            k1_loop_whole<NC>(st, ob, W, Wout, chunks, tasks, rcp, tid);
        } else if ((MODES & 4) && P.narrow) {
            const int nphase = (int)((p.in_frame * cur.f + P.in_off + (int64_t)band * 9 * P.k * W) & 15);
            k1_loop_narrow<NC>(st + nphase, ob, W, Wout, chunks, tasks, rcp, tid);
        } else if (MODES & 1) {
            k1_loop_wide<NC>(st, ob, W, Wout, chunks, tasks, rcp, tid);
        }
        // every lane of this warp has consumed its reads of slot s
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);

        uint8_t* dst = p.out + cur.f * p.out_frame + P.out_off + (int64_t)band * P.unit_out;
        if (p.unit_count != nullptr && tid == 0) atomicAdd(p.unit_count + cur.u, 1u);
        if (P.bulk_store) {
            fence_proxy_async_smem();      // generic-proxy smem writes -> async proxy
            named_bar_sync(1, NC);
            if (tid == 0) {
#if DS_K1_STORE_HINT
                // evict_first on the stores as on the loads: the output is
                // never re-read by this kernel (same-call A/B: +0.8% hd444,
                // +1% 4k420 under sw_power_cap, hd420 unchanged)
                bulk_s2g_hint(dst, ob, (uint32_t)P.unit_out, policy_evict_first());
#else
                bulk_s2g(dst, ob, (uint32_t)P.unit_out);
#endif
                bulk_commit();
                bulk_wait_read<1>();       // slot (oslot-1)%3 free before next barrier
            }
        } else {
            named_bar_sync(1, NC);
            for (int x = tid; x < P.unit_out; x += NC) dst[x] = ob[x];
        }
        if (++s == S) { s = 0; phase ^= 1; }
        if (++oslot == kOutSlots) oslot = 0;
    }
    if (tid == 0) bulk_wait_all();
}

// ------------------------------------------------------------------- K-N2 --
__device__ __forceinline__ int32_t nn_mod(int32_t a, int32_t m) {
    int32_t r = a % m;
    return r < 0 ? r + m : r;
}
__device__ __forceinline__ int32_t clamp255(int32_t v) { return v < 0 ? 0 : (v > 255 ? 255 : v); }

// Output (R, C) of a plane: V repetition r0 = R / Qv at slot kv = R % Qv,
// H repetition r1 = C / Qh at slot jh = C % Qh.  Its V pattern element i is
// the mid value at row (ov + Sv r0 + i) mod H, column C; each mid value is
// the H stage over columns (oh + Sh r1 + i') mod W of that row (S:248-252,
// S:517-520), rounded to u8 before the V stage.
__global__ void __launch_bounds__(256, 1) ds_generic_kernel(const __grid_constant__ GenericParams p) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < p.total_out;
         idx += stride) {
        const int64_t f = idx / p.out_frame;
        int64_t o = idx - f * p.out_frame;
        const int pi = (p.n_planes > 2 && o >= p.out_off[2])   ? 2
                       : (p.n_planes > 1 && o >= p.out_off[1]) ? 1
                                                               : 0;
        o -= p.out_off[pi];
        const int32_t W = p.W[pi], H = p.H[pi], Wout = p.Wout[pi];
        const int32_t R = (int32_t)(o / Wout), C = (int32_t)(o - (int64_t)R * Wout);
        const int32_t r0 = R / p.v.outputs, kv = R - r0 * p.v.outputs;
        const int32_t r1 = C / p.h.outputs, jh = C - r1 * p.h.outputs;
        const uint8_t* plane = p.in + f * p.in_frame + p.in_off[pi];
        int32_t accv = p.v.bias;
        for (int i = 0; i < p.v.pattern; ++i) {
            const int32_t wv = p.v.weight[kv][i];
            if (wv == 0) continue;
            const int32_t row = nn_mod(p.v.origin + p.v.paving * r0 + i, H);
            const uint8_t* rp = plane + (int64_t)row * W;
            int32_t acch = p.h.bias;
            for (int i2 = 0; i2 < p.h.pattern; ++i2) {
                const int32_t wh = p.h.weight[jh][i2];
                if (wh == 0) continue;
                acch += wh * (int32_t)__ldg(rp + nn_mod(p.h.origin + p.h.paving * r1 + i2, W));
            }
            accv += wv * clamp255(acch / p.h.divisor);
        }
        p.out[f * p.out_frame + p.out_off[pi] + o] = (uint8_t)clamp255(accv / p.v.divisor);
    }
}

// ------------------------------------------------------------------- K-N4 --
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void __launch_bounds__(256)
    ds_generate_kernel(uint8_t* dst, int64_t n, uint64_t base, int64_t start, int aligned) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 16;
    for (int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 16; i0 < n;
         i0 += stride) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t x = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const uint64_t h = splitmix64(base + (uint64_t)(start + i0 + 4 * q + b));
                x |= (uint32_t)(h >> 56) << (8 * b);
            }
            w[q] = x;
        }
        if (aligned && i0 + 16 <= n) {
            *reinterpret_cast<uint4*>(dst + i0) = make_uint4(w[0], w[1], w[2], w[3]);
        } else {
            for (int b = 0; b < 16 && i0 + b < n; ++b) dst[i0 + b] = (uint8_t)(w[b >> 2] >> (8 * (b & 3)));
        }
    }
}

}  // namespace ds
