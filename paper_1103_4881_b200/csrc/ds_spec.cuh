// ds_spec.cuh -- K-N1s: the fused band kernel with the filter spec compiled in
// (any separable Array-OL stage spec at HBM speed).
//
// Same job as K-N1g (ds_general.cuh): per (frame, plane, run of bands) an
// Array-OL horizontal task then a vertical task with the
// u8 intermediate in shared memory, for any stage spec -- halos
// P > S with toroidal wrap, origins, any taps -- but the spec is a
// compile-time type: taps, pattern/paving/outputs, divisor and the byte phase
// of the H windows are constants, so
//   * the H pass runs one dp4a per (output, aligned input word) whose
//     re-indexed weight word is nonzero -- no byte shifting, no zero taps
//     (the halo spec: 2 dp4a per output where the runtime-tap kernel needs 4);
//   * the V pass loads only the intermediate rows some tap reads, transposes
//     only 4-row blocks with >= 3 live rows, pairs 2-row blocks and folds
//     1-row blocks into shifted-weight dp4a;
//   * division is one multiply-high (or a shift), and clamps the spec proves
//     dead are not emitted.
// Data movement: the H pass loads its input straight from HBM into registers
// (coalesced 16-byte loads; a lane takes 4 consecutive H repetitions, and the
// window bytes its neighbour already fetched come from L1), so the input never
// passes through shared memory and there is no copy engine to feed: one copy
// instruction per row was the limit of the TMA-staged design (1-D bulk copies
// cannot stage a row and its wrap-around window at once, and at ~2 copies per
// row their issue rate, not HBM, bounded K-N1g).  The intermediate is the only
// shared-memory array (two buffers; a band's V halo rows are carried over
// from the previous band of the run), and V outputs go from registers to HBM
// as coalesced stores.  No mbarriers, no producer warp: one CTA barrier per
// band.
//
// This header is self-contained device code: it compiles under nvcc (the
// built-in instances, ds_spec.cu) and under NVRTC (any other spec, compiled
// at run time from this same source with a generated stage type).
#pragma once

#ifdef __CUDACC_RTC__
typedef unsigned char uint8_t;
typedef signed char int8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef int int32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
typedef unsigned long long uintptr_t;
#else
#include <cstdint>
#endif

#ifndef DS_SPEC_NW
#define DS_SPEC_NW 8                  // warps per CTA
#endif
#if DS_SPEC_NW == 8
#define DS_SPEC_LGNW 3
#elif DS_SPEC_NW == 16
#define DS_SPEC_LGNW 4
#elif DS_SPEC_NW == 4
#define DS_SPEC_LGNW 2
#else
#error "DS_SPEC_NW must be 4, 8 or 16"
#endif
#ifndef DS_SPEC_WS
#define DS_SPEC_WS 0                  // 1: warp-specialised (DS_SPEC_NW H warps + DS_SPEC_NWV V warps, named barriers)
#endif
#ifndef DS_SPEC_NWV
#define DS_SPEC_NWV 4                 // V warps of the warp-specialised kernel
#endif
#ifndef DS_SPEC_MINB
#if DS_SPEC_WS
#define DS_SPEC_MINB 2
#else
#define DS_SPEC_MINB 3                // CTAs per SM the register budget is sized for (4: 64 regs, constants rematerialised; measured slower)
#endif
#endif
#if DS_SPEC_WS
#define DS_SPEC_THREADS ((DS_SPEC_NW + DS_SPEC_NWV) * 32)
#else
#define DS_SPEC_THREADS (DS_SPEC_NW * 32)
#endif
#ifndef DS_SPEC_DEPTH3
#define DS_SPEC_DEPTH3 0              // 1: three rows of H loads in flight per warp instead of two
#endif
#ifndef DS_SPEC_MAXP
#define DS_SPEC_MAXP 3
#endif

namespace dss {

// ---------------------------------------------------------------- params --
struct SpecPlane {
    int64_t in_off, out_off;   // plane offsets inside one frame
    int32_t W, H, Wout;        // input row bytes, rows, output row bytes
    int32_t oh, ov;            // H origin reduced to (-W/2, W/2]; V origin reduced mod H (>= 0)
    int32_t np;                // H repetitions per row (W / Sh)
    int32_t nch;               // chunks of 4 repetitions per row: ceil(np / 4)
    int32_t segs, lgsegs;      // 32-chunk warp segments per row (a power of two >= nch / 32); log2
    int32_t lgrpw;             // log2 rows per warp (segs == 1): 32 >> lgrpw chunk lanes per row
    int32_t nwc, wch[4];       // chunks whose window crosses the row end (wrap pass)
    int32_t nb16, blk0;        // W / 16 (floor); floor(oh / 16): first window block of repetition 0 (may be < 0)
    int32_t k, nb;             // V repetitions per band, bands per plane ((H / Sv) / k)
    int32_t L;                 // bands per run (a unit); the V halo's mid rows carry over
    int32_t nq;                // intermediate column quads: ceil(Qh np / 4)
    uint32_t nq_rcp;           // ceil(2^32 / nq) (nq > 1)
    int32_t mp;                // intermediate row stride (>= 4 Qh nch)
    int32_t unit_start;        // first unit of the plane within a frame
};

struct SpecParams {
    const uint8_t* in;
    uint8_t* out;
    uint32_t* unit_count;      // debug: +1 per unit processed, else null
    int64_t in_frame, out_frame, n_units;
    int32_t upf, n_planes, mid_stride, ovl;   // ovl = max(Pv - Sv, 0): rows a band shares with the next
    int32_t out_al4;                          // 1: every output row starts 4-byte aligned
    int32_t in_mis;                           // AL = 1 instances: input pointer mod 4 (every row start's)
    SpecPlane pl[DS_SPEC_MAXP];
};

// --------------------------------------------------- compile-time helpers --
template <int V>
struct IC {
    static constexpr int value = V;
};
template <int I, int N, class F>
__device__ __forceinline__ void sfor(F&& f) {
    if constexpr (I < N) {
        f(IC<I>{});
        sfor<I + 1, N>(f);
    }
}

// A stage type ST provides: P, S, Q, D, B (bias), O (origin) as static
// constexpr ints and  static constexpr int w(int j, int i)  (0 outside the
// taps).  Derived constants:
template <class ST>
struct StageInfo {
    // accumulator range over all windows: bias + 255 * (sum of positive / negative taps)
    __host__ __device__ static constexpr int64_t acc_max() {
        int64_t m = -(int64_t(1) << 62);
        for (int j = 0; j < ST::Q; ++j) {
            int64_t s = ST::B;
            for (int i = 0; i < ST::P; ++i) s += ST::w(j, i) > 0 ? 255 * ST::w(j, i) : 0;
            m = s > m ? s : m;
        }
        return m;
    }
    __host__ __device__ static constexpr int64_t acc_min() {
        int64_t m = int64_t(1) << 62;
        for (int j = 0; j < ST::Q; ++j) {
            int64_t s = ST::B;
            for (int i = 0; i < ST::P; ++i) s += ST::w(j, i) < 0 ? 255 * ST::w(j, i) : 0;
            m = s < m ? s : m;
        }
        return m;
    }
    __host__ __device__ static constexpr int hi_tap() {   // last tap index with a nonzero weight (any output)
        int h = 0;
        for (int j = 0; j < ST::Q; ++j)
            for (int i = 0; i < ST::P; ++i)
                if (ST::w(j, i) != 0 && i > h) h = i;
        return h;
    }
    __host__ __device__ static constexpr bool live(int i) {   // some output reads tap i
        for (int j = 0; j < ST::Q; ++j)
            if (ST::w(j, i) != 0) return true;
        return false;
    }
    // Float division (fs = 1 or 2; 0 = not used): floor(a / D) = round((fs a - c) / (fs D))
    // with c = fs (D - 1) / 2 an integer (fs = 2 for even D), since the exact
    // value then sits >= 1 / (2 fs D) away from a rounding tie.  The dot product
    // accumulates fs a - c on top of the bit pattern of 2^23 (0x4B000000 + y is
    // the float 2^23 + y for 0 <= y < 2^23), so one FADD recovers fs a - c as a
    // float and one FFMA with 1 / (fs D) plus the magic 1.5 * 2^23 rounds it to
    // an integer in the low mantissa bits -- byte 0 of the result is the
    // quotient.  Two FMA-pipe ops that either FMA unit can run, instead of an
    // IMAD.HI on the heavy unit the dp4a also need.  Used when: D > 1 is not a
    // power of two, 0 <= fs amin - c, fs amax < 2^20 (error < 1 / (16 D) from
    // 1 / (fs D) in float), amax / D <= 255 (no clamp), fs w fits s8.
    __host__ __device__ static constexpr int fs_for(int s) {
        if (ST::D <= 1 || (ST::D & (ST::D - 1)) == 0) return 0;
        if (acc_min() < 0) return 0;
        const int64_t c = (int64_t)s * (ST::D - 1) / 2;
        if ((int64_t)s * acc_min() < c || (int64_t)s * acc_max() >= (int64_t(1) << 20)) return 0;
        if (acc_max() / ST::D > 255) return 0;
        for (int j = 0; j < ST::Q; ++j)
            for (int i = 0; i < ST::P; ++i)
                if (s * ST::w(j, i) < -128 || s * ST::w(j, i) > 127) return 0;
        return s;
    }
    __host__ __device__ static constexpr int fs() {
#ifdef DS_SPEC_NO_FDIV
        return 0;
#else
        return fs_for(ST::D % 2 ? 1 : 2);
#endif
    }
    // the accumulator's start value and tap weights as the dot products use them
    __host__ __device__ static constexpr int32_t acc0() {
        return fs() ? (int32_t)(0x4B000000 + fs() * ST::B - fs() * (ST::D - 1) / 2) : ST::B;
    }
    __host__ __device__ static constexpr int ws(int j, int i) { return fs() ? fs() * ST::w(j, i) : ST::w(j, i); }
    // s8-packed weights of output j on the aligned word b when the pattern
    // starts at byte `off` of the word grid: byte t <-> tap 4b + t - off
    __host__ __device__ static constexpr uint32_t wword(int j, int b, int off) {
        uint32_t r = 0;
        for (int t = 0; t < 4; ++t) {
            const int i = 4 * b + t - off;
            if (i >= 0 && i < ST::P) r |= (uint32_t)(uint8_t)(int8_t)ws(j, i) << (8 * t);
        }
        return r;
    }
    // M = ceil(2^32 / D): floor(a / D) = umulhi(a, M) for 0 <= a <= acc_max iff acc_max * e < 2^32
    __host__ __device__ static constexpr uint64_t M() { return ((uint64_t(1) << 32) + ST::D - 1) / ST::D; }
    __host__ __device__ static constexpr bool fastdiv() {
        return ST::D > 1 && acc_max() < 0x7fffffff &&
               (uint64_t)acc_max() * (M() * ST::D - (uint64_t(1) << 32)) < (uint64_t(1) << 32);
    }
};

__host__ __device__ constexpr int log2i(int d) { return d <= 1 ? 0 : 1 + log2i(d >> 1); }

// clamp_0^255(trunc(acc / D)) (round-half-up bias, truncating
// division, clamp) with everything the spec proves dead removed
template <class ST>
__device__ __forceinline__ uint32_t qdiv(int32_t acc) {
    using I = StageInfo<ST>;
    constexpr int64_t amax = I::acc_max(), amin = I::acc_min();
    // a non-positive accumulator truncates to a non-positive quotient -> 0
    const uint32_t a = amin >= 0 ? (uint32_t)acc : (uint32_t)max(acc, 0);
    uint32_t q;
    if constexpr (ST::D == 1) {
        q = a;
    } else if constexpr ((ST::D & (ST::D - 1)) == 0) {
        q = a >> log2i(ST::D);
    } else if constexpr (I::fastdiv()) {
        q = __umulhi(a, (uint32_t)I::M());
    } else {
        q = a / (uint32_t)ST::D;
    }
    if constexpr (amax / ST::D > 255) q = min(q, 255u);
    return q;
}
// the output byte of an accumulator started at StageInfo<ST>::acc0(): byte 0
// of the result is clamp_0^255(trunc(acc / D)) (higher bytes are not defined)
template <class ST>
__device__ __forceinline__ uint32_t qbyte(int32_t acc) {
    using I = StageInfo<ST>;
    if constexpr (I::fs() != 0) {
        constexpr int sD = I::fs() * ST::D;
        constexpr int64_t ymax = I::fs() * I::acc_max();
        if constexpr (ymax * sD < (int64_t(1) << 21)) {
            // one FFMA: with R = n / 2^23 (n = round(2^23 / (fs D))), 2^23 R is an
            // integer, so K = 1.5 * 2^23 - 2^23 R is exact and (2^23 + y) R + K =
            // 1.5 * 2^23 + y R; |y (R - 1 / (fs D))| <= ymax 2^-24 < 1 / (8 fs D)
            constexpr int64_t n = ((int64_t(1) << 24) / sD + 1) / 2;   // round(2^23 / sD)
            constexpr float R = (float)n / 8388608.0f;
            constexpr float K = 12582912.0f - (float)n;
            return __float_as_uint(fmaf(__uint_as_float((uint32_t)acc), R, K));
        } else {
            constexpr float R = 1.0f / (float)sD;
            const float y = __uint_as_float((uint32_t)acc) - 8388608.0f;    // fs a - c, exact
            return __float_as_uint(fmaf(y, R, 12582912.0f));
        }
    } else {
        return qdiv<ST>(acc);
    }
}

__device__ __forceinline__ int32_t dp4a_us(uint32_t a, uint32_t b, int32_t c) {
    int32_t d;
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// ------------------------------------------------------------ PTX helpers --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    uint32_t r;
    asm("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
// store only when p (no branch: inactive lanes of a warp fall through)
__device__ __forceinline__ void sts32_if(uint32_t a, uint32_t v, bool p) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n}" ::"r"(a), "r"(v),
                 "r"((uint32_t)p)
                 : "memory");
}
__device__ __forceinline__ void lds128(uint32_t a, uint32_t& x, uint32_t& y, uint32_t& z, uint32_t& w) {
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(a));
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// named barriers (warp-specialised kernel): arrive does not wait
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
// L2 prefetch of a contiguous range (TMA engine; no shared memory, no wait)
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// the 16-byte aligned part of a range (the bulk prefetch needs 16-byte
// aligned addresses and sizes; rows of AL < 16 calls lose at most 15 + 15 bytes)
__device__ __forceinline__ void prefetch_range(const uint8_t* p, uint32_t bytes) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p), s = (a + 15) & ~(uintptr_t)15, e = (a + bytes) & ~(uintptr_t)15;
    if (e > s) prefetch_l2(reinterpret_cast<const void*>(s), (uint32_t)(e - s));
}
__device__ __forceinline__ void ldg128(const uint8_t* p, uint32_t& x, uint32_t& y, uint32_t& z, uint32_t& w) {
    asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "l"(p));
}
__device__ __forceinline__ void ldg64(const uint8_t* p, uint32_t& x, uint32_t& y) {
    asm volatile("ld.global.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "l"(p));
}
__device__ __forceinline__ uint32_t ldg32(const uint8_t* p) {
    uint32_t v;
    asm volatile("ld.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
// streaming global stores (the output is never re-read)
__device__ __forceinline__ void stg32_cs(uint8_t* p, uint32_t v) {
    asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void stg16(uint8_t* p, uint32_t v) {
    asm volatile("st.global.cs.u16 [%0], %1;" ::"l"(p), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ void stg8(uint8_t* p, uint32_t v) {
    asm volatile("st.global.cs.u8 [%0], %1;" ::"l"(p), "h"((unsigned short)(v & 0xff)) : "memory");
}

// ------------------------------------------------------------- the H pass --
// One lane: a chunk = 4 consecutive H repetitions r1 = 4c .. 4c+3 of one row.
// Their windows start at bytes o + Sh r1 (o: the plane's H origin reduced to
// (-W/2, W/2]); relative to the chunk's first 16-byte block B = floor(o / 16)
// + (Sh / 4) c that is PH + Sh m (PH = o mod 16, a compile-time constant of
// the instance).  The lane loads exactly the words any live tap reads (loads
// of up to AL bytes by word runs: AL = 16, 8 or 4 is the alignment of every
// row start in the call; AL = 17, 18, 19: every row starts s = AL - 16 words
// past a 16-byte boundary (16-byte rows, a pointer 4, 8 or 12 bytes off), so
// the lane loads the aligned 16-byte blocks around its window and renames
// words; AL = 1: rows start m = 1..3 bytes past a 4-byte boundary, and each
// window word is funnel-shifted out of the two aligned words it straddles),
// then every output is a dp4a per aligned word with a nonzero re-indexed
// weight word.
template <class HS, int PH, int AL = 16>
struct HChunk {
    using I = StageInfo<HS>;
    static_assert(AL == 16 || AL == 8 || AL == 4 || AL == 1 || (AL >= 17 && AL <= 19),
                  "row alignment 16, 8, 4, 1 (funnelled) or 17..19 (16-byte blocks, word shift)");
    static constexpr int kLo = PH / 4;                                   // first word read
    static constexpr int kHi = (PH + 3 * HS::S + I::hi_tap()) / 4;       // last word read
    static constexpr int kWords = kHi + 1;                               // words from B's start
    static constexpr int kBlk = (kWords + 3) / 4;                        // 16-byte blocks touched
    static_assert(kBlk <= 8, "H window too wide for the compiled H pass");

    // x: words kLo .. kHi of the window whose block 0 is block B of the row
    // (B may be negative or run past the row end; others untouched), taken mod
    // W.  Used by the wrap pass for the few chunks per row whose window
    // crosses the row end.  16-byte rows (AL = 16): whole blocks mod W / 16;
    // else word by word (W % 4 == 0, so no word straddles the row end).
    __device__ __forceinline__ static void load_wrap(const uint8_t* row, int B, int W, uint32_t (&x)[4 * kBlk],
                                                     int mis = 0) {
        if constexpr (AL == 1) {
            // each word from the two aligned words around it: both hold one of
            // its (valid) bytes, so neither read leaves the allocation
            const uint8_t* ra = row - mis;
            sfor<kLo, kHi + 1>([&](auto w) {
                int off = 16 * B + 4 * decltype(w)::value;
                if (off < 0) off += W;
                else if (off >= W) off -= W;
                const uint32_t lo = ldg32(ra + off), hi = ldg32(ra + off + 4);
                x[decltype(w)::value] = __funnelshift_r(lo, hi, 8 * mis);
            });
        } else if constexpr (AL == 16) {
            const int nb16 = W >> 4;
            sfor<0, kBlk>([&](auto b) {
                constexpr int w0 = 4 * decltype(b)::value, wlo = w0 > kLo ? w0 : kLo, whi = w0 + 3 < kHi ? w0 + 3 : kHi;
                int blk = B + decltype(b)::value;
                if (blk < 0) blk += nb16;
                else if (blk >= nb16) blk -= nb16;
                const uint8_t* a = row + 16 * blk;
                if constexpr (wlo == w0 && whi == w0 + 3) {
                    ldg128(a, x[w0], x[w0 + 1], x[w0 + 2], x[w0 + 3]);
                } else if constexpr (whi >= wlo) {
                    sfor<wlo - w0, whi - w0 + 1>([&](auto t) { x[w0 + decltype(t)::value] = ldg32(a + 4 * decltype(t)::value); });
                }
            });
        } else {
            sfor<kLo, kHi + 1>([&](auto w) {
                int off = 16 * B + 4 * decltype(w)::value;
                if (off < 0) off += W;
                else if (off >= W) off -= W;
                x[decltype(w)::value] = ldg32(row + off);
            });
        }
    }
    // the same words from a base pointer to the chunk's first block (no wrap)
    __device__ __forceinline__ static void load_at(const uint8_t* base, uint32_t (&x)[4 * kBlk], int mis = 0) {
        if constexpr (AL == 1) {
            // aligned words kLo .. kHi + 1 from base - mis, then one funnel
            // shift per window word (the last aligned word holds a valid byte)
            const uint8_t* ba = base - mis;
            uint32_t a[kHi - kLo + 2];
            sfor<0, kHi - kLo + 2>([&](auto t) { a[decltype(t)::value] = ldg32(ba + 4 * (kLo + decltype(t)::value)); });
            sfor<0, kHi - kLo + 1>([&](auto t) {
                x[kLo + decltype(t)::value] = __funnelshift_r(a[decltype(t)::value], a[decltype(t)::value + 1], 8 * mis);
            });
            return;
        }
        if constexpr (AL > 16) {
            // window word w is aligned word w + s of the 16-byte aligned base;
            // every touched aligned block is loaded whole (it holds a window
            // word, so it lies in the allocation's pages)
            constexpr int sh = AL - 16, alo = kLo + sh, ahi = kHi + sh;
            const uint8_t* ab = base - 4 * sh;
            uint32_t a[4 * (ahi / 4 + 1)];
            sfor<alo / 4, ahi / 4 + 1>([&](auto b) {
                constexpr int w0 = 4 * decltype(b)::value;
                ldg128(ab + 16 * decltype(b)::value, a[w0], a[w0 + 1], a[w0 + 2], a[w0 + 3]);
            });
            sfor<kLo, kHi + 1>([&](auto w) { x[decltype(w)::value] = a[decltype(w)::value + sh]; });
            return;
        }
        sfor<0, kBlk>([&](auto b) {
            constexpr int w0 = 4 * decltype(b)::value, wlo = w0 > kLo ? w0 : kLo, whi = w0 + 3 < kHi ? w0 + 3 : kHi;
            const uint8_t* a = base + 16 * decltype(b)::value;
            if constexpr (AL == 16 && wlo == w0 && whi == w0 + 3) {
                ldg128(a, x[w0], x[w0 + 1], x[w0 + 2], x[w0 + 3]);
            } else if constexpr (whi >= wlo) {
                sfor<wlo - w0, whi - w0 + 1>([&](auto t) {
                    constexpr int w = w0 + decltype(t)::value;
                    if constexpr (AL >= 8 && (w & 1) == 0 && w + 1 <= whi) ldg64(a + 4 * decltype(t)::value, x[w], x[w + 1]);
                    else if constexpr (AL >= 8 && (w & 1) == 1 && w - 1 >= wlo) { /* loaded with w - 1 */ }
                    else x[w] = ldg32(a + 4 * decltype(t)::value);
                });
            }
        });
    }
    // the chunk's 4 Q output bytes, packed little-endian into Q words
    __device__ __forceinline__ static void compute(const uint32_t (&x)[4 * kBlk], uint32_t (&o)[HS::Q]) {
        uint32_t q[4 * HS::Q];
        sfor<0, 4>([&](auto m) {
            sfor<0, HS::Q>([&](auto j) {
                int32_t acc = I::acc0();
                sfor<kLo, kHi + 1>([&](auto b) {
                    constexpr uint32_t wq = I::wword(decltype(j)::value, decltype(b)::value, PH + HS::S * decltype(m)::value);
                    if constexpr (wq != 0) acc = dp4a_us(x[decltype(b)::value], wq, acc);
                });
                q[HS::Q * decltype(m)::value + decltype(j)::value] = qbyte<HS>(acc);
            });
        });
        sfor<0, HS::Q>([&](auto w) {
            const uint32_t lo = __byte_perm(q[4 * decltype(w)::value], q[4 * decltype(w)::value + 1], 0x0040);
            const uint32_t hi = __byte_perm(q[4 * decltype(w)::value + 2], q[4 * decltype(w)::value + 3], 0x0040);
            o[decltype(w)::value] = __byte_perm(lo, hi, 0x5410);
        });
    }
};

// ------------------------------------------------------------- the V pass --
// One lane: V repetition g, 4 intermediate columns (one word per row).  Rows
// no tap reads are not loaded; 4-row blocks with >= 3 live rows are
// transposed into column words (8 PRMT), 2 live rows paired (4 PRMT), a
// single live row folded into shifted-weight dp4a (no PRMT).
template <class VS>
struct VQuad {
    using I = StageInfo<VS>;
    static constexpr int kBlocks = (I::hi_tap() + 4) / 4;
    __host__ __device__ static constexpr int live_in_block(int b) {
        int n = 0;
        for (int t = 0; t < 4; ++t)
            if (4 * b + t < VS::P && I::live(4 * b + t)) ++n;
        return n;
    }
    __host__ __device__ static constexpr int nth_live(int b, int k) {   // row (within the block) of the k-th live row
        for (int t = 0; t < 4; ++t)
            if (4 * b + t < VS::P && I::live(4 * b + t)) {
                if (k == 0) return t;
                --k;
            }
        return 0;
    }

    // mb: shared address of row 0 of the repetition at this lane's 4 columns
    __device__ __forceinline__ static void run(uint32_t mb, int mp, int32_t (&acc)[VS::Q][4]) {
        sfor<0, VS::Q>([&](auto kk) {
            sfor<0, 4>([&](auto e) { acc[decltype(kk)::value][decltype(e)::value] = I::acc0(); });
        });
        sfor<0, kBlocks>([&](auto b) {
            constexpr int nl = live_in_block(decltype(b)::value);
            if constexpr (nl == 1) {
                constexpr int t = nth_live(decltype(b)::value, 0), i = 4 * decltype(b)::value + t;
                const uint32_t r = lds32(mb + i * mp);
                sfor<0, VS::Q>([&](auto kk) {
                    constexpr int wv = I::ws(decltype(kk)::value, i);
                    if constexpr (wv != 0) {
                        sfor<0, 4>([&](auto e) {
                            constexpr uint32_t ws = (uint32_t)(uint8_t)(int8_t)wv << (8 * decltype(e)::value);
                            acc[decltype(kk)::value][decltype(e)::value] = dp4a_us(r, ws, acc[decltype(kk)::value][decltype(e)::value]);
                        });
                    }
                });
            } else if constexpr (nl == 2) {
                constexpr int t0 = nth_live(decltype(b)::value, 0), t1 = nth_live(decltype(b)::value, 1);
                const uint32_t r0 = lds32(mb + (4 * decltype(b)::value + t0) * mp), r1 = lds32(mb + (4 * decltype(b)::value + t1) * mp);
                uint32_t c[4];
                sfor<0, 4>([&](auto e) { c[decltype(e)::value] = __byte_perm(r0, r1, decltype(e)::value | ((4 + decltype(e)::value) << 4)); });
                sfor<0, VS::Q>([&](auto kk) {
                    constexpr uint32_t wq = (uint32_t)(uint8_t)(int8_t)I::ws(decltype(kk)::value, 4 * decltype(b)::value + t0) |
                                            ((uint32_t)(uint8_t)(int8_t)I::ws(decltype(kk)::value, 4 * decltype(b)::value + t1) << 8);
                    if constexpr (wq != 0) {
                        sfor<0, 4>([&](auto e) { acc[decltype(kk)::value][decltype(e)::value] = dp4a_us(c[decltype(e)::value], wq, acc[decltype(kk)::value][decltype(e)::value]); });
                    }
                });
            } else if constexpr (nl >= 3) {
                uint32_t r[4];
                sfor<0, 4>([&](auto t) {
                    constexpr int i = 4 * decltype(b)::value + decltype(t)::value;
                    if constexpr (i < VS::P && I::live(i)) r[decltype(t)::value] = lds32(mb + i * mp);
                    else r[decltype(t)::value] = 0;
                });
                const uint32_t ta = __byte_perm(r[0], r[1], 0x5140), tb = __byte_perm(r[2], r[3], 0x5140);
                const uint32_t tc = __byte_perm(r[0], r[1], 0x7362), td = __byte_perm(r[2], r[3], 0x7362);
                const uint32_t c[4] = {__byte_perm(ta, tb, 0x5410), __byte_perm(ta, tb, 0x7632),
                                       __byte_perm(tc, td, 0x5410), __byte_perm(tc, td, 0x7632)};
                sfor<0, VS::Q>([&](auto kk) {
                    constexpr uint32_t wq = I::wword(decltype(kk)::value, decltype(b)::value, 0);
                    if constexpr (wq != 0) {
                        sfor<0, 4>([&](auto e) { acc[decltype(kk)::value][decltype(e)::value] = dp4a_us(c[decltype(e)::value], wq, acc[decltype(kk)::value][decltype(e)::value]); });
                    }
                });
            }
        });
    }
};

// ------------------------------------------------------------ the kernel --
template <class HS, class VS, int PH, int AL>
__global__ void __launch_bounds__(DS_SPEC_THREADS, DS_SPEC_MINB) ds_spec_kernel(const __grid_constant__ SpecParams p) {
    // NW warps run the H pass (NT threads); with DS_SPEC_WS, NWV more warps run
    // the V pass (NTV threads) and the two groups hand the two intermediate
    // buffers back and forth through named barriers: FULL[b] = 1 + b (H arrives,
    // V waits), EMPTY[b] = 3 + b (V arrives, H waits), 5: the H warps alone
    constexpr int NW = DS_SPEC_NW, NT = NW * 32;
    [[maybe_unused]] constexpr int NTALL = DS_SPEC_THREADS;
#if DS_SPEC_WS
    constexpr int NTV = DS_SPEC_NWV * 32;
#else
    constexpr int NTV = NT;
#endif
    static_assert(HS::S % 4 == 0, "a chunk of 4 H repetitions must start on a 16-byte block");
    using HC = HChunk<HS, PH, AL>;
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t mid0 = smem_u32(smem);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    // Units: CTA b takes units b, b + grid, ...; unit u -> frame f = u / upf and
    // unit (u mod upf + f) mod upf of that frame: rotating by the frame index is
    // a bijection per frame, and it hands a CTA every unit kind even when upf
    // divides the grid (units differ in size: planes, run lengths; unrotated,
    // 1200 HD halo frames ran 25% slower).  Incremental: no division per unit.
    const int32_t n_units = (int32_t)p.n_units;          // < 2^31 (the host splits larger calls)
    const int32_t upf = p.upf;
    int32_t u = blockIdx.x;
    int32_t f = (int32_t)(blockIdx.x / (uint32_t)upf);
    int32_t lraw = (int32_t)blockIdx.x - f * upf;        // u mod upf
    int32_t fm = (int32_t)((uint32_t)f % (uint32_t)upf); // f mod upf
    const int32_t gdiv = (int32_t)(gridDim.x / (uint32_t)upf), gmod = (int32_t)gridDim.x - gdiv * upf;
    const int32_t gdm = (int32_t)((uint32_t)gdiv % (uint32_t)upf);
    auto rot = [&](int32_t lr, int32_t fmod) { const int32_t l = lr + fmod; return l >= upf ? l - upf : l; };
    auto advance = [&](int32_t& f_, int32_t& lr, int32_t& fm_) {
        f_ += gdiv;
        fm_ += gdm;
        lr += gmod;
        if (lr >= upf) { lr -= upf; ++f_; ++fm_; }
        if (fm_ >= upf) fm_ -= upf;
    };
    int32_t local = rot(lraw, fm);
    int mpar = 0;

    // L2 prefetch (one thread) of the new input rows of band `band` of unit
    // (f_, local_): rows (ov + Sv k band + reuse + i) mod H, i < rows, as one or
    // two contiguous ranges -- the TMA engine streams them into L2 while the CTA
    // computes the current band, so the H loads of the next band hit L2
    auto prefetch_band = [&](int64_t f_, int32_t local_, int band_rel) {
        const int pi_ = (p.n_planes > 2 && local_ >= p.pl[2].unit_start) ? 2
                        : (p.n_planes > 1 && local_ >= p.pl[1].unit_start) ? 1 : 0;
        const SpecPlane& Q = p.pl[pi_];
        const int bnd = (local_ - Q.unit_start) * Q.L + band_rel;
        if (bnd >= Q.nb) return;
        const int reuse_ = band_rel > 0 ? p.ovl : 0;
        const int rows_ = VS::S * (Q.k - 1) + VS::P - reuse_;
        int r0 = (int)((uint32_t)(Q.ov + VS::S * Q.k * bnd + reuse_) % (uint32_t)Q.H);   // < 2^31
        const uint8_t* pl_ = p.in + f_ * p.in_frame + Q.in_off;
        const int n1 = min(rows_, Q.H - r0);
        prefetch_range(pl_ + (int64_t)r0 * Q.W, (uint32_t)n1 * (uint32_t)Q.W);
        if (rows_ > n1) prefetch_range(pl_, (uint32_t)min(rows_ - n1, Q.H) * (uint32_t)Q.W);
    };
    if (tid == 0 && u < n_units) prefetch_band(f, local, 0);
#if DS_SPEC_WS
    const bool hrole = warp < NW;
    const int vtid = tid - NT;                            // V role: 0 .. NTV - 1
    if (!hrole) {                                         // both buffers start empty
        named_arrive(3, NTALL);
        named_arrive(4, NTALL);
    }
#else
    constexpr bool hrole = true;
    const int vtid = tid;
#endif

    for (; u < n_units; u += gridDim.x) {
        const int pi = (p.n_planes > 2 && local >= p.pl[2].unit_start) ? 2
                       : (p.n_planes > 1 && local >= p.pl[1].unit_start) ? 1 : 0;
        const SpecPlane& P = p.pl[pi];
        const int run = local - P.unit_start;
        const int b0 = run * P.L, b1 = min(b0 + P.L, P.nb);
        const uint8_t* plane = p.in + f * p.in_frame + P.in_off;
        uint8_t* oplane = p.out + f * p.out_frame + P.out_off;
        if (p.unit_count != nullptr && tid == 0) atomicAdd(p.unit_count + u, 1u);
        const int mp = P.mp;
        const int rfirst = VS::S * (P.k - 1) + VS::P;             // rows of a run's first band
        // next unit of this CTA (for the prefetch of its first band)
        int32_t fn = f, lrn = lraw, fmn = fm;
        advance(fn, lrn, fmn);
        const int32_t ln = rot(lrn, fmn);

        // A warp keeps one 32-chunk segment of the row for the whole unit (segs is a
        // power of two dividing NW): its window blocks are fixed; it walks rows
        // i = warp >> lgsegs, + step, ... with a running row pointer.  Chunks whose
        // window crosses the row end (at most a few per row) are left to a
        // small wrap pass, so the main loop has no per-block index arithmetic.
        // Rows of at most 16 chunks: a warp takes 2^lgrpw rows at once, lane
        // groups of 32 >> lgrpw chunk lanes (row lane rsub).
        const int lgrpw = P.lgrpw, cwm = (32 >> lgrpw) - 1;
        const int seg = warp & (P.segs - 1), step = (NW >> P.lgsegs) << lgrpw;
        const int ch = seg * 32 + (lane & cwm);
        // the chunk's window words inside the row: the main loop's; else the wrap pass's
        int B = P.blk0 + (HS::S / 4) * ch;
        const bool act = ch < P.nch && 16 * B + 4 * HC::kLo >= 0 && 16 * B + 4 * (HC::kHi + 1) <= P.W;
        if (!act) B = P.nb16 - HC::kBlk;                            // in-bounds loads, result unused
        const int i0w = (warp >> P.lgsegs) << lgrpw;               // the warp's first row
        const int i0 = i0w + (lane >> (5 - lgrpw));                 // this lane's
        // issue cursor: a 32-bit byte offset of the lane's window in the plane
        // (planes are < 2^31 bytes); it advances `step` rows per issue and wraps
        // at the plane bottom by one compare and subtract
        const uint32_t rowstep = (uint32_t)(step * P.W), plane_bytes = (uint32_t)P.H * (uint32_t)P.W;
        const uint8_t* const wbase = plane + 16 * B;
        uint32_t roff = 0;
        uint32_t x0[4 * HC::kBlk], x1[4 * HC::kBlk];
#if DS_SPEC_DEPTH3
        uint32_t x2[4 * HC::kBlk];
#endif
        auto seek = [&](int first_row) {
            int rr = first_row + i0;
            while (rr >= P.H) rr -= P.H;
            roff = (uint32_t)rr * (uint32_t)P.W;
        };
        auto issue = [&](uint32_t (&x)[4 * HC::kBlk]) {
            HC::load_at(wbase + roff, x, p.in_mis);
            roff += rowstep;
            if (roff >= plane_bytes) roff -= plane_bytes;
        };
        // passes of this warp over a band of `rows` rows: rows i0w + rsub, + step,
        // ...; a later row lane may run one row past the band in the last pass
        // (its result lands in the buffer's spare rows, never read)
        const int lgstep = DS_SPEC_LGNW - P.lgsegs + lgrpw;        // step is a power of two
        auto my_rows = [&](int rows) { return rows > i0w ? (rows - i0w + step - 1) >> lgstep : 0; };
        bool preloaded = false;

        for (int band = b0; band < b1; ++band) {
            const uint32_t mid = mid0 + mpar * p.mid_stride;
            const int reuse = band > b0 ? p.ovl : 0;
          if (hrole) {
#if DS_SPEC_WS
            named_sync(3 + mpar, NTALL);                  // V is done with this buffer (band - 2)
            if (reuse) named_sync(5, NT);                 // every H warp is done with band - 1
#endif
            if (tid == 0) {
                if (band + 1 < b1) {
                    prefetch_band(f, local, band + 1 - b0);
                } else if (u + (int32_t)gridDim.x < n_units) {    // the next unit's first band
                    prefetch_band(fn, ln, 0);
                }
            }
            if (reuse) {
                // the previous band's intermediate rows [Sv k, Sv k + ovl) are this
                // band's rows [0, ovl): contiguous, so a 16-byte vector copy
                const uint32_t src = mid0 + (mpar ^ 1) * p.mid_stride + VS::S * P.k * mp;
                for (int x = 16 * tid; x < reuse * mp; x += 16 * NT) {
                    uint32_t a0, a1, a2, a3;
                    lds128(src + x, a0, a1, a2, a3);
                    sts128(mid + x, a0, a1, a2, a3);
                }
            }
            // ---- H task: input rows (ov + Sv k band + reuse + i) mod H -> intermediate rows reuse + i;
            // the next row's loads are in flight while a row computes (two register
            // buffers); the first row of the next band is issued before this band's
            // V pass
            const int rows = rfirst - reuse;
            int row0 = P.ov + VS::S * P.k * band + reuse;
            while (row0 >= P.H) row0 -= P.H;
            // inactive lanes (past the row, or a wrapping chunk left to the wrap
            // pass) store their garbage into a scratch chunk past the row's
            // chunks (mp >= 4 Qh ((cwm + 1) segs + 1)), so the stores need no predicate
            const uint32_t mcol = mid + (reuse + i0) * mp + 4 * HS::Q * (act ? ch : (cwm + 1) * P.segs);
            const uint32_t mstep = step * mp;
            auto finish = [&](int k, const uint32_t (&x)[4 * HC::kBlk]) {
                uint32_t o[HS::Q];
                HC::compute(x, o);
                const uint32_t mo = mcol + k * mstep;
                sfor<0, HS::Q>([&](auto w) { sts32(mo + 4 * decltype(w)::value, o[decltype(w)::value]); });
            };
            const int n_my = my_rows(rows);
            if (!preloaded && n_my > 0) {
                seek(row0);
                issue(x0);
            }
            int k = 0;
#if DS_SPEC_DEPTH3
            // three register buffers: rows k, k + 1, k + 2 in flight
            if (n_my > 1) issue(x1);
            for (; k + 3 <= n_my; k += 3) {
                issue(x2);
                finish(k, x0);
                if (k + 3 < n_my) issue(x0);
                finish(k + 1, x1);
                if (k + 4 < n_my) issue(x1);
                finish(k + 2, x2);
            }
            if (k < n_my) finish(k, x0);
            if (k + 1 < n_my) finish(k + 1, x1);
#else
            for (; k + 2 <= n_my; k += 2) {                             // rows k and k + 1 are this warp's
                issue(x1);
                finish(k, x0);
                if (k + 2 < n_my) issue(x0);
                finish(k + 1, x1);
            }
            if (k < n_my) finish(k, x0);
#endif
            // wrap pass: (row, wrapping chunk) items over all threads, from the last
            // warps down (they have the fewest main-loop rows)
            for (int it = NT - 1 - tid; it < rows * P.nwc; it += NT) {
                // it / nwc for nwc <= 4 and it < 2^14: a 16-bit reciprocal
                const int i = (int)(((uint32_t)it * (uint32_t)(P.nwc == 1 ? 65536 : P.nwc == 2 ? 32768 : P.nwc == 3 ? 21846 : 16384)) >> 16);
                const int c = P.wch[it - i * P.nwc];
                int r = row0 + i;
                while (r >= P.H) r -= P.H;
                uint32_t xw[4 * HC::kBlk], o[HS::Q];
                HC::load_wrap(plane + (int64_t)r * P.W, P.blk0 + (HS::S / 4) * c, P.W, xw, p.in_mis);
                HC::compute(xw, o);
                const uint32_t mo = mid + (reuse + i) * mp + 4 * HS::Q * c;
                sfor<0, HS::Q>([&](auto w) { sts32(mo + 4 * decltype(w)::value, o[decltype(w)::value]); });
            }
            // the next band's first row (same unit) is issued across the barrier
            preloaded = band + 1 < b1 && my_rows(rfirst - p.ovl) > 0;
            if (preloaded) {
                int nrow0 = P.ov + VS::S * P.k * (band + 1) + p.ovl;
                while (nrow0 >= P.H) nrow0 -= P.H;
                seek(nrow0);
                issue(x0);
            }
#if DS_SPEC_WS
            named_arrive(1 + mpar, NTALL);                // intermediate complete
          }
          if (!hrole) {
            named_sync(1 + mpar, NTALL);
#else
          }
            __syncthreads();                                               // intermediate complete
#endif

            // ---- V task: intermediate -> output rows, straight to HBM
            {
                const int wm = HS::Q * P.np;
                const int items = P.k * P.nq;
                uint8_t* obase = oplane + (int64_t)VS::Q * P.k * band * P.Wout;
                auto vitem = [&](int it, auto fast) {
                    const int g = P.nq > 1 ? (int)__umulhi((uint32_t)it, P.nq_rcp) : it;
                    const int q = it - g * P.nq;
                    int32_t acc[VS::Q][4];
                    VQuad<VS>::run(mid + VS::S * g * mp + 4 * q, mp, acc);
                    uint8_t* o = obase + (int64_t)VS::Q * g * P.Wout + 4 * q;
                    sfor<0, VS::Q>([&](auto kk) {
                        const uint32_t c0 = qbyte<VS>(acc[decltype(kk)::value][0]), c1 = qbyte<VS>(acc[decltype(kk)::value][1]),
                                       c2 = qbyte<VS>(acc[decltype(kk)::value][2]), c3 = qbyte<VS>(acc[decltype(kk)::value][3]);
                        uint8_t* d = o + (int64_t)decltype(kk)::value * P.Wout;
                        if constexpr (decltype(fast)::value == 1) {
                            stg32_cs(d, __byte_perm(__byte_perm(c0, c1, 0x0040), __byte_perm(c2, c3, 0x0040), 0x5410));
                        } else {
                            const bool whole = 4 * q + 4 <= wm;
                            const uint32_t al = (uint32_t)(uintptr_t)d & 3;
                            if (whole && al == 0) {
                                stg32_cs(d, __byte_perm(__byte_perm(c0, c1, 0x0040), __byte_perm(c2, c3, 0x0040), 0x5410));
                            } else if (whole && al == 2) {                 // e.g. CIF chroma: 66-byte rows
                                stg16(d, __byte_perm(c0, c1, 0x0040));
                                stg16(d + 2, __byte_perm(c2, c3, 0x0040));
                            } else {
                                const int n = whole ? 4 : wm - 4 * q;
                                stg8(d, c0);
                                if (n > 1) stg8(d + 1, c1);
                                if (n > 2) stg8(d + 2, c2);
                                if (n > 3) stg8(d + 3, c3);
                            }
                        }
                    });
                };
                if (p.out_al4 && wm % 4 == 0) {                         // every quad a whole aligned word
                    for (int it = vtid; it < items; it += NTV) vitem(it, IC<1>{});
                } else {
                    for (int it = vtid; it < items; it += NTV) vitem(it, IC<0>{});
                }
            }
#if DS_SPEC_WS
            named_arrive(3 + mpar, NTALL);                // this buffer may be refilled
          }
#endif
            mpar ^= 1;
        }
        f = fn;
        lraw = lrn;
        fm = fmn;
        local = ln;
    }
#if DS_SPEC_WS
    if (hrole) {                                          // take the V warps' last two arrivals
        named_sync(3 + mpar, NTALL);
        named_sync(3 + (mpar ^ 1), NTALL);
    }
#endif
}

}  // namespace dss
