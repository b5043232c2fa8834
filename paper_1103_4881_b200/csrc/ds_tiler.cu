// ds_tiler.cu -- SURVEY f4: a general Array-OL repetitive task on sm_100a
// (arbitrary <= 4-D origin / paving / fitting tilers), SPEC's launch
// topology rule as an optional launch policy, and check_coverage
// on the device.  Citations: P:n = PAPER.md line n, S:n = SPEC.md
// line n.
//
// Element indices follow S:248-252 exactly: (origin + paving.r + fitting.f)
// mod shape with the non-negative modulo.  The host reduces origin, paving
// columns and the per-pattern-element fitting offsets modulo the shape once;
// a thread then needs, per array dim, one product-sum and one modulo per
// repetition plus one conditional subtraction per pattern element.
#include <algorithm>
#include <climits>
#include <cstring>

#include "ds.h"
#include "ds_internal.h"

namespace {

struct TTiler {
    int32_t ndim, npe;                 // array dims, pattern elements
    int64_t shape[4];
    int64_t stride[4];                 // row-major element strides
    int64_t origin[4];                 // reduced mod shape
    int64_t pav[4][4];                 // [array dim][rep dim], reduced mod shape
    int64_t foff[DS_MAX_PATTERN][4];   // fitting . f for each pattern element, reduced mod shape
};

// n / d and n % d for 0 <= n < 2^31 by multiply-high (d > 1), after the
// classic round-up reciprocal: p = 31 + ceil(log2 d), m = ceil(2^p / d).
struct FastDiv {
    uint32_t d, m, s;
};

struct TaskParams {
    const uint8_t* in;
    uint8_t* out;
    int64_t n_reps;
    int32_t fast32;                    // every index quantity < 2^31 (host-checked)
    int32_t noclamp;                   // fastdiv and every acc in [0, 256 D): output = umulhi(acc, M)
    FastDiv rdiv[4];                   // repetition extents
    FastDiv sdiv_in[4], sdiv_out[4];   // array extents
    int32_t nrep;
    int32_t policy;
    int64_t rep[4];
    TTiler tin, tout;
    int32_t n_in, n_out, divisor, bias;
    int32_t w[DS_MAX_OUTPUTS][DS_MAX_PATTERN];
    // DS_TOPO_SPEC: collapsed multiplicity (row-major, last fastest) and the
    // CUDA axis (0 = x, 1 = y, 2 = z) each collapsed dim is launched along
    int32_t tdim;
    int64_t tmult[3];
    int32_t tax[3];
    // Affine path (host-proved: no tiler index wraps anywhere in the box, so the
    // element offset is A + sum_j a[j] r_j + b[e], all in [0, n) < 2^31)
    int32_t affine;                    // 0: modulo path; 1: byte loads; 2: word loads + dp4a;
                                       // 3: 4 consecutive repetitions (columns) per thread
    uint32_t in_A, out_A;
    uint32_t in_a[4], out_a[4];
    int32_t in_b[DS_MAX_PATTERN], out_b[DS_MAX_OUTPUTS];
    uint32_t wp[DS_MAX_OUTPUTS][DS_MAX_PATTERN / 4];   // s8-packed weights (affine == 2)
    // exact division: clamp(trunc(acc / D)) = min(umulhi(max(acc + fb - bias, lo), M), 255)
    // when fastdiv (host-checked range), else the integer division
    int32_t fastdiv, fbias;
    uint32_t M, lo;
    int32_t dense;                     // affine == 2 and both tilers are dense row-major runs
    uint32_t in_live;                  // bit e: pattern element e has a nonzero tap for some output
    // column path: in_b with every element that has no tap (dead, or past
    // n_in) aliased to the first live one, so all 4 NB word loads are
    // unconditional (zero taps ignore the value; the repeat is an L1 hit)
    int32_t in_bl[DS_MAX_PATTERN];
    // word path: (in + element offset) mod 4, the same for every repetition
    // (all repetition strides are multiples of 4); nonzero -> NI/4 + 1 aligned
    // words funnelled by m bytes
    int32_t in_shift;
};

__device__ __forceinline__ int64_t t_mod(int64_t a, int64_t m) {
    const int64_t r = a % m;
    return r < 0 ? r + m : r;
}

// Base index (origin + paving.r) mod shape for every array dim.
__device__ __forceinline__ void t_base(const TTiler& t, int nrep, const int64_t* r, int64_t* base) {
    for (int d = 0; d < t.ndim; ++d) {
        int64_t v = t.origin[d];
        for (int j = 0; j < nrep; ++j) v += (t.pav[d][j] * r[j]) % t.shape[d];
        base[d] = t_mod(v, t.shape[d]);
    }
}

__device__ __forceinline__ int64_t t_lin(const TTiler& t, const int64_t* base, int f) {
    int64_t off = 0;
    for (int d = 0; d < t.ndim; ++d) {
        int64_t i = base[d] + t.foff[f][d];
        if (i >= t.shape[d]) i -= t.shape[d];
        off += i * t.stride[d];
    }
    return off;
}

__device__ __forceinline__ void t_unravel(int64_t q, int nrep, const int64_t* rep, int64_t* r) {
    for (int j = nrep - 1; j >= 0; --j) {
        r[j] = q % rep[j];
        q /= rep[j];
    }
}

__device__ __forceinline__ uint32_t fdiv(const FastDiv& f, uint32_t n) {
    return f.d == 1 ? n : (__umulhi(n, f.m) >> f.s);
}
__device__ __forceinline__ uint32_t fmod32(const FastDiv& f, uint32_t n) { return n - fdiv(f, n) * f.d; }

// 32-bit path: origin + paving.r stays < 2^31 (host bound), one modulo per
// dim.  Loops are fully unrolled over the maximum extents with predicates so
// the pattern and index arrays stay in registers.
// base[] is already reduced mod shape (t_base32) and foff < shape, so each
// element index needs one conditional subtraction, not a modulo.
__device__ __forceinline__ uint32_t t_lin32(const TTiler& t, const FastDiv* sd, const uint32_t* base,
                                            int f) {
    uint32_t off = 0;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
        if (d < t.ndim) {
            uint32_t i = base[d] + (uint32_t)t.foff[f][d];
            if (i >= sd[d].d) i -= sd[d].d;
            off += i * (uint32_t)t.stride[d];
        }
    }
    return off;
}

// (origin + paving.r) mod shape per array dim: one modulo per dim per repetition
__device__ __forceinline__ void t_base32(const TTiler& t, const FastDiv* sd, int nrep, const uint32_t* r,
                                         uint32_t* base) {
#pragma unroll
    for (int d = 0; d < 4; ++d) {
        uint32_t v = (uint32_t)t.origin[d];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (j < nrep) v += (uint32_t)t.pav[d][j] * r[j];
        base[d] = d < t.ndim ? fmod32(sd[d], v) : 0u;
    }
}

// d = c + sum_i a.u8[i] * b.s8[i]
__device__ __forceinline__ int32_t t_dp4a(uint32_t a, uint32_t b, int32_t c) {
    int32_t d;
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint8_t t_out(const TaskParams& p, int32_t acc) {
    if (p.fastdiv) return (uint8_t)min(__umulhi((uint32_t)max(acc, (int32_t)p.lo), p.M), 255u);
    int32_t v = acc / p.divisor;                          // truncation toward zero
    return (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v));
}

// t_out where the host proved the clamps never fire (noclamp): one umulhi
template <bool NC>
__device__ __forceinline__ uint32_t t_outc(const TaskParams& p, int32_t acc) {
    if (NC) return __umulhi((uint32_t)acc, p.M);
    return t_out(p, acc);
}

// Modulo path, 32-bit: NI = n_in rounded up to 4 (the MAC loop runs over NI
// taps, not DS_MAX_PATTERN); exact multiply-high division when host-proved.
template <int NI>
__device__ __forceinline__ void task_one32(const TaskParams& p, uint32_t q) {
    uint32_t r[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 3; j >= 0; --j) {
        if (j == 0) {
            r[0] = q;                          // q < rep[0]: no division
        } else if (j < p.nrep) {
            const uint32_t qq = fdiv(p.rdiv[j], q);
            r[j] = q - qq * p.rdiv[j].d;
            q = qq;
        }
    }
    uint32_t base[4];
    t_base32(p.tin, p.sdiv_in, p.nrep, r, base);
    int32_t pat[NI];
#pragma unroll
    for (int f = 0; f < NI; ++f)
        pat[f] = (f < p.n_in && ((p.in_live >> f) & 1u))
                     ? (int32_t)__ldg(p.in + t_lin32(p.tin, p.sdiv_in, base, f)) : 0;
    t_base32(p.tout, p.sdiv_out, p.nrep, r, base);
#pragma unroll
    for (int k = 0; k < DS_MAX_OUTPUTS; ++k) {
        if (k < p.n_out) {
            int32_t acc = p.fastdiv ? p.fbias : p.bias;
#pragma unroll
            for (int f = 0; f < NI; ++f) acc += p.w[k][f] * pat[f];
            p.out[t_lin32(p.tout, p.sdiv_out, base, k)] = t_out(p, acc);
        }
    }
}

template <int NI>
__device__ __forceinline__ void task_one(const TaskParams& p, int64_t q) {
    if (p.fast32) {
        task_one32<NI>(p, (uint32_t)q);
        return;
    }
    int64_t r[4] = {0, 0, 0, 0}, base[4];
    t_unravel(q, p.nrep, p.rep, r);
    uint8_t pat[DS_MAX_PATTERN];
    t_base(p.tin, p.nrep, r, base);
    for (int f = 0; f < p.n_in; ++f) pat[f] = __ldg(p.in + t_lin(p.tin, base, f));
    t_base(p.tout, p.nrep, r, base);
    for (int k = 0; k < p.n_out; ++k) {
        int32_t acc = p.bias;
        for (int f = 0; f < p.n_in; ++f) acc += p.w[k][f] * (int32_t)pat[f];
        int32_t v = acc / p.divisor;                      // truncation toward zero
        v = v < 0 ? 0 : (v > 255 ? 255 : v);
        p.out[t_lin(p.tout, base, k)] = (uint8_t)v;
    }
}

// One elementary task on the affine path (same result as task_one: the
// offsets are the S:248-252 element indices, proved wrap-free on the host).
// NI = n_in rounded up to 4 (weights past n_in are zero); WORDS: the pattern is
// NI contiguous, 4-byte aligned input bytes and the taps fit s8.
template <int NI, bool WORDS, int Q>
__device__ __forceinline__ void task_affine(const TaskParams& p, uint32_t q) {
    uint32_t bi = p.in_A, bo = p.out_A;
#pragma unroll
    for (int j = 3; j >= 0; --j) {
        if (j == 0) {                          // q < rep[0]: no division
            bi += p.in_a[0] * q;
            bo += p.out_a[0] * q;
        } else if (j < p.nrep) {
            const uint32_t qq = fdiv(p.rdiv[j], q);
            const uint32_t r = q - qq * p.rdiv[j].d;
            bi += p.in_a[j] * r;
            bo += p.out_a[j] * r;
            q = qq;
        }
    }
    int32_t acc[Q];
    if (WORDS) {
        uint32_t x[NI / 4];
        const uint32_t* src = reinterpret_cast<const uint32_t*>(p.in + bi - p.in_shift);
        if (p.in_shift) {
            // the last aligned word holds byte bi + NI - 1, so it stays inside the allocation
            const uint32_t sel = 0x3210u + 0x1111u * (uint32_t)p.in_shift;
            uint32_t lo = __ldg(src);
#pragma unroll
            for (int i = 0; i < NI / 4; ++i) {
                const uint32_t hi = __ldg(src + i + 1);
                x[i] = __byte_perm(lo, hi, sel);
                lo = hi;
            }
        } else {
#pragma unroll
            for (int i = 0; i < NI / 4; ++i) x[i] = __ldg(src + i);
        }
#pragma unroll
        for (int k = 0; k < Q; ++k) {
            int32_t a = p.bias;
#pragma unroll
            for (int i = 0; i < NI / 4; ++i) a = t_dp4a(x[i], p.wp[k][i], a);
            acc[k] = a;
        }
    } else {
        int32_t pat[NI];
#pragma unroll
        for (int e = 0; e < NI; ++e) pat[e] = (int32_t)__ldg(p.in + bi + p.in_bl[e]);   // aliased: no predicates
#pragma unroll
        for (int k = 0; k < Q; ++k) {
            int32_t a = p.bias;
#pragma unroll
            for (int e = 0; e < NI; ++e) a += p.w[k][e] * pat[e];
            acc[k] = a;
        }
    }
#pragma unroll
    for (int k = 0; k < Q; ++k) p.out[bo + p.out_b[k]] = t_out(p, acc[k] + (p.fastdiv ? p.fbias - p.bias : 0));
}

template <int NI, bool WORDS, int Q>
__global__ void __launch_bounds__(256) ds_task_affine_kernel(const __grid_constant__ TaskParams p) {
    if (p.policy == DS_TOPO_SPEC) {
        const uint32_t hw[3] = {blockIdx.x * blockDim.x + threadIdx.x, blockIdx.y * blockDim.y + threadIdx.y,
                                blockIdx.z * blockDim.z + threadIdx.z};
        uint32_t q = 0;
        for (int d = 0; d < p.tdim; ++d) {
            const uint32_t c = hw[p.tax[d]];
            if (c >= (uint32_t)p.tmult[d]) return;        // guard
            q = q * (uint32_t)p.tmult[d] + c;
        }
        task_affine<NI, WORDS, Q>(p, q);
        return;
    }
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < (uint32_t)p.n_reps; q += stride)
        task_affine<NI, WORDS, Q>(p, q);
}

// Dense task (host-proved: input element offset in_A + n_in q + e, output
// offset out_A + n_out q + k, q the row-major repetition index; taps s8,
// n_in % 4 == 0, input run 16-byte aligned, output run 4-byte aligned): a
// streaming map.  Each lane takes 4 consecutive repetitions (16-byte loads);
// the warp stages its 128 Q output bytes in shared memory and writes them as
// coalesced words.  Repetitions past the last full warp use task_affine.
template <int NI, int Q, bool NC>
__device__ __forceinline__ void dense_loop(const TaskParams& p, uint32_t* b) {
    const int lane = threadIdx.x & 31;
    const uint32_t full = (uint32_t)(p.n_reps / 128);
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const int32_t b0 = p.fastdiv ? p.fbias : p.bias;
    for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < full; w += nw) {
        const uint32_t rep0 = w * 128 + 4 * lane;
        const uint4* src = reinterpret_cast<const uint4*>(p.in + p.in_A + (uint32_t)NI * rep0);
        uint32_t x[NI];
#pragma unroll
        for (int i = 0; i < NI / 4; ++i) {
            const uint4 v = __ldg(src + i);
            x[4 * i] = v.x; x[4 * i + 1] = v.y; x[4 * i + 2] = v.z; x[4 * i + 3] = v.w;
        }
        // the lane's 4 repetitions x Q outputs are 4 Q consecutive bytes: Q words
        uint32_t ow[Q];
#pragma unroll
        for (int j = 0; j < Q; ++j) ow[j] = 0;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
#pragma unroll
            for (int k = 0; k < Q; ++k) {
                int32_t acc = b0;
#pragma unroll
                for (int i = 0; i < NI / 4; ++i) acc = t_dp4a(x[r * (NI / 4) + i], p.wp[k][i], acc);
                ow[(r * Q + k) >> 2] |= t_outc<NC>(p, acc) << (8 * ((r * Q + k) & 3));
            }
        }
#pragma unroll
        for (int j = 0; j < Q; ++j) b[lane * Q + j] = ow[j];
        __syncwarp();
        uint32_t* dst = reinterpret_cast<uint32_t*>(p.out + p.out_A + Q * 128 * w);
#pragma unroll
        for (int j = 0; j < Q; ++j) dst[lane + 32 * j] = b[lane + 32 * j];
        __syncwarp();
    }
}
template <int NI, int Q>
__global__ void __launch_bounds__(256) ds_task_dense_kernel(const __grid_constant__ TaskParams p) {
    __shared__ __align__(16) uint32_t buf[8][32 * Q];
    uint32_t* b = buf[threadIdx.x >> 5];
    if (p.noclamp) dense_loop<NI, Q, true>(p, b);
    else dense_loop<NI, Q, false>(p, b);
    const uint32_t full = (uint32_t)(p.n_reps / 128);
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t q = full * 128 + blockIdx.x * blockDim.x + threadIdx.x; q < (uint32_t)p.n_reps; q += stride)
        task_affine<NI, true, Q>(p, q);
}

template <int NB>
__device__ __forceinline__ void cols_load(const TaskParams& p, uint32_t q4, uint32_t (&x)[4 * NB], uint32_t& bo) {
    uint32_t q = 4 * q4, bi = p.in_A;
    bo = p.out_A;
#pragma unroll
    for (int j = 3; j >= 0; --j) {
        if (j == 0) {                          // q < rep[0]: no division
            bi += p.in_a[0] * q;
            bo += p.out_a[0] * q;
        } else if (j < p.nrep) {
            const uint32_t qq = fdiv(p.rdiv[j], q);
            const uint32_t r = q - qq * p.rdiv[j].d;
            bi += p.in_a[j] * r;
            bo += p.out_a[j] * r;
            q = qq;
        }
    }
    const uint8_t* src = p.in + bi;
#pragma unroll
    for (int e = 0; e < 4 * NB; ++e)           // elements with no nonzero tap re-read a live one
        x[e] = __ldg(reinterpret_cast<const uint32_t*>(src + p.in_bl[e]));
}
template <int NB, int Q, bool NC>
__device__ __forceinline__ void cols_compute(const TaskParams& p, const uint32_t (&x)[4 * NB], uint32_t bo) {
    int32_t acc[Q][4];
    const int32_t b0 = p.fastdiv ? p.fbias : p.bias;
#pragma unroll
    for (int k = 0; k < Q; ++k)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[k][c] = b0;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const uint32_t r0 = x[4 * b], r1 = x[4 * b + 1], r2 = x[4 * b + 2], r3 = x[4 * b + 3];
        const uint32_t ta = __byte_perm(r0, r1, 0x5140), tb = __byte_perm(r2, r3, 0x5140);
        const uint32_t tc = __byte_perm(r0, r1, 0x7362), td = __byte_perm(r2, r3, 0x7362);
        const uint32_t c0 = __byte_perm(ta, tb, 0x5410), c1 = __byte_perm(ta, tb, 0x7632),
                       c2 = __byte_perm(tc, td, 0x5410), c3 = __byte_perm(tc, td, 0x7632);
#pragma unroll
        for (int k = 0; k < Q; ++k) {
            const uint32_t wq = p.wp[k][b];
            acc[k][0] = t_dp4a(c0, wq, acc[k][0]);
            acc[k][1] = t_dp4a(c1, wq, acc[k][1]);
            acc[k][2] = t_dp4a(c2, wq, acc[k][2]);
            acc[k][3] = t_dp4a(c3, wq, acc[k][3]);
        }
    }
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        const uint32_t o = t_outc<NC>(p, acc[k][0]) | (t_outc<NC>(p, acc[k][1]) << 8) |
                           (t_outc<NC>(p, acc[k][2]) << 16) | (t_outc<NC>(p, acc[k][3]) << 24);
        *reinterpret_cast<uint32_t*>(p.out + bo + p.out_b[k]) = o;
    }
}

// Column-vector task (host-proved: the innermost repetition dimension is
// unit-stride in both arrays with an extent divisible by 4, every other
// offset 4-byte aligned, s8 taps): a thread takes 4 consecutive repetitions.
// Pattern element e of the 4 repetitions is one aligned word; 4 elements x 4
// repetitions are transposed into 4 column words (one dp4a per 4 taps per
// repetition), and output element k of the 4 repetitions is one word store.
// This is the shape of the paper's V task (9 rows down a column -> 4 rows).
// (Two quads per thread step measured slower: 64-99 registers, spills.)
// registers scale with the live words (4 NB) and accumulators (4 Q): small
// shapes (the paper's V task: NB 3, Q 4) run 8 blocks per SM, large ones fewer
constexpr int cols_minb(int nb, int q) { return nb * q <= 12 ? 8 : nb * q <= 24 ? 6 : 4; }
template <int NB, int Q, bool NC>
__device__ __forceinline__ void cols_loop(const TaskParams& p) {
    const uint32_t quads = (uint32_t)(p.n_reps >> 2);
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t q4 = blockIdx.x * blockDim.x + threadIdx.x; q4 < quads; q4 += stride) {
        uint32_t x[4 * NB], bo;
        cols_load<NB>(p, q4, x, bo);
        cols_compute<NB, Q, NC>(p, x, bo);
    }
}
template <int NB, int Q>
__global__ void __launch_bounds__(256, cols_minb(NB, Q)) ds_task_cols_kernel(const __grid_constant__ TaskParams p) {
    if (p.noclamp) cols_loop<NB, Q, true>(p);
    else cols_loop<NB, Q, false>(p);
}

using TaskFn = void (*)(const TaskParams);
template <int NB>
TaskFn cols_fn_q(int q) {
    switch (q) {
        case 1: return ds_task_cols_kernel<NB, 1>;
        case 2: return ds_task_cols_kernel<NB, 2>;
        case 3: return ds_task_cols_kernel<NB, 3>;
        case 4: return ds_task_cols_kernel<NB, 4>;
        case 5: return ds_task_cols_kernel<NB, 5>;
        case 6: return ds_task_cols_kernel<NB, 6>;
        case 7: return ds_task_cols_kernel<NB, 7>;
        default: return ds_task_cols_kernel<NB, 8>;
    }
}
TaskFn cols_fn(int ni, int no) {
    switch ((ni + 3) / 4) {
        case 1: return cols_fn_q<1>(no);
        case 2: return cols_fn_q<2>(no);
        case 3: return cols_fn_q<3>(no);
        default: return cols_fn_q<4>(no);
    }
}
template <int NI>
TaskFn dense_fn_q(int q) {
    switch (q) {
        case 1: return ds_task_dense_kernel<NI, 1>;
        case 2: return ds_task_dense_kernel<NI, 2>;
        case 3: return ds_task_dense_kernel<NI, 3>;
        case 4: return ds_task_dense_kernel<NI, 4>;
        case 5: return ds_task_dense_kernel<NI, 5>;
        case 6: return ds_task_dense_kernel<NI, 6>;
        case 7: return ds_task_dense_kernel<NI, 7>;
        default: return ds_task_dense_kernel<NI, 8>;
    }
}
TaskFn dense_fn(int ni, int no) {
    switch ((ni + 3) / 4) {
        case 1: return dense_fn_q<4>(no);
        case 2: return dense_fn_q<8>(no);
        case 3: return dense_fn_q<12>(no);
        default: return dense_fn_q<16>(no);
    }
}
template <int NI, bool WORDS>
TaskFn affine_fn_q(int q) {
    switch (q) {
        case 1: return ds_task_affine_kernel<NI, WORDS, 1>;
        case 2: return ds_task_affine_kernel<NI, WORDS, 2>;
        case 3: return ds_task_affine_kernel<NI, WORDS, 3>;
        case 4: return ds_task_affine_kernel<NI, WORDS, 4>;
        case 5: return ds_task_affine_kernel<NI, WORDS, 5>;
        case 6: return ds_task_affine_kernel<NI, WORDS, 6>;
        case 7: return ds_task_affine_kernel<NI, WORDS, 7>;
        default: return ds_task_affine_kernel<NI, WORDS, 8>;
    }
}
TaskFn affine_fn(int ni, bool words, int no) {
    switch ((ni + 3) / 4) {
        case 1: return words ? affine_fn_q<4, true>(no) : affine_fn_q<4, false>(no);
        case 2: return words ? affine_fn_q<8, true>(no) : affine_fn_q<8, false>(no);
        case 3: return words ? affine_fn_q<12, true>(no) : affine_fn_q<12, false>(no);
        default: return words ? affine_fn_q<16, true>(no) : affine_fn_q<16, false>(no);
    }
}

template <int NI>
__global__ void __launch_bounds__(256, 1) ds_task_kernel(const __grid_constant__ TaskParams p) {
    if (p.policy == DS_TOPO_SPEC) {
        // NDRange work-item = one elementary task; guarded padding
        const int64_t hw[3] = {(int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                               (int64_t)blockIdx.y * blockDim.y + threadIdx.y,
                               (int64_t)blockIdx.z * blockDim.z + threadIdx.z};
        int64_t q = 0;
        for (int d = 0; d < p.tdim; ++d) {
            const int64_t c = hw[p.tax[d]];
            if (c >= p.tmult[d]) return;                  // guard
            q = q * p.tmult[d] + c;
        }
        task_one<NI>(p, q);
        return;
    }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < p.n_reps; q += stride)
        task_one<NI>(p, q);
}

TaskFn modulo_fn(int ni) {
    switch ((ni + 3) / 4) {
        case 1: return ds_task_kernel<4>;
        case 2: return ds_task_kernel<8>;
        case 3: return ds_task_kernel<12>;
        default: return ds_task_kernel<16>;
    }
}

__global__ void __launch_bounds__(256) ds_cover_count_kernel(const __grid_constant__ TaskParams p,
                                                             uint32_t* count) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < p.n_reps; q += stride) {
        int64_t r[4] = {0, 0, 0, 0}, base[4];
        t_unravel(q, p.nrep, p.rep, r);
        t_base(p.tout, p.nrep, r, base);
        for (int k = 0; k < p.tout.npe; ++k) atomicAdd(count + t_lin(p.tout, base, k), 1u);
    }
}

__global__ void __launch_bounds__(256) ds_cover_reduce_kernel(const uint32_t* count, int64_t n,
                                                              unsigned long long* res) {
    unsigned long long over = 0, gap = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t c = count[i];
        over += c > 1;
        gap += c == 0;
    }
    for (int o = 16; o > 0; o >>= 1) {
        over += __shfl_xor_sync(0xffffffffu, over, o);
        gap += __shfl_xor_sync(0xffffffffu, gap, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (over) atomicAdd(res, over);
        if (gap) atomicAdd(res + 1, gap);
    }
}

int64_t h_mod(int64_t a, int64_t m) {
    const int64_t r = a % m;
    return r < 0 ? r + m : r;
}

int64_t pattern_elems(const ds_tiler& t) {
    int64_t n = 1;
    for (int k = 0; k < t.npat; ++k) n *= t.pattern[k];
    return n;
}

// Validate a tiler against the limits of include/ds.h and reduce it.
int prep_tiler(const ds_tiler& t, int32_t nrep, TTiler* o, int64_t* elems) {
    if (t.ndim < 1 || t.ndim > 4 || t.nrep != nrep || t.npat < 0 || t.npat > 4) return DS_EINVAL;
    const int64_t lim = 1LL << 40;
    int64_t n = 1;
    for (int d = 0; d < t.ndim; ++d) {
        if (t.shape[d] < 1) return DS_EINVAL;
        if (t.shape[d] > (1LL << 32) || n > (1LL << 32) / t.shape[d]) return DS_EUNSUPPORTED;
        n *= t.shape[d];
        if (t.origin[d] < -lim || t.origin[d] > lim) return DS_EUNSUPPORTED;
        for (int j = 0; j < nrep; ++j)
            if (t.paving[d][j] < -lim || t.paving[d][j] > lim) return DS_EUNSUPPORTED;
        for (int k = 0; k < t.npat; ++k)
            if (t.fitting[d][k] < -lim || t.fitting[d][k] > lim) return DS_EUNSUPPORTED;
    }
    for (int k = 0; k < t.npat; ++k)
        if (t.pattern[k] < 1) return DS_EINVAL;
    const int64_t npe = pattern_elems(t);
    if (npe > DS_MAX_PATTERN) return DS_EUNSUPPORTED;
    std::memset(o, 0, sizeof *o);
    o->ndim = t.ndim;
    o->npe = (int32_t)npe;
    int64_t st = 1;
    for (int d = t.ndim - 1; d >= 0; --d) {
        o->shape[d] = t.shape[d];
        o->stride[d] = st;
        st *= t.shape[d];
        o->origin[d] = h_mod(t.origin[d], t.shape[d]);
        for (int j = 0; j < nrep; ++j) o->pav[d][j] = h_mod(t.paving[d][j], t.shape[d]);
    }
    for (int64_t e = 0; e < npe; ++e) {
        int64_t f[4] = {0, 0, 0, 0}, rem = e;
        for (int k = t.npat - 1; k >= 0; --k) { f[k] = rem % t.pattern[k]; rem /= t.pattern[k]; }
        for (int d = 0; d < t.ndim; ++d) {
            int64_t v = 0;
            for (int k = 0; k < t.npat; ++k) v += h_mod(t.fitting[d][k], t.shape[d]) * f[k];
            o->foff[e][d] = h_mod(v, t.shape[d]);
        }
    }
    *elems = n;
    return DS_OK;
}

int prep_reps(int32_t nrep, const int64_t* rep, TaskParams* p) {
    if (nrep < 1 || nrep > 4 || !rep) return DS_EINVAL;
    int64_t n = 1;
    for (int j = 0; j < nrep; ++j) {
        if (rep[j] < 1) return DS_EINVAL;
        if (rep[j] >= (1LL << 31) || n > LLONG_MAX / rep[j]) return DS_EUNSUPPORTED;
        n *= rep[j];
        p->rep[j] = rep[j];
    }
    p->nrep = nrep;
    p->n_reps = n;
    return DS_OK;
}

FastDiv make_fdiv(int64_t d) {
    FastDiv f{(uint32_t)d, 0u, 0u};
    if (d > 1) {
        uint32_t l = 0;
        while ((1ULL << l) < (uint64_t)d) ++l;            // ceil(log2 d)
        const uint64_t pw = 31 + l;
        f.m = (uint32_t)(((1ULL << pw) + (uint64_t)d - 1) / (uint64_t)d);
        f.s = (uint32_t)(pw - 32);
    }
    return f;
}

// The 32-bit path applies when every quantity it forms stays below 2^31:
// reps, array extents, and origin + foff + sum_j pav[d][j] * (rep_j - 1).
bool fits32(const TaskParams& p, const TTiler& t) {
    const int64_t lim = (1LL << 31);
    for (int d = 0; d < t.ndim; ++d) {
        if (t.shape[d] >= lim) return false;
        int64_t foff_max = 0;
        for (int e = 0; e < t.npe; ++e) foff_max = std::max(foff_max, t.foff[e][d]);
        int64_t b = t.origin[d] + foff_max;
        for (int j = 0; j < p.nrep; ++j) b += t.pav[d][j] * (p.rep[j] - 1);
        if (b >= lim) return false;
    }
    int64_t n = 1;
    for (int d = 0; d < t.ndim; ++d) n *= t.shape[d];
    return n < lim;
}

// Affine analysis of a tiler over the repetition box (host).  Every origin /
// paving / fitting coefficient c may be replaced by any value congruent to it
// mod the extent s; for each array dim, search the two
// representatives c mod s and c mod s - s of every coefficient with a nonzero
// range for a choice under which origin + paving.r + fitting.f stays inside
// [0, s) over the whole box.  If every dim has one, no modulo ever applies and
// the row-major element offset is A + sum_j a[j] r_j + b[e].
bool affine_tiler(const ds_tiler& t, int32_t nrep, const int64_t* rep, uint32_t* A, uint32_t* a,
                  int32_t* b, int nb_max) {
    int64_t stride[4], st = 1;
    for (int d = t.ndim - 1; d >= 0; --d) { stride[d] = st; st *= t.shape[d]; }
    if (st >= (1LL << 31)) return false;
    const int64_t npe = pattern_elems(t);
    if (npe > nb_max) return false;
    int64_t A64 = 0, a64[4] = {0, 0, 0, 0};
    int64_t fit[4][4] = {};
    for (int d = 0; d < t.ndim; ++d) {
        const int64_t s = t.shape[d];
        const int64_t o = h_mod(t.origin[d], s);
        // coefficients (reps then pattern dims) and their index ranges
        int64_t c[8], n[8];
        int nc = 0;
        for (int j = 0; j < nrep; ++j) { c[nc] = h_mod(t.paving[d][j], s); n[nc++] = rep[j] - 1; }
        for (int k = 0; k < t.npat; ++k) { c[nc] = h_mod(t.fitting[d][k], s); n[nc++] = t.pattern[k] - 1; }
        bool found = false;
        int64_t best[8];
        for (uint32_t m = 0; m < (1u << nc) && !found; ++m) {
            int64_t lo = o, hi = o, v[8];
            bool skip = false;
            for (int i = 0; i < nc; ++i) {
                const bool neg = (m >> i) & 1u;
                if (neg && (c[i] == 0 || n[i] == 0)) { skip = true; break; }   // one choice suffices
                v[i] = neg ? c[i] - s : c[i];
                const int64_t ext = v[i] * n[i];
                (ext < 0 ? lo : hi) += ext;
            }
            if (skip || lo < 0 || hi >= s) continue;
            found = true;
            for (int i = 0; i < nc; ++i) best[i] = v[i];
        }
        if (!found) return false;
        A64 += o * stride[d];
        for (int j = 0; j < nrep; ++j) a64[j] += best[j] * stride[d];
        for (int k = 0; k < t.npat; ++k) fit[d][k] = best[nrep + k];
    }
    for (int64_t e = 0; e < npe; ++e) {
        int64_t f[4] = {0, 0, 0, 0}, rem = e;
        for (int k = t.npat - 1; k >= 0; --k) { f[k] = rem % t.pattern[k]; rem /= t.pattern[k]; }
        int64_t off = 0;
        for (int d = 0; d < t.ndim; ++d)
            for (int k = 0; k < t.npat; ++k) off += fit[d][k] * f[k] * stride[d];
        b[e] = (int32_t)off;
    }
    *A = (uint32_t)A64;
    for (int j = 0; j < 4; ++j) a[j] = (uint32_t)(j < nrep ? a64[j] : 0);
    return true;
}

int64_t next_pow2(int64_t x) {
    int64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

}  // namespace

namespace {

// Plan and launch one (validated) task.  With allow_peel, a task whose
// tilers are not wrap-free over the whole box is split when a thin slab at one
// end of one repetition dimension carries all the wrapping: the interior runs
// on the affine / dense / column paths, the slab (origin moved to its start)
// on the modulo path.  Output tilers are exact, so the parts write disjoint
// elements and the split changes nothing but speed.
int launch_task(const uint8_t* in, const ds_tiler& t_in, uint8_t* out, const ds_tiler& t_out, int32_t nrep,
                const int64_t* rep_shape, const ds_task_body* body, int32_t policy, cudaStream_t st, int sms,
                bool allow_peel) {
    TaskParams p;
    std::memset(&p, 0, sizeof p);
    int rc = prep_reps(nrep, rep_shape, &p);
    if (rc) return rc;
    int64_t nin = 0, nout = 0;
    if ((rc = prep_tiler(t_in, nrep, &p.tin, &nin))) return rc;
    if ((rc = prep_tiler(t_out, nrep, &p.tout, &nout))) return rc;
    p.in = in;
    p.out = out;
    p.policy = policy;
    p.fast32 = (p.n_reps < (1LL << 31) && fits32(p, p.tin) && fits32(p, p.tout)) ? 1 : 0;
    for (int j = 0; j < nrep; ++j) p.rdiv[j] = make_fdiv(p.rep[j]);
    for (int d = 0; d < p.tin.ndim; ++d) p.sdiv_in[d] = make_fdiv(p.tin.shape[d]);
    for (int d = 0; d < p.tout.ndim; ++d) p.sdiv_out[d] = make_fdiv(p.tout.shape[d]);
    p.n_in = body->n_in;
    p.n_out = body->n_out;
    p.divisor = body->divisor;
    p.bias = body->bias;
    for (int k = 0; k < p.n_out; ++k)              // taps past n_in (or n_out) are zero
        for (int e = 0; e < p.n_in; ++e) p.w[k][e] = body->weight[k][e];
    // taps: s8-packed copies, live pattern elements, and the exact
    // multiply-high division (same derivation as K-N1g's FASTDIV) -- all paths
    bool s8 = true;
    int64_t amax = 0, amin = 0;
    for (int k = 0; k < p.n_out; ++k) {
        int64_t pos = body->bias, neg = body->bias;
        for (int e = 0; e < p.n_in; ++e) {
            const int32_t w = body->weight[k][e];
            if (w < -128 || w > 127) s8 = false;
            if (w > 0) pos += 255LL * w;
            if (w < 0) neg += 255LL * w;
            if (w != 0) p.in_live |= 1u << e;
            p.wp[k][e / 4] |= (uint32_t)(uint8_t)(int8_t)(w < -128 || w > 127 ? 0 : w) << (8 * (e % 4));
        }
        amax = std::max(amax, pos);
        amin = k == 0 ? neg : std::min(amin, neg);
    }
    {
        const uint64_t D = (uint64_t)body->divisor;
        if (D == 1) {
            if (amax < 0x7fffffffLL) { p.fastdiv = 1; p.M = 0xffffffffu; p.lo = 1; p.fbias = body->bias + 1; }
        } else {
            const uint64_t M = ((1ULL << 32) + D - 1) / D, e = M * D - (1ULL << 32);
            if ((unsigned __int128)(uint64_t)amax * e < ((unsigned __int128)1 << 32)) {
                p.fastdiv = 1; p.M = (uint32_t)M; p.lo = 0; p.fbias = body->bias;
            }
        }
        // neither clamp can fire: acc (+1 when D == 1) >= lo and trunc(amax / D) <= 255
        p.noclamp = p.fastdiv && amin >= 0 && (uint64_t)amax / D <= 255;
    }
    // affine path: both tilers wrap-free, 32-bit offsets and repetition index
    if (p.n_reps < (1LL << 31) && affine_tiler(t_in, nrep, rep_shape, &p.in_A, p.in_a, p.in_b, DS_MAX_PATTERN) &&
        affine_tiler(t_out, nrep, rep_shape, &p.out_A, p.out_a, p.out_b, DS_MAX_OUTPUTS)) {
        p.affine = 1;
        bool words = s8 && p.n_in % 4 == 0;
        for (int j = 0; j < nrep; ++j) words = words && p.in_a[j] % 4 == 0;
        for (int e = 0; e < p.n_in; ++e) words = words && p.in_b[e] == e;
        if (words) {
            p.affine = 2;
            p.in_shift = (int32_t)((reinterpret_cast<uintptr_t>(in) + p.in_A) & 3);
        }
        // dense: both tilers are row-major runs over the repetition index
        bool dense = words && policy == DS_TOPO_FLAT &&
                     ((reinterpret_cast<uintptr_t>(in) + p.in_A) & 15) == 0 &&
                     ((reinterpret_cast<uintptr_t>(out) + p.out_A) & 3) == 0;
        int64_t inner = 1;
        for (int j = nrep - 1; j >= 0; --j) {
            dense = dense && p.in_a[j] == (uint64_t)(p.n_in * inner) && p.out_a[j] == (uint64_t)(p.n_out * inner);
            inner *= rep_shape[j];
        }
        for (int k = 0; k < p.n_out; ++k) dense = dense && p.out_b[k] == k;
        p.dense = dense ? 1 : 0;
        // column vectors: innermost repetition dim unit-stride in both arrays
        // (extent % 4 == 0), all other offsets and both pointers 4-aligned, s8 taps
        if (!dense && policy == DS_TOPO_FLAT && s8) {
            const int jl = nrep - 1;
            bool cols = p.in_a[jl] == 1 && p.out_a[jl] == 1 && rep_shape[jl] % 4 == 0 &&
                        p.in_A % 4 == 0 && p.out_A % 4 == 0 &&
                        (reinterpret_cast<uintptr_t>(in) & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 3) == 0;
            for (int j = 0; j < jl; ++j) cols = cols && p.in_a[j] % 4 == 0 && p.out_a[j] % 4 == 0;
            for (int e = 0; e < p.n_in; ++e) cols = cols && (p.in_b[e] & 3) == 0;
            for (int k = 0; k < p.n_out; ++k) cols = cols && (p.out_b[k] & 3) == 0;
            if (cols) p.affine = 3;
        }
        // loads of elements with no tap (dead, or past n_in) re-read the first
        // live element: unconditional loads, the zero taps ignore the value
        int first = 0;
        while (first < p.n_in - 1 && !((p.in_live >> first) & 1u)) ++first;
        for (int e = 0; e < DS_MAX_PATTERN; ++e)
            p.in_bl[e] = (e < p.n_in && ((p.in_live >> e) & 1u)) ? p.in_b[e] : p.in_b[first];
    }
    if (!p.affine && allow_peel && p.n_reps < (1LL << 31)) {
        // a wrap confined to <= 8 repetitions at one end of one repetition dim
        uint32_t A, a[4];
        int32_t bi[DS_MAX_PATTERN], bo[DS_MAX_OUTPUTS];
        auto shifted = [&](const ds_tiler& t, int j, int64_t by) {
            ds_tiler u = t;
            for (int d = 0; d < t.ndim; ++d)
                u.origin[d] = h_mod(h_mod(t.origin[d], t.shape[d]) + h_mod(t.paving[d][j], t.shape[d]) * by,
                                    t.shape[d]);
            return u;
        };
        for (int j = nrep - 1; j >= 0; --j) {
            const int64_t R = rep_shape[j];
            for (int64_t t : {1, 2, 3, 4, 8}) {
                if (t >= R) break;
                int64_t rin[4], rsl[4];
                for (int q = 0; q < nrep; ++q) rin[q] = rsl[q] = rep_shape[q];
                rin[j] = R - t;
                rsl[j] = t;
                // slab at the end: interior [0, R - t) keeps the tilers
                if (affine_tiler(t_in, nrep, rin, &A, a, bi, DS_MAX_PATTERN) &&
                    affine_tiler(t_out, nrep, rin, &A, a, bo, DS_MAX_OUTPUTS)) {
                    if ((rc = launch_task(in, t_in, out, t_out, nrep, rin, body, policy, st, sms, false))) return rc;
                    return launch_task(in, shifted(t_in, j, R - t), out, shifted(t_out, j, R - t), nrep, rsl, body,
                                       policy, st, sms, false);
                }
                // slab at the start: interior [t, R) has its origin moved by t
                const ds_tiler hin = shifted(t_in, j, t), hout = shifted(t_out, j, t);
                if (affine_tiler(hin, nrep, rin, &A, a, bi, DS_MAX_PATTERN) &&
                    affine_tiler(hout, nrep, rin, &A, a, bo, DS_MAX_OUTPUTS)) {
                    if ((rc = launch_task(in, hin, out, hout, nrep, rin, body, policy, st, sms, false))) return rc;
                    return launch_task(in, t_in, out, t_out, nrep, rsl, body, policy, st, sms, false);
                }
            }
        }
    }
    const TaskFn fn = p.dense ? dense_fn(p.n_in, p.n_out)
                      : p.affine == 3 ? cols_fn(p.n_in, p.n_out)
                      : p.affine ? affine_fn(p.n_in, p.affine == 2, p.n_out) : modulo_fn(p.n_in);
    if (policy == DS_TOPO_SPEC) {
        ds_topology topo;
        if ((rc = ds_compute_topology(nrep, rep_shape, 1024, 3, 64, 256, &topo))) return rc;
        p.tdim = topo.ndim;
        // CUDA limits: block (1024, 1024, 64), grid (2^31 - 1, 65535, 65535).
        // Each collapsed dim goes to its own axis; the preferred assignment
        // puts the last (fastest) dim on x, the first permutation of the
        // axes that fits both limits is launched.
        const int64_t blim[3] = {1024, 1024, 64}, glim[3] = {2147483647LL, 65535LL, 65535LL};
        static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
        bool placed = false;
        for (int pi = 0; pi < 6 && !placed; ++pi) {
            // perms[pi][k] = axis of the k-th dim counted from the last one
            bool fits = true;
            for (int k = 0; k < topo.ndim && fits; ++k) {
                const int d = topo.ndim - 1 - k, ax = perms[pi][k];
                if (topo.ndim < 3 && ax >= topo.ndim) fits = false;
                if (topo.local[d] > blim[ax] || topo.global[d] / topo.local[d] > glim[ax]) fits = false;
            }
            if (!fits) continue;
            dim3 block(1, 1, 1), grid(1, 1, 1);
            for (int k = 0; k < topo.ndim; ++k) {
                const int d = topo.ndim - 1 - k, ax = perms[pi][k];
                p.tmult[d] = topo.multiplicity[d];
                p.tax[d] = ax;
                (ax == 0 ? block.x : ax == 1 ? block.y : block.z) = (unsigned)topo.local[d];
                (ax == 0 ? grid.x : ax == 1 ? grid.y : grid.z) = (unsigned)(topo.global[d] / topo.local[d]);
            }
            fn<<<grid, block, 0, st>>>(p);
            placed = true;
        }
        if (!placed) return DS_EUNSUPPORTED;
    } else {
        const int64_t items = p.affine == 3 ? p.n_reps / 4 : p.n_reps;      // column quads
        const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, (int64_t)sms * 16));
        fn<<<(unsigned)blocks, 256, 0, st>>>(p);
    }
    return cudaGetLastError() == cudaSuccess ? DS_OK : DS_ECUDA;
}


}  // namespace

extern "C" {

DS_API int ds_compute_topology(int32_t nrep, const int64_t* mult, int32_t max_wg, int32_t max_dims,
                               int32_t min_items, int32_t wg_threshold, ds_topology* out) {
    if (!out || !mult || nrep < 1 || nrep > 4 || max_wg < 1 || max_dims < 1 || max_dims > 3 ||
        min_items < 0 || wg_threshold < 1)
        return DS_EINVAL;
    for (int j = 0; j < nrep; ++j)
        if (mult[j] < 1) return DS_EINVAL;
    ds_topology t;
    std::memset(&t, 0, sizeof t);
    // (1) collapse dimensions beyond max_dims by multiplying trailing extents
    t.ndim = std::min(nrep, max_dims);
    for (int d = 0; d < t.ndim; ++d) t.multiplicity[d] = mult[d];
    for (int j = t.ndim; j < nrep; ++j) t.multiplicity[t.ndim - 1] *= mult[j];
    int64_t total = 1;
    for (int d = 0; d < t.ndim; ++d) total *= t.multiplicity[d];
    const int64_t cap_raw = std::min<int64_t>(max_wg, wg_threshold);
    int64_t cap = 1;
    while (cap * 2 <= cap_raw) cap *= 2;
    if (total < min_items && total <= cap_raw) {
        // (2) small multiplicity: one work-group sized to it
        for (int d = 0; d < t.ndim; ++d) {
            t.local[d] = (int32_t)t.multiplicity[d];
            t.global[d] = t.multiplicity[d];
        }
        t.guarded = 0;
        *out = t;
        return DS_OK;
    }
    // (3) power-of-two box, round-robin from the largest dimension, keeping
    // the padded size < 2 x multiplicity (the padding bound of S:651)
    int order[3] = {0, 1, 2};
    std::stable_sort(order, order + t.ndim,
                     [&](int a, int b) { return t.multiplicity[a] > t.multiplicity[b]; });
    int64_t loc[3] = {1, 1, 1};
    bool frozen[3] = {false, false, false};
    int64_t prod = 1;
    bool progress = true;
    while (progress && prod * 2 <= cap) {
        progress = false;
        for (int oi = 0; oi < t.ndim && prod * 2 <= cap; ++oi) {
            const int d = order[oi];
            if (frozen[d]) continue;
            const int64_t cand = loc[d] * 2;
            if (cand > next_pow2(t.multiplicity[d])) { frozen[d] = true; continue; }
            int64_t padded = 1;
            for (int e = 0; e < t.ndim; ++e) {
                const int64_t l = e == d ? cand : loc[e];
                padded *= (t.multiplicity[e] + l - 1) / l * l;
            }
            if (padded >= 2 * total) { frozen[d] = true; continue; }
            loc[d] = cand;
            prod *= 2;
            progress = true;
        }
    }
    // (4) global = smallest multiple of local >= multiplicity
    t.guarded = 0;
    for (int d = 0; d < t.ndim; ++d) {
        t.local[d] = (int32_t)loc[d];
        t.global[d] = (t.multiplicity[d] + loc[d] - 1) / loc[d] * loc[d];
        if (t.global[d] != t.multiplicity[d]) t.guarded = 1;
    }
    *out = t;
    return DS_OK;
}

DS_API int ds_run_task(const uint8_t* in, const ds_tiler* t_in, uint8_t* out, const ds_tiler* t_out,
                       int32_t nrep, const int64_t* rep_shape, const ds_task_body* body,
                       int32_t policy, ds_stream_t stream) {
    if (!in || !out || !t_in || !t_out || !body) return DS_EINVAL;
    if (policy != DS_TOPO_FLAT && policy != DS_TOPO_SPEC) return DS_EINVAL;
    TaskParams p;
    std::memset(&p, 0, sizeof p);
    int rc = prep_reps(nrep, rep_shape, &p);
    if (rc) return rc;
    int64_t nin = 0, nout = 0;
    if ((rc = prep_tiler(*t_in, nrep, &p.tin, &nin))) return rc;
    if ((rc = prep_tiler(*t_out, nrep, &p.tout, &nout))) return rc;
    if (body->n_in != p.tin.npe || body->n_out != p.tout.npe || body->n_out > DS_MAX_OUTPUTS ||
        body->divisor < 1)
        return DS_EINVAL;
    if (body->divisor > (1 << 24) || body->bias < -(1 << 24) || body->bias > (1 << 24))
        return DS_EUNSUPPORTED;
    for (int k = 0; k < DS_MAX_OUTPUTS; ++k)
        for (int i = 0; i < DS_MAX_PATTERN; ++i)
            if (body->weight[k][i] < -65535 || body->weight[k][i] > 65535) return DS_EUNSUPPORTED;
    if (dsi::ranges_overlap(in, nin, out, nout)) return DS_EINVAL;
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
        cudaGetLastError();
        return DS_ECUDA;
    }
    if (!dsi::device_ptr_on(in, dev) || !dsi::device_ptr_on(out, dev)) return DS_EINVAL;
    return launch_task(in, *t_in, out, *t_out, nrep, rep_shape, body, policy,
                       reinterpret_cast<cudaStream_t>(stream), sms, policy == DS_TOPO_FLAT);
}

DS_API int ds_tiler_coverage(const ds_tiler* t, int32_t nrep, const int64_t* rep_shape, int64_t* overlaps,
                             int64_t* gaps, ds_stream_t stream) {
    if (!t || !overlaps || !gaps) return DS_EINVAL;
    TaskParams p;
    std::memset(&p, 0, sizeof p);
    int rc = prep_reps(nrep, rep_shape, &p);
    if (rc) return rc;
    int64_t n = 0;
    if ((rc = prep_tiler(*t, nrep, &p.tout, &n))) return rc;
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
        cudaGetLastError();
        return DS_ECUDA;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    uint32_t* count = nullptr;
    unsigned long long* res = nullptr;
    if (cudaMallocAsync(&count, (size_t)n * 4, st) != cudaSuccess ||
        cudaMallocAsync(&res, 16, st) != cudaSuccess) {
        cudaGetLastError();
        if (count) cudaFreeAsync(count, st);
        return DS_ENOMEM;
    }
    cudaMemsetAsync(count, 0, (size_t)n * 4, st);
    cudaMemsetAsync(res, 0, 16, st);
    const int64_t b1 = std::max<int64_t>(1, std::min<int64_t>((p.n_reps + 255) / 256, (int64_t)sms * 16));
    ds_cover_count_kernel<<<(unsigned)b1, 256, 0, st>>>(p, count);
    const int64_t b2 = std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms * 16));
    ds_cover_reduce_kernel<<<(unsigned)b2, 256, 0, st>>>(count, n, res);
    unsigned long long h[2] = {0, 0};
    cudaMemcpyAsync(h, res, 16, cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(count, st);
    cudaFreeAsync(res, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) {
        cudaGetLastError();
        return DS_ECUDA;
    }
    *overlaps = (int64_t)h[0];
    *gaps = (int64_t)h[1];
    return DS_OK;
}

}  // extern "C"
