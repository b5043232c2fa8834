// ds_tasks.cuh -- K-N3: the paper's unfused structure on sm_100a.
//
// PAPER sec. 3.1: "the six repetitive tasks in horizontal and vertical
// filters are allocated onto the GPU in order to generate kernels" -- one
// kernel per task, the intermediate array (the H task's output) held
// in global memory between them.  Here that structure is kept as an A/B
// baseline for the fused kernel and as the device side of the transfer
// schedules of S:369-387 (ds_run_schedule):
//
//   ds_htask_kernel   H task, SPEC taps: the input stream is a flat array of
//                     8-byte packets (W % 8 == 0), packet p -> Mid bytes
//                     3p..3p+2 (the H output tiler is exact), so
//                     any contiguous byte range of frames/planes maps to the
//                     Mid range at 3/8 of its offset.  16-byte loads, warp
//                     repack through shared memory into 16-byte stores.
//   ds_vtask_kernel   V task, SPEC taps: item = (frame, plane, 9-row group,
//                     4 Mid columns) in one flat 32-bit item space; 8 LDG.32
//                     per item (row 4 has zero weight), 4 STG.32, two items
//                     per thread step with all loads issued first.
//   ds_htask_generic / ds_vtask_generic: any ds_stage_spec, one thread per
//                     output element, literal tiler indexing.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ds.h"
#include "ds_pipeline.cuh"

namespace ds {

struct TaskPlanes {
    int64_t in_frame, mid_frame, out_frame;
    int64_t in_off[DS_MAX_PLANES], mid_off[DS_MAX_PLANES], out_off[DS_MAX_PLANES];
    int32_t W[DS_MAX_PLANES], H[DS_MAX_PLANES], Wm[DS_MAX_PLANES], Hout[DS_MAX_PLANES];
    int32_t plane_first, plane_count;
    int64_t n_frames;
};

// ------------------------------------------------------------ H task, SPEC --
__device__ __forceinline__ uint32_t t_div6(uint32_t x) { return __umulhi(x, 0x2AAAAAABu); }

// 16 input bytes (two packets) -> 6 mid bytes, returned as lo (4 bytes) + hi (2 bytes)
__device__ __forceinline__ void t_hchunk(uint4 v, uint32_t& lo, uint32_t& hi) {
    const uint32_t tA = __byte_perm(v.x, v.y, 0x7643);
    const uint32_t tB = __byte_perm(v.z, v.w, 0x7643);
    const uint32_t a0 = t_div6(__dp4a(v.x, 0x0501u, 3u));
    const uint32_t a1 = __dp4a(tA, 0x0101u, 1u) >> 1;
    const uint32_t a2 = t_div6(__dp4a(tA, 0x01050000u, 3u));
    const uint32_t b0 = t_div6(__dp4a(v.z, 0x0501u, 3u));
    const uint32_t b1 = __dp4a(tB, 0x0101u, 1u) >> 1;
    const uint32_t b2 = t_div6(__dp4a(tB, 0x01050000u, 3u));
    lo = a0 | (a1 << 8) | (a2 << 16) | (b0 << 24);
    hi = b1 | (b2 << 8);
}

// n_chunks 16-byte input chunks at `in` (16-byte aligned) -> 6 * n_chunks
// bytes at `mid` (2-byte aligned; kVec: 16-byte aligned).
template <bool kVec>
__global__ void __launch_bounds__(256)
    ds_htask_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ mid, int64_t n_chunks) {
    __shared__ __align__(16) uint8_t stage[8][192];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + w * 32; base < n_chunks;
         base += stride) {
        const int64_t c = base + lane;
        const int64_t valid = n_chunks - base < 32 ? n_chunks - base : 32;
        uint32_t lo = 0, hi = 0;
        if (c < n_chunks) {
            const uint4 v = __ldcs(reinterpret_cast<const uint4*>(in) + c);
            t_hchunk(v, lo, hi);
        }
        if (kVec && valid == 32) {
            uint8_t* s = stage[w] + 6 * lane;
            *reinterpret_cast<uint16_t*>(s) = (uint16_t)lo;
            *reinterpret_cast<uint16_t*>(s + 2) = (uint16_t)(lo >> 16);
            *reinterpret_cast<uint16_t*>(s + 4) = (uint16_t)hi;
            __syncwarp();
            if (lane < 12)
                __stcs(reinterpret_cast<uint4*>(mid + 6 * base) + lane,
                       *reinterpret_cast<const uint4*>(stage[w] + 16 * lane));
            __syncwarp();
        } else if (c < n_chunks) {
            uint16_t* d = reinterpret_cast<uint16_t*>(mid + 6 * c);
            d[0] = (uint16_t)lo;
            d[1] = (uint16_t)(lo >> 16);
            d[2] = (uint16_t)hi;
        }
    }
}

// H task on the TMA pipeline (the K-N1 building blocks without the V step):
// a persistent grid streams units of `unit_in` bytes of the flat packet
// stream (a multiple of 128) through a ring of bulk copies; consumers turn
// 16-byte chunks into 6 Mid bytes in a shared output slot, which thread 0
// bulk-stores to Mid at 3/8 of the unit's offset (16-byte aligned).  The last
// unit may be short; a non-16-multiple output tail is stored cooperatively.
template <int NCW>
__global__ void __launch_bounds__((NCW + 1) * 32, 1)
    ds_htask_tma_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ mid, int64_t n_bytes,
                        int32_t unit_in, int32_t stages) {
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int NC = NCW * 32;
    const int S = stages;
    const int out_stride = (unit_in / 8 * 3 + 127) & ~127;
    uint8_t* ring = smem;
    uint8_t* outs = smem + (size_t)S * unit_in;
    uint64_t* full = reinterpret_cast<uint64_t*>(outs + (size_t)3 * out_stride);
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
    const int64_t n_units = (n_bytes + unit_in - 1) / unit_in;
    const int warp = tid >> 5, lane = tid & 31;
    int s = 0;
    uint32_t phase = 0;
    if (warp == NCW) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            bool first_round = true;
            for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
                if (!first_round) mbar_wait_sleep(&empty[s], phase ^ 1);
                const uint32_t bytes = (uint32_t)min((int64_t)unit_in, n_bytes - u * unit_in);
                mbar_arrive_expect_tx(&full[s], bytes);
                bulk_g2s(ring + (size_t)s * unit_in, in + u * unit_in, bytes, &full[s], pol);
                if (++s == S) { s = 0; phase ^= 1; first_round = false; }
            }
        }
        return;
    }
    int oslot = 0;
    for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
        const int bytes = (int)min((int64_t)unit_in, n_bytes - u * unit_in);
        const int chunks = bytes >> 4;
        const uint8_t* st = ring + (size_t)s * unit_in;
        uint8_t* ob = outs + (size_t)oslot * out_stride;
        mbar_wait(&full[s], phase);
        for (int c = tid; c < chunks; c += NC) {
            uint32_t lo, hi;
            t_hchunk(lds128(st + 16 * c), lo, hi);
            uint8_t* d = ob + 6 * c;
            sts16(d, lo);
            sts16(d + 2, lo >> 16);
            sts16(d + 4, hi);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        const int out_bytes = 6 * chunks;
        uint8_t* dst = mid + u * (unit_in / 8 * 3);
        if ((out_bytes & 15) == 0) {
            fence_proxy_async_smem();
            named_bar_sync(1, NC);
            if (tid == 0) {
                bulk_s2g_hint(dst, ob, (uint32_t)out_bytes, policy_evict_first());
                bulk_commit();
                bulk_wait_read<1>();
            }
        } else {
            named_bar_sync(1, NC);
            for (int x = tid; x < out_bytes; x += NC) dst[x] = ob[x];
        }
        if (++s == S) { s = 0; phase ^= 1; }
        oslot = oslot == 2 ? 0 : oslot + 1;
    }
    if (tid == 0) bulk_wait_all();
}

// ------------------------------------------------------------ V task, SPEC --
// Four mid columns per thread; rows 9g + {0,1,2,3,5,6,7,8}.
__device__ __forceinline__ uint32_t t_vquad(uint32_t a, uint32_t b, uint32_t wa, uint32_t wb) {
    // bytes -> two 16-bit-lane pairs, V on both, quotients are byte 1 of each lane
    const uint32_t a_lo = __byte_perm(a, 0, 0x4140), a_hi = __byte_perm(a, 0, 0x4342);
    const uint32_t b_lo = __byte_perm(b, 0, 0x4140), b_hi = __byte_perm(b, 0, 0x4342);
    const uint32_t s_lo = a_lo * wa + b_lo * wb + 0x00800080u;
    const uint32_t s_hi = a_hi * wa + b_hi * wb + 0x00800080u;
    return __byte_perm(s_lo, s_hi, 0x7531);
}

// n / d for 0 <= n < 2^31 by multiply-high (host: m = ceil(2^(31+l) / d),
// l = ceil(log2 d), s = l - 1; d = 1: m = 0 marks the identity)
struct TDiv {
    uint32_t d, m, s;
};
__device__ __forceinline__ uint32_t t_fdiv(const TDiv& f, uint32_t n) {
    return f.m == 0 ? n : (__umulhi(n, f.m) >> f.s);
}

// Flat V-task item space over a block of frames: item = ((f * per_frame) +
// plane start + g * quads + q), all < 2^31 (the host splits longer streams).
struct VFlat {
    uint32_t per_frame;                 // sum over the planes of quads * groups
    TDiv fdiv;                          // / per_frame
    uint32_t pstart[DS_MAX_PLANES];     // first item of each plane within a frame
    TDiv qdiv[DS_MAX_PLANES];           // / quads of each plane
    int32_t planes;
};

// item -> (column pointer into Mid, output pointer, row stride in VEC-byte words)
template <typename VEC>
__device__ __forceinline__ void t_vitem(const uint8_t* __restrict__ mid, uint8_t* __restrict__ out,
                                        const TaskPlanes& tp, const VFlat& vf, int64_t f0, uint32_t it,
                                        const VEC*& col, VEC*& o, int& wq) {
    const uint32_t f = t_fdiv(vf.fdiv, it);
    uint32_t r = it - f * vf.per_frame;
    const int pl = (vf.planes > 2 && r >= vf.pstart[2]) ? 2 : (vf.planes > 1 && r >= vf.pstart[1]) ? 1 : 0;
    r -= vf.pstart[pl];
    const uint32_t g = t_fdiv(vf.qdiv[pl], r);
    const uint32_t q = r - g * vf.qdiv[pl].d;
    const int p = tp.plane_first + pl;
    const int64_t fr = f0 + f;
    wq = tp.Wm[p] / (int)sizeof(VEC);
    col = reinterpret_cast<const VEC*>(mid + fr * tp.mid_frame + tp.mid_off[p] + (int64_t)9 * g * tp.Wm[p]) + q;
    o = reinterpret_cast<VEC*>(out + fr * tp.out_frame + tp.out_off[p] + (int64_t)4 * g * tp.Wm[p]) + q;
}

__device__ __forceinline__ uint32_t t_vq(uint32_t a, uint32_t b, uint32_t wa, uint32_t wb) {
    return t_vquad(a, b, wa, wb);
}
__device__ __forceinline__ uint2 t_vq(uint2 a, uint2 b, uint32_t wa, uint32_t wb) {
    return make_uint2(t_vquad(a.x, b.x, wa, wb), t_vquad(a.y, b.y, wa, wb));
}

// V task, SPEC taps: item = (frame, plane, 9-row group g, sizeof(VEC) Mid
// columns q); 8 row loads per item (row 4 has zero weight), 4 row stores.
// Each thread takes two items per step (it, it + stride) and issues all 16
// loads first.
template <typename VEC>
__global__ void __launch_bounds__(256)
    ds_vtask_kernel(const uint8_t* __restrict__ mid, uint8_t* __restrict__ out,
                    const __grid_constant__ TaskPlanes tp, const __grid_constant__ VFlat vf, int64_t f0,
                    uint32_t items) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t it = blockIdx.x * blockDim.x + threadIdx.x; it < items; it += 2 * stride) {
        const VEC* ca;
        VEC* oa;
        int wa;
        t_vitem<VEC>(mid, out, tp, vf, f0, it, ca, oa, wa);
        const bool two = it + stride < items;
        const VEC* cb = ca;
        VEC* ob = oa;
        int wb = wa;
        if (two) t_vitem<VEC>(mid, out, tp, vf, f0, it + stride, cb, ob, wb);
        const VEC a0 = __ldcs(ca), a1 = __ldcs(ca + wa), a2 = __ldcs(ca + 2 * wa), a3 = __ldcs(ca + 3 * wa),
                  a5 = __ldcs(ca + 5 * wa), a6 = __ldcs(ca + 6 * wa), a7 = __ldcs(ca + 7 * wa),
                  a8 = __ldcs(ca + 8 * wa);
        VEC b0{}, b1{}, b2{}, b3{}, b5{}, b6{}, b7{}, b8{};
        if (two) {
            b0 = __ldcs(cb); b1 = __ldcs(cb + wb); b2 = __ldcs(cb + 2 * wb); b3 = __ldcs(cb + 3 * wb);
            b5 = __ldcs(cb + 5 * wb); b6 = __ldcs(cb + 6 * wb); b7 = __ldcs(cb + 7 * wb); b8 = __ldcs(cb + 8 * wb);
        }
        __stcs(oa, t_vq(a0, a1, 96u, 160u));
        __stcs(oa + wa, t_vq(a2, a3, 32u, 224u));
        __stcs(oa + 2 * wa, t_vq(a5, a6, 224u, 32u));
        __stcs(oa + 3 * wa, t_vq(a7, a8, 160u, 96u));
        if (two) {
            __stcs(ob, t_vq(b0, b1, 96u, 160u));
            __stcs(ob + wb, t_vq(b2, b3, 32u, 224u));
            __stcs(ob + 2 * wb, t_vq(b5, b6, 224u, 32u));
            __stcs(ob + 3 * wb, t_vq(b7, b8, 160u, 96u));
        }
    }
}

// --------------------------------------------------------- generic task kernels --
__device__ __forceinline__ int32_t t_mod(int32_t a, int32_t m) {
    int32_t r = a % m;
    return r < 0 ? r + m : r;
}
__device__ __forceinline__ int32_t t_clamp(int32_t v) { return v < 0 ? 0 : (v > 255 ? 255 : v); }

struct GenericTask {
    TaskPlanes tp;
    ds_stage_spec s;
};

// H task, any spec: Mid[row][Qh r1 + j] = stage_h(In[row][(oh + Sh r1 + i) mod W]).
__global__ void __launch_bounds__(256) ds_htask_generic(const uint8_t* __restrict__ in,
                                                        uint8_t* __restrict__ mid,
                                                        const __grid_constant__ GenericTask gt) {
    const TaskPlanes& tp = gt.tp;
    const ds_stage_spec& s = gt.s;
    const int p = tp.plane_first + blockIdx.y;
    const int64_t items = (int64_t)tp.H[p] * tp.Wm[p];
    for (int64_t f = blockIdx.z; f < tp.n_frames; f += gridDim.z) {
        const uint8_t* ip = in + f * tp.in_frame + tp.in_off[p];
        uint8_t* mp = mid + f * tp.mid_frame + tp.mid_off[p];
        for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < items;
             it += (int64_t)gridDim.x * blockDim.x) {
            const int row = (int)(it / tp.Wm[p]), col = (int)(it - (int64_t)row * tp.Wm[p]);
            const int r1 = col / s.outputs, j = col - r1 * s.outputs;
            int32_t acc = s.bias;
            for (int i = 0; i < s.pattern; ++i) {
                const int32_t w = s.weight[j][i];
                if (w) acc += w * (int32_t)__ldg(ip + (int64_t)row * tp.W[p] +
                                                  t_mod(s.origin + s.paving * r1 + i, tp.W[p]));
            }
            mp[it] = (uint8_t)t_clamp(acc / s.divisor);
        }
    }
}

// V task, any spec: Out[Qv r0 + k][c] = stage_v(Mid[(ov + Sv r0 + i) mod H][c]).
__global__ void __launch_bounds__(256) ds_vtask_generic(const uint8_t* __restrict__ mid,
                                                        uint8_t* __restrict__ out,
                                                        const __grid_constant__ GenericTask gt) {
    const TaskPlanes& tp = gt.tp;
    const ds_stage_spec& s = gt.s;
    const int p = tp.plane_first + blockIdx.y;
    const int64_t items = (int64_t)tp.Hout[p] * tp.Wm[p];
    for (int64_t f = blockIdx.z; f < tp.n_frames; f += gridDim.z) {
        const uint8_t* mp = mid + f * tp.mid_frame + tp.mid_off[p];
        uint8_t* op = out + f * tp.out_frame + tp.out_off[p];
        for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < items;
             it += (int64_t)gridDim.x * blockDim.x) {
            const int R = (int)(it / tp.Wm[p]), col = (int)(it - (int64_t)R * tp.Wm[p]);
            const int r0 = R / s.outputs, k = R - r0 * s.outputs;
            int32_t acc = s.bias;
            for (int i = 0; i < s.pattern; ++i) {
                const int32_t w = s.weight[k][i];
                if (w) acc += w * (int32_t)__ldg(mp + (int64_t)t_mod(s.origin + s.paving * r0 + i,
                                                                      tp.H[p]) * tp.Wm[p] + col);
            }
            op[it] = (uint8_t)t_clamp(acc / s.divisor);
        }
    }
}

}  // namespace ds
