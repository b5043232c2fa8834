// bw_probe.cu -- HBM ceilings on this B200 for the traffic mixes of the
// downscaler.  Standalone, not part of libds.so.
//   read      : LDG.128 stream, XOR-reduced (read-only)
//   copy      : 1:1 LDG.128 -> STG.128
//   r6w1      : 6 bytes read per byte written (the HD 4:2:0 mix: 2,764,800
//               live input bytes vs 518,400 output bytes per frame ~ 5.3:1)
//   tma_read  : 1-D cp.async.bulk ring into shared memory, nothing computed
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/bw_probe.cu -o bw_probe
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void k_read(const uint4* __restrict__ in, size_t n, uint32_t* out) {
    uint32_t acc = 0;
    size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
        uint4 a = __ldcs(in + i), b = __ldcs(in + i + stride), c = __ldcs(in + i + 2 * stride),
              d = __ldcs(in + i + 3 * stride);
        acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
    }
    for (; i < n; i += stride) { uint4 a = __ldcs(in + i); acc ^= a.x ^ a.y ^ a.z ^ a.w; }
    if (acc == 0x12345678u) out[0] = acc;
}

__global__ void k_copy(const uint4* __restrict__ in, uint4* __restrict__ out, size_t n) {
    size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + stride < n; i += 2 * stride) {
        uint4 a = __ldcs(in + i), b = __ldcs(in + i + stride);
        __stcs(out + i, a); __stcs(out + i + stride, b);
    }
    for (; i < n; i += stride) __stcs(out + i, __ldcs(in + i));
}

// each thread reads 6 consecutive uint4 groups (strided by `stride` vectors) and writes 1
__global__ void k_r6w1(const uint4* __restrict__ in, uint4* __restrict__ out, size_t n_out) {
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_out; i += stride) {
        size_t base = (i / blockDim.x) * blockDim.x * 6 + (i % blockDim.x);
        uint4 r = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            uint4 a = __ldcs(in + base + (size_t)j * blockDim.x);
            r.x ^= a.x; r.y ^= a.y; r.z ^= a.z; r.w ^= a.w;
        }
        __stcs(out + i, r);
    }
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// persistent ring: one lane issues bulk copies of `chunk` bytes, the rest of
// the warp waits on the mbarrier then releases the slot (no compute)
__global__ void k_tma_read(const uint8_t* in, size_t n_chunks, uint32_t chunk, int stages) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * chunk);
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    size_t i = 0;
    size_t issued = 0;
    size_t my = 0;
    for (size_t c = blockIdx.x; c < n_chunks; c += gridDim.x) ++my;
    size_t c_issue = blockIdx.x;
    // prologue
    for (; issued < my && issued < (size_t)stages; ++issued, c_issue += gridDim.x) {
        int s = issued % stages;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(chunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(smem + (size_t)s * chunk)), "l"(in + c_issue * chunk), "r"(chunk), "r"(su32(&full[s])) : "memory");
    }
    for (; i < my; ++i) {
        int s = i % stages;
        uint32_t ph = (i / stages) & 1;
        asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}"
                     ::"r"(su32(&full[s])), "r"(ph) : "memory");
        if (issued < my) {
            int s2 = issued % stages;   // == s
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s2])), "r"(chunk) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su32(smem + (size_t)s2 * chunk)), "l"(in + c_issue * chunk), "r"(chunk), "r"(su32(&full[s2])) : "memory");
            ++issued; c_issue += gridDim.x;
        }
    }
}

// TMA ring that also writes: after each chunk lands, bulk-store `wbytes`
// of it to `out` (the downscaler's 5.33:1 read:write mix with wbytes = chunk*3/16)
__global__ void k_tma_rw(const uint8_t* in, uint8_t* out, size_t n_chunks, uint32_t chunk,
                         uint32_t wbytes, int stages) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * chunk);
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    size_t my = 0;
    for (size_t c = blockIdx.x; c < n_chunks; c += gridDim.x) ++my;
    size_t issued = 0, c_issue = blockIdx.x, c_done = blockIdx.x;
    for (; issued < my && issued < (size_t)stages; ++issued, c_issue += gridDim.x) {
        int s = issued % stages;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(chunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(smem + (size_t)s * chunk)), "l"(in + c_issue * chunk), "r"(chunk), "r"(su32(&full[s])) : "memory");
    }
    for (size_t i = 0; i < my; ++i, c_done += gridDim.x) {
        int s = i % stages;
        uint32_t ph = (i / stages) & 1;
        asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}"
                     ::"r"(su32(&full[s])), "r"(ph) : "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + c_done * wbytes),
                     "r"(su32(smem + (size_t)s * chunk)), "r"(wbytes) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        if (issued < my) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(chunk) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su32(smem + (size_t)s * chunk)), "l"(in + c_issue * chunk), "r"(chunk), "r"(su32(&full[s])) : "memory");
            ++issued; c_issue += gridDim.x;
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <class F>
float best_ms(F f, int reps = 10) {
    cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    f(); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
        float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
    }
    return best;
}

int main() {
    const size_t bytes = 2ull << 30;   // 2 GiB source
    uint8_t *in, *out; uint32_t* sink;
    CK(cudaMalloc(&in, bytes)); CK(cudaMalloc(&out, bytes)); CK(cudaMalloc(&sink, 64));
    CK(cudaMemset(in, 1, bytes)); CK(cudaMemset(out, 0, bytes));
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t nv = bytes / 16;
    for (int bpsm : {4, 8}) {
        int grid = sms * bpsm;
        float t = best_ms([&] { k_read<<<grid, 256>>>((const uint4*)in, nv, sink); });
        printf("read     grid=%5d : %7.1f GB/s\n", grid, bytes / t / 1e6);
        t = best_ms([&] { k_copy<<<grid, 256>>>((const uint4*)in, (uint4*)out, nv / 2); });
        printf("copy     grid=%5d : %7.1f GB/s (read+write)\n", grid, bytes / t / 1e6);
        size_t nout = nv / 7;
        nout = nout / 256 * 256;
        t = best_ms([&] { k_r6w1<<<grid, 256>>>((const uint4*)in, (uint4*)out, nout); });
        printf("r6w1     grid=%5d : %7.1f GB/s (read+write)\n", grid, nout * 16.0 * 7 / t / 1e6);
    }
    for (uint32_t chunk : {15360u, 30720u}) for (int stages : {2, 4, 6}) for (int cps : {1, 2}) {
        size_t smem = (size_t)stages * chunk + 64;
        if (smem * cps > 225 * 1024) continue;
        CK(cudaFuncSetAttribute(k_tma_read, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        size_t nch = bytes / chunk;
        int grid = sms * cps;
        float t = best_ms([&] { k_tma_read<<<grid, 32, smem>>>(in, nch, chunk, stages); });
        printf("tma_read chunk=%5u stages=%d ctas/sm=%d : %7.1f GB/s (%.0f KB in flight/SM)\n", chunk, stages, cps,
               nch * (double)chunk / t / 1e6, stages * cps * chunk / 1024.0);
    }
    for (uint32_t chunk : {15360u, 30720u}) for (int stages : {3, 4, 5}) {
        size_t smem = (size_t)stages * chunk + 64;
        CK(cudaFuncSetAttribute(k_tma_rw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        size_t nch = bytes / chunk;
        uint32_t wb = chunk * 3 / 16;          // 30720 -> 5760 (the HD unit's output band)
        int grid = sms;
        float t = best_ms([&] { k_tma_rw<<<grid, 32, smem>>>(in, out, nch, chunk, wb, stages); });
        printf("tma_rw   chunk=%5u out=%5u stages=%d ctas/sm=1 : %7.1f GB/s (read+write)\n", chunk, wb, stages,
               nch * (double)(chunk + wb) / t / 1e6);
    }
    return 0;
}
