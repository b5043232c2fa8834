// ds_sched.cu -- the paper's unfused task structure (K-N3) and its host <->
// device transfer schedules.  Citations: P:n = PAPER.md line
// n, S:n = SPEC.md line n.
//
// ds_run_htask / ds_run_vtask launch one repetitive task over a plane range
// (one kernel per task; "six repetitive tasks").  ds_run_schedule runs
// a host-resident stream frame by frame under one of
//   NAIVE      S:369-377: before every launch an H2D of the task's input
//              array, after it a D2H of its output array -> 12 transfers per
//              frame (the paper's "not optimized program");
//   OPTIMIZED  S:379-387: residency-aware, the intermediates stay on the
//              device -> 3 H2D + 3 D2H per frame (the paper's "performance
//              tuning");
//   FUSED      the same per-frame host loop with one H2D, one K-N1 launch and
//              one D2H per frame;
//   STREAMED   ds_run_host: chunked, three overlapped streams;
// and times every step on the device with CUDA events (the paper's "Time
// Distribution on the GPU").
#include <algorithm>
#include <cstring>

#include "ds.h"
#include "ds_internal.h"
#include "ds_tasks.cuh"

using namespace dsi;

namespace {

int64_t mid_frame_bytes(const ds_handle* h) {
    int64_t b = 0;
    for (int p = 0; p < h->plan.n_planes; ++p) b += (int64_t)h->plan.in_h[p] * h->plan.out_w[p];
    return b;
}

ds::TaskPlanes task_planes(const ds_handle* h, int64_t n, int p0, int pc) {
    ds::TaskPlanes tp;
    std::memset(&tp, 0, sizeof tp);
    const ds_plan_info& pi = h->plan;
    tp.in_frame = pi.in_frame_bytes;
    tp.out_frame = pi.out_frame_bytes;
    tp.mid_frame = mid_frame_bytes(h);
    int64_t moff = 0;
    for (int p = 0; p < pi.n_planes; ++p) {
        tp.in_off[p] = pi.in_offset[p];
        tp.out_off[p] = pi.out_offset[p];
        tp.mid_off[p] = moff;
        tp.W[p] = pi.in_w[p];
        tp.H[p] = pi.in_h[p];
        tp.Wm[p] = pi.out_w[p];          // Mid width = Qh * W / Sh = output width
        tp.Hout[p] = pi.out_h[p];
        moff += (int64_t)pi.in_h[p] * pi.out_w[p];
    }
    tp.plane_first = p0;
    tp.plane_count = pc;
    tp.n_frames = n;
    return tp;
}

bool spec_is_default(const ds_stage_spec& s, bool horizontal) {
    ds_filter_spec d;
    default_spec(&d);
    return stage_equal(s, horizontal ? d.h : d.v);
}

bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

ds::TDiv tdiv(uint32_t d) {
    ds::TDiv f{d, 0u, 0u};
    if (d > 1) {
        uint32_t l = 0;
        while ((1ULL << l) < d) ++l;                       // ceil(log2 d)
        f.m = (uint32_t)(((1ULL << (31 + l)) + d - 1) / d);
        f.s = l - 1;
    }
    return f;
}

dim3 task_grid(const ds_handle* h, int64_t items, int pc, int64_t n) {
    const int64_t target = (int64_t)h->sm_count * 8;
    int64_t x = std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, target));
    int64_t z = std::max<int64_t>(1, std::min<int64_t>(n, std::max<int64_t>(1, target / (x * pc))));
    z = std::min<int64_t>(z, 65535);
    return dim3((unsigned)x, (unsigned)pc, (unsigned)z);
}

int launch_htask(ds_handle* h, const uint8_t* in, int64_t n, uint8_t* mid, int p0, int pc,
                 cudaStream_t st) {
    const ds::TaskPlanes tp = task_planes(h, n, p0, pc);
    bool fast = spec_is_default(h->spec.h, true) && aligned(in, 16) && aligned(mid, 2);
    for (int p = p0; p < p0 + pc && fast; ++p) fast = (tp.W[p] % 16 == 0);
    if (fast) {
        // contiguous byte ranges of the flat packet stream: all planes of all
        // frames at once, or one range per frame for a plane subset
        const bool all = (p0 == 0 && pc == h->plan.n_planes);
        const int64_t ranges = all ? 1 : n;
        for (int64_t f = 0; f < ranges; ++f) {
            const int64_t ib = all ? 0 : f * tp.in_frame + tp.in_off[p0];
            const int64_t mb = all ? 0 : f * tp.mid_frame + tp.mid_off[p0];
            int64_t bytes = 0;
            for (int p = p0; p < p0 + pc; ++p) bytes += (int64_t)tp.W[p] * tp.H[p];
            if (all) bytes *= n;
            const int64_t chunks = bytes / 16;
            const int64_t blocks =
                std::max<int64_t>(1, std::min<int64_t>((chunks + 255) / 256, (int64_t)h->sm_count * 16));
            if (kHtaskTma && all && aligned(in, 16) && aligned(mid, 16) && bytes >= kHtaskUnit) {
                // one flat range: the TMA pipeline (persistent, one CTA per SM)
                constexpr int kStages = 4;
                const int out_stride = (int)((kHtaskUnit / 8 * 3 + 127) & ~127);
                const int smem = kStages * (int)kHtaskUnit + 3 * out_stride + 2 * kStages * 8;
                if (!h->htask_tma_ready) {
                    if (cudaFuncSetAttribute(ds::ds_htask_tma_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             smem) != cudaSuccess) {
                        cudaGetLastError();
                        return DS_ECUDA;
                    }
                    h->htask_tma_ready = true;
                }
                const int64_t units = (bytes + kHtaskUnit - 1) / kHtaskUnit;
                const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(units, h->sm_count));
                ds::ds_htask_tma_kernel<8><<<grid, 9 * 32, smem, st>>>(in, mid, bytes, (int32_t)kHtaskUnit, kStages);
            } else if (aligned(mid + mb, 16))
                ds::ds_htask_kernel<true><<<(unsigned)blocks, 256, 0, st>>>(in + ib, mid + mb, chunks);
            else
                ds::ds_htask_kernel<false><<<(unsigned)blocks, 256, 0, st>>>(in + ib, mid + mb, chunks);
        }
    } else {
        ds::GenericTask gt;
        gt.tp = tp;
        gt.s = h->spec.h;
        int64_t items = 0;
        for (int p = p0; p < p0 + pc; ++p) items = std::max<int64_t>(items, (int64_t)tp.H[p] * tp.Wm[p]);
        ds::ds_htask_generic<<<task_grid(h, items, pc, n), 256, 0, st>>>(in, mid, gt);
    }
    return cudaGetLastError() == cudaSuccess ? DS_OK : DS_ECUDA;
}

int launch_vtask(ds_handle* h, const uint8_t* mid, int64_t n, uint8_t* out, int p0, int pc,
                 cudaStream_t st) {
    const ds::TaskPlanes tp = task_planes(h, n, p0, pc);
    bool fast = spec_is_default(h->spec.v, false) && aligned(mid, 4) && aligned(out, 4) &&
                tp.mid_frame % 4 == 0 && tp.out_frame % 4 == 0;
    for (int p = p0; p < p0 + pc && fast; ++p)
        fast = (tp.Wm[p] % 4 == 0) && (tp.mid_off[p] % 4 == 0) && (tp.out_off[p] % 4 == 0);
    if (fast) {
        // one flat item space per block of frames (32-bit indices); 8-byte
        // column groups when every plane's rows and offsets allow it
        bool v8 = aligned(mid, 8) && aligned(out, 8) && tp.mid_frame % 8 == 0 && tp.out_frame % 8 == 0;
        for (int p = p0; p < p0 + pc && v8; ++p)
            v8 = (tp.Wm[p] % 8 == 0) && (tp.mid_off[p] % 8 == 0) && (tp.out_off[p] % 8 == 0);
        const int vec = v8 ? 8 : 4;
        ds::VFlat vf;
        std::memset(&vf, 0, sizeof vf);
        vf.planes = pc;
        uint32_t per = 0;
        for (int i = 0; i < pc; ++i) {
            const int p = p0 + i;
            const uint32_t quads = (uint32_t)(tp.Wm[p] / vec);
            vf.pstart[i] = per;
            vf.qdiv[i] = tdiv(quads);
            per += quads * (uint32_t)(tp.H[p] / 9);
        }
        vf.per_frame = per;
        vf.fdiv = tdiv(per);
        const int64_t fmax = std::max<int64_t>(1, ((1LL << 31) - 1) / std::max<uint32_t>(per, 1));
        for (int64_t f0 = 0; f0 < n && per > 0; f0 += fmax) {
            const int64_t nf = std::min<int64_t>(fmax, n - f0);
            const uint32_t items = (uint32_t)(nf * per);
            const int64_t blocks = std::max<int64_t>(
                1, std::min<int64_t>(((int64_t)items + 511) / 512, (int64_t)h->sm_count * 8));
            if (v8)
                ds::ds_vtask_kernel<uint2><<<(unsigned)blocks, 256, 0, st>>>(mid, out, tp, vf, f0, items);
            else
                ds::ds_vtask_kernel<uint32_t><<<(unsigned)blocks, 256, 0, st>>>(mid, out, tp, vf, f0, items);
        }
    } else {
        ds::GenericTask gt;
        gt.tp = tp;
        gt.s = h->spec.v;
        int64_t items = 0;
        for (int p = p0; p < p0 + pc; ++p) items = std::max<int64_t>(items, (int64_t)tp.Hout[p] * tp.Wm[p]);
        ds::ds_vtask_generic<<<task_grid(h, items, pc, n), 256, 0, st>>>(mid, out, gt);
    }
    return cudaGetLastError() == cudaSuccess ? DS_OK : DS_ECUDA;
}

int check_planes(const ds_handle* h, int p0, int pc) {
    return (p0 >= 0 && pc >= 1 && p0 + pc <= h->plan.n_planes) ? DS_OK : DS_EINVAL;
}

// ------------------------------------------------------------- schedules --
// Per-frame step lists.  Kinds: 0 = H2D, 1 = kernel, 2 = D2H.
struct Step {
    int kind;
    int plane;          // -1 = whole frame
    int task;           // 0 = H, 1 = V, 2 = fused (kernels only)
    int array;          // 0 = input, 1 = mid, 2 = output (copies only)
};

int steps_for(const ds_handle* h, int sched, Step* out) {
    const int P = h->plan.n_planes;
    int k = 0;
    if (sched == DS_SCHED_NAIVE) {
        // tasks in topological order (each plane's H before its V,
        // S:127), each preceded by H2D of its input and followed by D2H of its output
        for (int p = 0; p < P; ++p) {
            out[k++] = {0, p, -1, 0};
            out[k++] = {1, p, 0, -1};
            out[k++] = {2, p, -1, 1};
            out[k++] = {0, p, -1, 1};
            out[k++] = {1, p, 1, -1};
            out[k++] = {2, p, -1, 2};
        }
    } else if (sched == DS_SCHED_OPTIMIZED) {
        // 3 H2D (channel inputs) + 6 launches + 3 D2H (channel outputs)
        for (int p = 0; p < P; ++p) out[k++] = {0, p, -1, 0};
        for (int p = 0; p < P; ++p) {
            out[k++] = {1, p, 0, -1};
            out[k++] = {1, p, 1, -1};
        }
        for (int p = 0; p < P; ++p) out[k++] = {2, p, -1, 2};
    } else if (sched == DS_SCHED_FUSED) {
        out[k++] = {0, -1, -1, 0};
        out[k++] = {1, -1, 2, -1};
        out[k++] = {2, -1, -1, 2};
    }
    return k;
}

int64_t array_bytes(const ds_handle* h, int array, int plane) {
    const ds_plan_info& pi = h->plan;
    if (plane < 0)
        return array == 0 ? pi.in_frame_bytes : array == 1 ? mid_frame_bytes(h) : pi.out_frame_bytes;
    if (array == 0) return (int64_t)pi.in_w[plane] * pi.in_h[plane];
    if (array == 1) return (int64_t)pi.in_h[plane] * pi.out_w[plane];
    return (int64_t)pi.out_w[plane] * pi.out_h[plane];
}

int64_t array_offset(const ds_handle* h, int array, int plane) {
    if (plane < 0) return 0;
    if (array == 0) return h->plan.in_offset[plane];
    if (array == 2) return h->plan.out_offset[plane];
    int64_t off = 0;
    for (int q = 0; q < plane; ++q) off += (int64_t)h->plan.in_h[q] * h->plan.out_w[q];
    return off;
}

int sched_alloc(ds_handle* h) {
    SchedState& s = h->sched;
    if (s.ready) return DS_OK;
    if (cudaMalloc(&s.d_in, h->plan.in_frame_bytes) != cudaSuccess ||
        cudaMalloc(&s.d_mid, mid_frame_bytes(h)) != cudaSuccess ||
        cudaMalloc(&s.d_out, h->plan.out_frame_bytes) != cudaSuccess ||
        cudaHostAlloc(&s.h_mid, mid_frame_bytes(h), cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        free_sched_state(h);
        return DS_ENOMEM;
    }
    s.ready = true;
    return DS_OK;
}

}  // namespace

namespace dsi {
void free_sched_state(ds_handle* h) {
    SchedState& s = h->sched;
    if (s.d_in) cudaFree(s.d_in);
    if (s.d_mid) cudaFree(s.d_mid);
    if (s.d_out) cudaFree(s.d_out);
    if (s.h_mid) cudaFreeHost(s.h_mid);
    for (cudaEvent_t e : s.events) cudaEventDestroy(e);
    s = SchedState{};
}
}  // namespace dsi

// ================================================================ C ABI ==
extern "C" {

DS_API int64_t ds_mid_frame_bytes(const ds_handle* h) { return h ? mid_frame_bytes(h) : -1; }

DS_API int ds_run_htask(ds_handle* h, const uint8_t* in, int64_t n, uint8_t* mid, int32_t plane_first,
                        int32_t plane_count, ds_stream_t stream) {
    if (!h || n < 0) return DS_EINVAL;
    if (check_planes(h, plane_first, plane_count)) return DS_EINVAL;
    if (n == 0) return DS_OK;
    if (!in || !mid) return DS_EINVAL;
    if (ranges_overlap(in, n * h->plan.in_frame_bytes, mid, n * mid_frame_bytes(h))) return DS_EINVAL;
    DeviceGuard g(h->device);
    if (!g.ok) { cudaGetLastError(); return DS_ECUDA; }
    if (!device_ptr_on(in, h->device) || !device_ptr_on(mid, h->device)) return DS_EINVAL;
    return launch_htask(h, in, n, mid, plane_first, plane_count, reinterpret_cast<cudaStream_t>(stream));
}

DS_API int ds_run_vtask(ds_handle* h, const uint8_t* mid, int64_t n, uint8_t* out, int32_t plane_first,
                        int32_t plane_count, ds_stream_t stream) {
    if (!h || n < 0) return DS_EINVAL;
    if (check_planes(h, plane_first, plane_count)) return DS_EINVAL;
    if (n == 0) return DS_OK;
    if (!mid || !out) return DS_EINVAL;
    if (ranges_overlap(mid, n * mid_frame_bytes(h), out, n * h->plan.out_frame_bytes)) return DS_EINVAL;
    DeviceGuard g(h->device);
    if (!g.ok) { cudaGetLastError(); return DS_ECUDA; }
    if (!device_ptr_on(mid, h->device) || !device_ptr_on(out, h->device)) return DS_EINVAL;
    return launch_vtask(h, mid, n, out, plane_first, plane_count, reinterpret_cast<cudaStream_t>(stream));
}

DS_API int ds_schedule_plan(int32_t frame_w, int32_t frame_h, int32_t channels,
                            const ds_filter_spec* spec, int32_t schedule, ds_schedule_stats* s) {
    if (!s) return DS_EINVAL;
    ds_handle hh;                       // host-only: geometry, no CUDA state
    const int prc = make_plan(frame_w, frame_h, channels, spec, &hh.spec, &hh.plan);
    if (prc) return prc;
    hh.channels = channels;
    const ds_handle* h = &hh;
    std::memset(s, 0, sizeof *s);
    s->frames = 1;
    if (schedule == DS_SCHED_STREAMED) {
        // per frame, amortised: one H2D and one D2H per chunk of frames; with
        // SPEC's taps the dead row 9g+4 of every plane is not transferred
        ds_filter_spec def;
        default_spec(&def);
        const bool skip = stage_equal(h->spec.h, def.h) && stage_equal(h->spec.v, def.v) &&
                          h->plan.fused_eligible;
        s->h2d_bytes = skip ? h->plan.in_frame_bytes / 9 * 8 : h->plan.in_frame_bytes;
        s->d2h_bytes = h->plan.out_frame_bytes;
        s->h2d_count = s->d2h_count = s->launches = 1;
        return DS_OK;
    }
    Step steps[64];
    const int ns = steps_for(h, schedule, steps);
    if (ns == 0) return DS_EINVAL;
    for (int i = 0; i < ns; ++i) {
        const Step& st = steps[i];
        if (st.kind == 0) { ++s->h2d_count; s->h2d_bytes += array_bytes(h, st.array, st.plane); }
        if (st.kind == 2) { ++s->d2h_count; s->d2h_bytes += array_bytes(h, st.array, st.plane); }
        if (st.kind == 1) ++s->launches;
    }
    return DS_OK;
}

DS_API int ds_run_schedule(ds_handle* h, const uint8_t* host_in, int64_t n, uint8_t* host_out,
                           int32_t schedule, ds_schedule_stats* stats, ds_stream_t stream) {
    if (!h || n < 0 || !stats) return DS_EINVAL;
    if (n > 0 && (!host_in || !host_out)) return DS_EINVAL;
    const int64_t fin = h->plan.in_frame_bytes, fout = h->plan.out_frame_bytes;
    if (n > 0 && ranges_overlap(host_in, n * fin, host_out, n * fout)) return DS_EINVAL;
    std::memset(stats, 0, sizeof *stats);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (schedule == DS_SCHED_STREAMED) {
        int rc;
        cudaEvent_t a, b;
        {
            DeviceGuard g(h->device);
            if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) {
                cudaGetLastError();
                return DS_ECUDA;
            }
            cudaEventRecord(a, st);
        }
        rc = ds_run_host(h, host_in, n, host_out, stream);
        DeviceGuard g(h->device);
        cudaEventRecord(b, st);
        if (cudaEventSynchronize(b) != cudaSuccess) { cudaGetLastError(); rc = rc ? rc : DS_ECUDA; }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        if (rc) return rc;
        const int64_t chunk = h->host_chunk > 0 ? h->host_chunk
                                                : std::max<int64_t>(1, kHostChunkBytes / std::max<int64_t>(fin, 1));
        const int64_t chunks = n ? (n + chunk - 1) / chunk : 0;
        stats->frames = n;
        stats->h2d_count = stats->d2h_count = stats->launches = chunks;
        ds_schedule_stats pf;
        ds_schedule_plan(h->W, h->H, h->channels, &h->spec, DS_SCHED_STREAMED, &pf);
        stats->h2d_bytes = n * pf.h2d_bytes;
        stats->d2h_bytes = n * fout;
        stats->total_ms = ms;
        return DS_OK;
    }
    Step steps[64];
    const int ns = steps_for(h, schedule, steps);
    if (ns == 0) return DS_EINVAL;
    std::lock_guard<std::mutex> lk(h->host_mu);
    DeviceGuard g(h->device);
    if (!g.ok) { cudaGetLastError(); return DS_ECUDA; }
    int rc = sched_alloc(h);
    if (rc) return rc;
    SchedState& S = h->sched;
    const int64_t batch = std::max<int64_t>(1, std::min<int64_t>(n, 64));
    const size_t need = (size_t)(2 * ns * batch + 2);
    while (S.events.size() < need) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) { cudaGetLastError(); return DS_ECUDA; }
        S.events.push_back(e);
    }
    cudaEvent_t first = S.events[need - 2], last = S.events[need - 1];
    if (n == 0) return DS_OK;
    cudaEventRecord(first, st);
    for (int64_t f0 = 0; f0 < n; f0 += batch) {
        const int64_t m = std::min(batch, n - f0);
        int e = 0;
        for (int64_t f = f0; f < f0 + m; ++f) {
            for (int i = 0; i < ns; ++i) {
                const Step& sp = steps[i];
                cudaEventRecord(S.events[e++], st);
                if (sp.kind == 0) {
                    const int64_t off = array_offset(h, sp.array, sp.plane), bytes = array_bytes(h, sp.array, sp.plane);
                    const uint8_t* src = sp.array == 0 ? host_in + f * fin + off : S.h_mid + off;
                    uint8_t* dst = (sp.array == 0 ? S.d_in : S.d_mid) + off;
                    rc = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st) == cudaSuccess ? DS_OK : DS_ECUDA;
                } else if (sp.kind == 2) {
                    const int64_t off = array_offset(h, sp.array, sp.plane), bytes = array_bytes(h, sp.array, sp.plane);
                    const uint8_t* src = (sp.array == 1 ? S.d_mid : S.d_out) + off;
                    uint8_t* dst = sp.array == 1 ? S.h_mid + off : host_out + f * fout + off;
                    rc = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st) == cudaSuccess ? DS_OK : DS_ECUDA;
                } else if (sp.task == 2) {
                    rc = run_device(h, S.d_in, 1, S.d_out, st);
                } else if (sp.task == 0) {
                    rc = launch_htask(h, S.d_in, 1, S.d_mid, sp.plane, 1, st);
                } else {
                    rc = launch_vtask(h, S.d_mid, 1, S.d_out, sp.plane, 1, st);
                }
                cudaEventRecord(S.events[e++], st);
                if (rc) { cudaGetLastError(); return rc; }
            }
        }
        if (cudaEventSynchronize(S.events[e - 1]) != cudaSuccess) { cudaGetLastError(); return DS_ECUDA; }
        e = 0;
        for (int64_t f = f0; f < f0 + m; ++f)
            for (int i = 0; i < ns; ++i) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, S.events[e], S.events[e + 1]);
                e += 2;
                const Step& sp = steps[i];
                if (sp.kind == 0) {
                    stats->h2d_ms += ms; ++stats->h2d_count; stats->h2d_bytes += array_bytes(h, sp.array, sp.plane);
                } else if (sp.kind == 2) {
                    stats->d2h_ms += ms; ++stats->d2h_count; stats->d2h_bytes += array_bytes(h, sp.array, sp.plane);
                } else {
                    stats->kernel_ms += ms; ++stats->launches;
                    if (sp.plane >= 0) stats->kernel_ms_plane[sp.plane] += ms;
                }
            }
    }
    cudaEventRecord(last, st);
    if (cudaEventSynchronize(last) != cudaSuccess) { cudaGetLastError(); return DS_ECUDA; }
    float tot = 0.f;
    cudaEventElapsedTime(&tot, first, last);
    stats->total_ms = tot;
    stats->frames = n;
    return DS_OK;
}

}  // extern "C"
