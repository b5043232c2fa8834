// ds_spec_jit.cu -- run-time compilation of K-N1s (ds_spec.cuh) for filter
// specs without a built-in instance (any separable stage spec).
//
// The kernel source is compiled into libds.so as a string (ds_spec_src.inc,
// generated from ds_spec.cuh by _build.py).  For a spec, the library writes
// its two stage types in the form of ds_spec_builtin.cuh (taps, pattern,
// paving, outputs, divisor, bias, origin as constants), compiles
// dss::ds_spec_kernel<JitH, JitV, PH> for the device's architecture with
// NVRTC straight to a cubin, and loads it with the driver API.  NVRTC is
// opened with dlopen and the driver entry points come from
// cudaGetDriverEntryPoint, so libds.so has no link-time dependency on either:
// without a runtime compiler the compiled variant is simply unavailable and
// K-N1g runs the spec with runtime taps.  Compiled kernels are cached per
// (device, source) for the life of the process.
#include <cuda.h>
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "ds.h"
#include "ds_internal.h"
#include "ds_spec.cuh"

namespace {

#include "ds_spec_src.inc"   // static const char kSpecSrc[]: the text of ds_spec.cuh

// ---- NVRTC, opened at run time
typedef int nvrtcResult_t;
typedef struct _nvrtcProgram* nvrtcProgram_t;
struct Nvrtc {
    void* so = nullptr;
    nvrtcResult_t (*create)(nvrtcProgram_t*, const char*, const char*, int, const char* const*, const char* const*) = nullptr;
    nvrtcResult_t (*destroy)(nvrtcProgram_t*) = nullptr;
    nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char* const*) = nullptr;
    nvrtcResult_t (*add_name)(nvrtcProgram_t, const char*) = nullptr;
    nvrtcResult_t (*lowered)(nvrtcProgram_t, const char*, const char**) = nullptr;
    nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t*) = nullptr;
    nvrtcResult_t (*cubin)(nvrtcProgram_t, char*) = nullptr;
    nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t*) = nullptr;
    nvrtcResult_t (*log)(nvrtcProgram_t, char*) = nullptr;
    bool ok = false;
};

// ---- driver API entry points
struct Drv {
    CUresult (*module_load)(CUmodule*, const void*) = nullptr;
    CUresult (*get_function)(CUfunction*, CUmodule, const char*) = nullptr;
    CUresult (*func_set_attr)(CUfunction, CUfunction_attribute, int) = nullptr;
    CUresult (*occupancy)(int*, CUfunction, int, size_t) = nullptr;
    CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream,
                       void**, void**) = nullptr;
    bool ok = false;
};

std::mutex g_mu;
Nvrtc g_nvrtc;
Drv g_drv;
bool g_init = false;
std::map<std::string, CUfunction> g_cache;
std::string g_last_log;

template <class F>
bool sym(void* so, const char* name, F& f) {
    f = reinterpret_cast<F>(dlsym(so, name));
    return f != nullptr;
}
template <class F>
bool drv_sym(const char* name, F& f) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
        !p) {
        cudaGetLastError();
        return false;
    }
    f = reinterpret_cast<F>(p);
    return true;
}

void init_locked() {
    if (g_init) return;
    g_init = true;
    const char* env = getenv("DS_NVRTC");
    const char* names[] = {env ? env : "libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
    for (const char* n : names) {
        if (!n) continue;
        g_nvrtc.so = dlopen(n, RTLD_NOW | RTLD_LOCAL);
        if (g_nvrtc.so) break;
    }
    if (g_nvrtc.so) {
        Nvrtc& r = g_nvrtc;
        r.ok = sym(r.so, "nvrtcCreateProgram", r.create) && sym(r.so, "nvrtcDestroyProgram", r.destroy) &&
               sym(r.so, "nvrtcCompileProgram", r.compile) && sym(r.so, "nvrtcAddNameExpression", r.add_name) &&
               sym(r.so, "nvrtcGetLoweredName", r.lowered) && sym(r.so, "nvrtcGetCUBINSize", r.cubin_size) &&
               sym(r.so, "nvrtcGetCUBIN", r.cubin) && sym(r.so, "nvrtcGetProgramLogSize", r.log_size) &&
               sym(r.so, "nvrtcGetProgramLog", r.log);
    }
    Drv& d = g_drv;
    d.ok = drv_sym("cuModuleLoadData", d.module_load) && drv_sym("cuModuleGetFunction", d.get_function) &&
           drv_sym("cuFuncSetAttribute", d.func_set_attr) &&
           drv_sym("cuOccupancyMaxActiveBlocksPerMultiprocessor", d.occupancy) &&
           drv_sym("cuLaunchKernel", d.launch);
}

// A stage type in the form of ds_spec_builtin.cuh
std::string stage_source(const char* name, const ds_stage_spec& s) {
    std::string o = "struct ";
    o += name;
    char buf[256];
    std::snprintf(buf, sizeof buf, " {\n    static constexpr int P = %d, S = %d, Q = %d, D = %d, B = %d, O = %d;\n",
                  s.pattern, s.paving, s.outputs, s.divisor, s.bias, s.origin);
    o += buf;
    o += "    __host__ __device__ static constexpr int w(int j, int i) {\n        constexpr int t[Q][P] = {";
    for (int j = 0; j < s.outputs; ++j) {
        o += j ? ", {" : "{";
        for (int i = 0; i < s.pattern; ++i) {
            std::snprintf(buf, sizeof buf, i ? ", %d" : "%d", s.weight[j][i]);
            o += buf;
        }
        o += "}";
    }
    o += "};\n        return (j >= 0 && j < Q && i >= 0 && i < P) ? t[j][i] : 0;\n    }\n};\n";
    return o;
}

}  // namespace

namespace dsi {

bool spec_jit_available() {
    std::lock_guard<std::mutex> lk(g_mu);
    init_locked();
    return g_nvrtc.ok && g_drv.ok;
}

// The last compilation's log, copied per calling thread (stable until that
// thread calls again).
const char* spec_jit_log() {
    thread_local std::string copy;
    std::lock_guard<std::mutex> lk(g_mu);
    copy = g_last_log;
    return copy.c_str();
}

// Compile (or fetch from the cache) K-N1s for the handle's spec, window phase
// and row alignment on the current device.  Returns a CUfunction as SpecFn, or
// nullptr.
SpecFn spec_jit_kernel(ds_handle* h, int phase, int align) {
    std::lock_guard<std::mutex> lk(g_mu);
    init_locked();
    if (!g_nvrtc.ok || !g_drv.ok) {
        if (getenv("DS_JIT_VERBOSE"))
            std::fprintf(stderr, "ds_spec_jit: nvrtc %s, driver entry points %s\n", g_nvrtc.ok ? "ok" : "missing",
                         g_drv.ok ? "ok" : "missing");
        return nullptr;
    }
    int major = 0, minor = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, h->device) != cudaSuccess ||
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, h->device) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    char defs[256];
    std::snprintf(defs, sizeof defs,
                  "#define DS_SPEC_NW %d\n#define DS_SPEC_MINB %d\n#define DS_SPEC_MAXP %d\n#define DS_SPEC_WS %d\n"
                  "#define DS_SPEC_NWV %d\n",
                  DS_SPEC_NW, DS_SPEC_MINB, DS_SPEC_MAXP, DS_SPEC_WS, DS_SPEC_NWV);
    std::string src = defs;
    src += kSpecSrc;
    src += "\nnamespace dss {\n";
    src += stage_source("JitH", h->spec.h);
    src += stage_source("JitV", h->spec.v);
    src += "}  // namespace dss\n";
    char name[96];
    std::snprintf(name, sizeof name, "&dss::ds_spec_kernel<dss::JitH, dss::JitV, %d, %d>", phase, align);
    char arch[64];
    std::snprintf(arch, sizeof arch, "--gpu-architecture=sm_%d%d%s", major, minor, major >= 9 ? "a" : "");
    const std::string key = std::to_string(h->device) + "|" + arch + "|" + name + "|" + src;
    auto it = g_cache.find(key);
    if (it != g_cache.end()) return reinterpret_cast<SpecFn>(it->second);

    nvrtcProgram_t prog = nullptr;
    if (g_nvrtc.create(&prog, src.c_str(), "ds_spec_jit.cu", 0, nullptr, nullptr) != 0) return nullptr;
    g_nvrtc.add_name(prog, name);
    const char* opts[] = {arch, "-std=c++17", "-default-device", "-lineinfo"};
    const int rc = g_nvrtc.compile(prog, 4, opts);
    size_t ls = 0;
    g_nvrtc.log_size(prog, &ls);
    g_last_log.assign(ls, '\0');
    if (ls) g_nvrtc.log(prog, &g_last_log[0]);
    CUfunction fn = nullptr;
    if (rc == 0) {
        const char* lowered = nullptr;
        size_t cs = 0;
        if (g_nvrtc.lowered(prog, name, &lowered) == 0 && g_nvrtc.cubin_size(prog, &cs) == 0 && cs > 0) {
            std::vector<char> cubin(cs);
            CUmodule mod = nullptr;
            DeviceGuard g(h->device);
            if (g_nvrtc.cubin(prog, cubin.data()) == 0 && g_drv.module_load(&mod, cubin.data()) == CUDA_SUCCESS &&
                g_drv.get_function(&fn, mod, lowered) != CUDA_SUCCESS)
                fn = nullptr;
        }
    }
    g_nvrtc.destroy(&prog);
    if (getenv("DS_JIT_VERBOSE"))
        std::fprintf(stderr, "ds_spec_jit: nvrtc rc=%d fn=%p\n%s\n", rc, (void*)fn, g_last_log.c_str());
    if (fn) g_cache[key] = fn;
    return reinterpret_cast<SpecFn>(fn);
}

int spec_jit_set_smem(SpecFn fn, int smem) {
    return g_drv.func_set_attr(reinterpret_cast<CUfunction>(fn), CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                               smem) == CUDA_SUCCESS ? DS_OK : DS_ECUDA;
}

int spec_jit_occupancy(SpecFn fn, int threads, int smem, int* occ) {
    return g_drv.occupancy(occ, reinterpret_cast<CUfunction>(fn), threads, (size_t)smem) == CUDA_SUCCESS ? DS_OK
                                                                                                        : DS_ECUDA;
}

int spec_jit_launch(SpecFn fn, unsigned grid, unsigned threads, unsigned smem, cudaStream_t st, void** args) {
    return g_drv.launch(reinterpret_cast<CUfunction>(fn), grid, 1, 1, threads, 1, 1, smem, reinterpret_cast<CUstream>(st),
                        args, nullptr) == CUDA_SUCCESS ? DS_OK : DS_ECUDA;
}

}  // namespace dsi
