/* abi_smoke.c -- the C ABI (include/ds.h) used from plain C, no Python.
 * Host-only part (always): ds_default_spec / ds_plan / ds_schedule_plan /
 * ds_compute_topology / error paths.  With argv[1] == "gpu": ds_create +
 * ds_run on cudaMalloc'd buffers for CIF 4:2:0 frames, checked against the
 * closed forms (constant frames stay constant; a linear ramp 16y+2x
 * gives the hand-worked values of tests/golden/ramp_9x8.json). */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ds.h"

/* minimal CUDA runtime declarations (no CUDA headers needed to build) */
typedef int cudaError_t;
extern cudaError_t cudaMalloc(void** p, size_t n);
extern cudaError_t cudaFree(void* p);
extern cudaError_t cudaMemcpy(void* d, const void* s, size_t n, int kind);
extern cudaError_t cudaDeviceSynchronize(void);

#define CHECK(c) do { if (!(c)) { fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, #c); return 1; } } while (0)

static int host_part(void) {
    ds_filter_spec spec;
    CHECK(ds_default_spec(&spec) == DS_OK);
    CHECK(spec.h.weight[0][1] == 5 && spec.v.weight[1][3] == 7 && spec.h.divisor == 6);
    ds_plan_info pi;
    CHECK(ds_plan(352, 288, 3, NULL, &pi) == DS_OK);
    CHECK(pi.out_w[0] == 132 && pi.out_h[0] == 128 && pi.out_frame_bytes == 25344);
    CHECK(ds_plan(1920, 1080, 3, NULL, &pi) == DS_OK && pi.in_frame_bytes == 3110400);
    CHECK(ds_plan(350, 288, 3, NULL, &pi) == DS_ESHAPE);
    CHECK(ds_create(350, 288, 3, NULL) == NULL && ds_last_error() == DS_ESHAPE);
    ds_schedule_stats st;
    CHECK(ds_schedule_plan(352, 288, 3, NULL, DS_SCHED_NAIVE, &st) == DS_OK);
    CHECK(st.h2d_count + st.d2h_count == 12 && st.h2d_bytes == 209088);
    CHECK(ds_schedule_plan(352, 288, 3, NULL, DS_SCHED_OPTIMIZED, &st) == DS_OK);
    CHECK(st.h2d_count + st.d2h_count == 6 && st.d2h_bytes == 25344);
    int64_t mult[2] = {288, 44};
    ds_topology t;
    CHECK(ds_compute_topology(2, mult, 256, 3, 64, 256, &t) == DS_OK);
    CHECK(t.local[0] == 16 && t.local[1] == 16 && t.global[1] == 48 && t.guarded == 1);
    CHECK(ds_run(NULL, NULL, 1, NULL, NULL) == DS_EINVAL);
    CHECK(strlen(ds_strerror(DS_ECUDA)) > 0);
    ds_destroy(NULL);
    printf("host part ok\n");
    return 0;
}

static int gpu_part(void) {
    ds_handle* h = ds_create(352, 288, 3, NULL);
    CHECK(h != NULL);
    const int64_t fin = ds_in_frame_bytes(h), fout = ds_out_frame_bytes(h), n = 3;
    unsigned char* hin = (unsigned char*)malloc((size_t)(n * fin));
    unsigned char* hout = (unsigned char*)malloc((size_t)(n * fout));
    /* frame 0: constant 100; frames 1-2: per-plane ramp 16y + 2x (mod 256) */
    for (int64_t f = 0; f < n; ++f) {
        int64_t off = 0;
        for (int p = 0; p < 3; ++p) {
            int32_t w, hh;
            CHECK(ds_plane_dims(h, p, &w, &hh, NULL, NULL) == DS_OK);
            for (int y = 0; y < hh; ++y)
                for (int x = 0; x < w; ++x)
                    hin[f * fin + off + (int64_t)y * w + x] =
                        (unsigned char)(f == 0 ? 100 : ((16 * (y % 9) + 2 * (x % 8)) & 255));
            off += (int64_t)w * hh;
        }
    }
    void *din = NULL, *dout = NULL;
    CHECK(cudaMalloc(&din, (size_t)(n * fin)) == 0 && cudaMalloc(&dout, (size_t)(n * fout)) == 0);
    CHECK(cudaMemcpy(din, hin, (size_t)(n * fin), 1) == 0);           /* host -> device */
    CHECK(ds_run(h, (const uint8_t*)din, n, (uint8_t*)dout, NULL) == DS_OK);
    CHECK(cudaDeviceSynchronize() == 0);
    CHECK(cudaMemcpy(hout, dout, (size_t)(n * fout), 2) == 0);        /* device -> host */
    for (int64_t i = 0; i < fout; ++i) CHECK(hout[i] == 100);
    /* ramp tile repeats every 9 rows x 8 cols: Out (4x3) per tile, golden ramp_9x8 */
    static const int golden[4][3] = {{12, 17, 22}, {48, 53, 58}, {84, 89, 94}, {120, 125, 130}};
    for (int y = 0; y < 128; ++y)
        for (int x = 0; x < 132; ++x)
            CHECK(hout[fout + (int64_t)y * 132 + x] == golden[y % 4][x % 3]);
    /* host path: same result through ds_run_host (pageable buffers) */
    memset(hout, 0, (size_t)(n * fout));
    CHECK(ds_run_host(h, hin, n, hout, NULL) == DS_OK);
    CHECK(cudaDeviceSynchronize() == 0);
    for (int64_t i = 0; i < fout; ++i) CHECK(hout[i] == 100);
    CHECK(hout[fout + 5 * 132 + 7] == golden[5 % 4][7 % 3]);
    printf("gpu part ok (kernel %d)\n", ds_last_kernel(h));
    cudaFree(din);
    cudaFree(dout);
    free(hin);
    free(hout);
    ds_destroy(h);
    return 0;
}

int main(int argc, char** argv) {
    if (host_part()) return 1;
    if (argc > 1 && strcmp(argv[1], "gpu") == 0) return gpu_part();
    return 0;
}
