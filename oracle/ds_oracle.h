/*
 * ds_oracle.h -- CPU ORACLE for the arxiv 1103.4881 downscaler hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1103_4881_b200/, include/ds.h, libds.so) never
 * links, includes or calls anything here, and this file includes nothing
 * from it.  Plain C11, single-threaded, no SIMD intrinsics.
 *
 * Citation key: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n.
 *
 * What is computed (PAPER sec. 3; SPEC tiler + sim modules,
 * S:248-286):
 *   per frame, per colour plane, a horizontal Array-OL repetitive task
 *   (pattern 8 -> 3, "interpolating packets of 8 pixels") followed by
 *   a vertical one (9 -> 4, 288 -> 128 lines), each
 *   applied through tilers (origin, paving, fitting; P:110 + footnote),
 *   the intermediate array stored as u8.
 *
 * Three independent code paths:
 *   O1 orc_execute_plane  -- tiler executor (element_index / extract /
 *                            body / write in row-major repetition order,
 *                            S:517-520), generic integer stage bodies.
 *   O2 orc_direct_plane   -- nested loops with SPEC's literal
 *                            hfilter_8to3 / vfilter_9to4.
 *   O3 orc_pixel          -- one output pixel from its closed form
 *                            (default taps only), brute force.
 *
 * Parity status: see the header of ds_oracle.c and DESIGN.md sec. "Oracle".
 */
#ifndef DS_ORACLE_H
#define DS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_EINVAL = -1, ORC_ESHAPE = -2, ORC_ENOMEM = -5 };
enum { ORC_MAXDIM = 4, ORC_MAXPAT = 16, ORC_MAXOUT = 8 };

/* Array-OL tiler: origin (array dims), paving (array dims x
 * repetition dims), fitting (array dims x pattern dims), pattern shape. */
typedef struct {
    int32_t ndim;                          /* array dims, 1..4            */
    int64_t shape[ORC_MAXDIM];             /* array extents               */
    int64_t origin[ORC_MAXDIM];
    int32_t nrep;                          /* repetition dims, 1..4       */
    int64_t paving[ORC_MAXDIM][ORC_MAXDIM];   /* [array dim][rep dim]     */
    int32_t npat;                          /* pattern dims, 0..4          */
    int64_t fitting[ORC_MAXDIM][ORC_MAXDIM];  /* [array dim][pattern dim] */
    int64_t pattern[ORC_MAXDIM];           /* pattern extents             */
} orc_tiler;

/* One separable integer stage (the elementary function of a repetitive
 * task): out[k] = clamp_0^255( trunc( (sum_i w[k][i]*pat[i] + bias) / divisor ) ),
 * which for SPEC's taps is hfilter_8to3 / vfilter_9to4. */
typedef struct {
    int32_t pattern;                       /* input pattern length P       */
    int32_t paving;                        /* input paving step S          */
    int32_t origin;                        /* input tiler origin (axis)    */
    int32_t outputs;                       /* output pattern length Q      */
    int32_t weight[ORC_MAXOUT][ORC_MAXPAT];
    int32_t divisor;
    int32_t bias;
} orc_stage;

/* ---- tiler module ------------------------------------------ */
int orc_element_index(const orc_tiler* t, const int64_t* r, const int64_t* f,
                      int64_t* idx_out);
int orc_extract_pattern(const uint8_t* arr, const orc_tiler* t,
                        const int64_t* r, uint8_t* pat_out);
int orc_write_pattern(uint8_t* arr, const orc_tiler* t, const int64_t* r,
                      const uint8_t* pat);
/* 0 = exact, 1 = overlaps, 2 = gaps (overlap takes precedence); up to
 * max_wit row-major linear witness indices are written to wit. */
int orc_check_coverage(const orc_tiler* t, int32_t nrep, const int64_t* rep_shape,
                       int64_t* wit, int32_t max_wit, int32_t* n_wit);

/* ---- elementary functions ----------------------------------- */
void orc_hfilter_8to3(const uint8_t in[8], uint8_t out[3]);
void orc_vfilter_9to4(const uint8_t in[9], uint8_t out[4]);
void orc_stage_apply(const orc_stage* s, const uint8_t* pat, uint8_t* out);
void orc_default_stages(orc_stage* h, orc_stage* v);

/* ---- O1: tiler executor for one plane ------------------------
 * in: H x W u8 row-major; out: (Qv*H/Sv) x (Qh*W/Sh).  order 0 = row-major
 * repetition order, 1 = reverse (order-independence property).   */
int orc_execute_plane(const uint8_t* in, int32_t W, int32_t H,
                      const orc_stage* h, const orc_stage* v,
                      uint8_t* out, int32_t order);

int orc_execute_plane_mid(const uint8_t* in, int32_t W, int32_t H,
                          const orc_stage* h, const orc_stage* v,
                          uint8_t* mid_out, uint8_t* out, int32_t order);

/* ---- a general repetitive task with arbitrary tilers */
int orc_run_task(const uint8_t* in, const orc_tiler* tin, uint8_t* out,
                 const orc_tiler* tout, int32_t nrep, const int64_t* rep_shape,
                 const orc_stage* body, int32_t order);

/* ---- whole frames: planes Y, plane 1, plane 2 contiguous --------
 * chroma: 0 = 4:4:4 (three equal planes), 1 = 4:2:0 (W/2 x H/2 chroma).  */
int orc_plane_dims(int32_t W, int32_t H, int32_t channels, int32_t chroma,
                   int32_t plane, int32_t* pw, int32_t* ph);
int orc_execute_frames(const uint8_t* in, int64_t n, int32_t W, int32_t H,
                       int32_t channels, int32_t chroma,
                       const orc_stage* h, const orc_stage* v, uint8_t* out);

/* ---- O2: direct nested loops, default taps ------------------ */
int orc_direct_plane(const uint8_t* in, int32_t W, int32_t H, uint8_t* out);
int orc_direct_frames(const uint8_t* in, int64_t n, int32_t W, int32_t H,
                      int32_t channels, int32_t chroma, uint8_t* out);

/* ---- O3: one output pixel, closed form, default taps -------------------- */
int orc_pixel(const uint8_t* plane, int32_t W, int32_t H, int32_t R, int32_t C);

#ifdef __cplusplus
}
#endif
#endif
