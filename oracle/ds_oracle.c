/*
 * ds_oracle.c -- CPU ORACLE (test infrastructure only; see ds_oracle.h).
 *
 * Plain, slow, obviously-correct C11, single-threaded.  Every function cites
 * the passage it follows.  P:n = PAPER.md line n, S:n = SPEC.md line n.
 * Shares no code, header, table or constant with the CUDA path.
 *
 * Pins (tests/test_oracle.py, all `-m "not gpu"`):
 *   orc_element_index / extract / write / check_coverage
 *       SPEC worked examples S:254-256, S:264-265, S:274-275, S:284-286;
 *       linearity + write/extract identity + brute-force coverage on random
 *       tilers.
 *   orc_hfilter_8to3 / orc_vfilter_9to4 / orc_stage_apply (default taps)
 *       SPEC examples S:533-535; taps re-derived from SPEC's
 *       sample positions s_k=(k+1/2)P/Q-1/2 by linear
 *       interpolation; exhaustive 65,536-pair check against exact rational
 *       round-half-up; 0/255 fixed points, [min,max].
 *   orc_execute_plane (O1) / orc_direct_plane (O2) / orc_pixel (O3)
 *       printed geometry 352x288 -> 132x128, [288,44],
 *       176x144 -> 66x64; O1 == O2 == O3 on random frames;
 *       order independence; hand-worked goldens in tests/golden/;
 *       dead-tap liveness; independent exact-rational brute force.
 *   orc_execute_plane with general stages (halo P > S, origin != 0)
 *       roll invariance (toroidal modulo rule) and, for bias 0 /
 *       divisor 1, equality with the matrix form A_v . In . A_h^T.
 */
#include "ds_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------- */
/* tiler module                                                            */
/* ---------------------------------------------------------------------- */

/* Mathematical (non-negative) modulo, "with the mathematical (always
 * non-negative) modulo". */
static int64_t nn_mod(int64_t a, int64_t m) {
    int64_t r = a % m;
    return r < 0 ? r + m : r;
}

static int tiler_ok(const orc_tiler* t) {
    if (!t) return 0;
    if (t->ndim < 1 || t->ndim > ORC_MAXDIM) return 0;
    if (t->nrep < 1 || t->nrep > ORC_MAXDIM) return 0;
    if (t->npat < 0 || t->npat > ORC_MAXDIM) return 0;
    for (int d = 0; d < t->ndim; ++d)
        if (t->shape[d] < 1) return 0;
    for (int k = 0; k < t->npat; ++k)
        if (t->pattern[k] < 1) return 0;
    return 1;
}

/* element_index(tiler, r, f) = (origin + paving.r + fitting.f) mod shape,
 * component-wise. */
int orc_element_index(const orc_tiler* t, const int64_t* r, const int64_t* f,
                      int64_t* idx_out) {
    if (!tiler_ok(t) || !r || !idx_out || (t->npat > 0 && !f)) return ORC_EINVAL;
    for (int d = 0; d < t->ndim; ++d) {
        int64_t v = t->origin[d];
        for (int j = 0; j < t->nrep; ++j) v += t->paving[d][j] * r[j];
        for (int k = 0; k < t->npat; ++k) v += t->fitting[d][k] * f[k];
        idx_out[d] = nn_mod(v, t->shape[d]);
    }
    return ORC_OK;
}

/* row-major linearisation of an array index ("Row-major linearization
 * of patterns and arrays throughout"). */
static int64_t lin_index(const orc_tiler* t, const int64_t* idx) {
    int64_t off = 0;
    for (int d = 0; d < t->ndim; ++d) off = off * t->shape[d] + idx[d];
    return off;
}

static int64_t pattern_size(const orc_tiler* t) {
    int64_t n = 1;
    for (int k = 0; k < t->npat; ++k) n *= t->pattern[k];
    return n;
}

/* the row-major pattern coordinate f of the p-th pattern element */
static void pattern_coord(const orc_tiler* t, int64_t p, int64_t* f) {
    for (int k = t->npat - 1; k >= 0; --k) {
        f[k] = p % t->pattern[k];
        p /= t->pattern[k];
    }
}

/* extract_pattern: pattern[f] = array[element_index(t, r, f)], f iterated
 * row-major. */
int orc_extract_pattern(const uint8_t* arr, const orc_tiler* t,
                        const int64_t* r, uint8_t* pat_out) {
    if (!arr || !pat_out || !tiler_ok(t) || !r) return ORC_EINVAL;
    int64_t np = pattern_size(t);
    for (int64_t p = 0; p < np; ++p) {
        int64_t f[ORC_MAXDIM] = {0}, idx[ORC_MAXDIM];
        pattern_coord(t, p, f);
        orc_element_index(t, r, f, idx);
        pat_out[p] = arr[lin_index(t, idx)];
    }
    return ORC_OK;
}

/* write_pattern: array[element_index(t, r, f)] = p[f]. */
int orc_write_pattern(uint8_t* arr, const orc_tiler* t, const int64_t* r,
                      const uint8_t* pat) {
    if (!arr || !pat || !tiler_ok(t) || !r) return ORC_EINVAL;
    int64_t np = pattern_size(t);
    for (int64_t p = 0; p < np; ++p) {
        int64_t f[ORC_MAXDIM] = {0}, idx[ORC_MAXDIM];
        pattern_coord(t, p, f);
        orc_element_index(t, r, f, idx);
        arr[lin_index(t, idx)] = pat[p];
    }
    return ORC_OK;
}

/* check_coverage: brute-force enumeration of element_index over every
 * (r, f); exact iff every array element is hit exactly once. */
int orc_check_coverage(const orc_tiler* t, int32_t nrep, const int64_t* rep_shape,
                       int64_t* wit, int32_t max_wit, int32_t* n_wit) {
    if (!tiler_ok(t) || nrep != t->nrep || !rep_shape) return ORC_EINVAL;
    int64_t nelem = 1;
    for (int d = 0; d < t->ndim; ++d) nelem *= t->shape[d];
    int64_t nr = 1;
    for (int j = 0; j < nrep; ++j) {
        if (rep_shape[j] < 1) return ORC_EINVAL;
        nr *= rep_shape[j];
    }
    int64_t* count = (int64_t*)calloc((size_t)nelem, sizeof(int64_t));
    if (!count) return ORC_ENOMEM;
    int64_t np = pattern_size(t);
    for (int64_t q = 0; q < nr; ++q) {
        int64_t r[ORC_MAXDIM] = {0}, rem = q;
        for (int j = nrep - 1; j >= 0; --j) { r[j] = rem % rep_shape[j]; rem /= rep_shape[j]; }
        for (int64_t p = 0; p < np; ++p) {
            int64_t f[ORC_MAXDIM] = {0}, idx[ORC_MAXDIM];
            pattern_coord(t, p, f);
            orc_element_index(t, r, f, idx);
            count[lin_index(t, idx)] += 1;
        }
    }
    int result = 0;
    for (int64_t e = 0; e < nelem; ++e) if (count[e] > 1) { result = 1; break; }
    if (result == 0)
        for (int64_t e = 0; e < nelem; ++e) if (count[e] == 0) { result = 2; break; }
    int32_t nw = 0;
    if (result != 0) {
        for (int64_t e = 0; e < nelem && nw < max_wit; ++e) {
            int hit = (result == 1) ? (count[e] > 1) : (count[e] == 0);
            if (hit) { if (wit) wit[nw] = e; ++nw; }
        }
    }
    if (n_wit) *n_wit = nw;
    free(count);
    return result;
}

/* ---------------------------------------------------------------------- */
/* elementary functions                                                    */
/* ---------------------------------------------------------------------- */

static uint8_t clamp_u8(int64_t v) {
    return (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v));
}

/* hfilter_8to3, written literally:
 *   out0 = (1*in[0] + 5*in[1] + 3) / 6
 *   out1 = (3*in[3] + 3*in[4] + 3) / 6
 *   out2 = (5*in[6] + 1*in[7] + 3) / 6
 * integer (truncating) division, clamp 0..255.                          */
void orc_hfilter_8to3(const uint8_t in[8], uint8_t out[3]) {
    out[0] = clamp_u8((1 * (int64_t)in[0] + 5 * (int64_t)in[1] + 3) / 6);
    out[1] = clamp_u8((3 * (int64_t)in[3] + 3 * (int64_t)in[4] + 3) / 6);
    out[2] = clamp_u8((5 * (int64_t)in[6] + 1 * (int64_t)in[7] + 3) / 6);
}

/* vfilter_9to4, written literally:
 *   out0 = (3*in[0] + 5*in[1] + 4) / 8
 *   out1 = (1*in[2] + 7*in[3] + 4) / 8
 *   out2 = (7*in[5] + 1*in[6] + 4) / 8
 *   out3 = (5*in[7] + 3*in[8] + 4) / 8                                   */
void orc_vfilter_9to4(const uint8_t in[9], uint8_t out[4]) {
    out[0] = clamp_u8((3 * (int64_t)in[0] + 5 * (int64_t)in[1] + 4) / 8);
    out[1] = clamp_u8((1 * (int64_t)in[2] + 7 * (int64_t)in[3] + 4) / 8);
    out[2] = clamp_u8((7 * (int64_t)in[5] + 1 * (int64_t)in[6] + 4) / 8);
    out[3] = clamp_u8((5 * (int64_t)in[7] + 3 * (int64_t)in[8] + 4) / 8);
}

/* Generic separable integer stage: the same fixed-point interpolation form
 * as S:530/S:540 with a tap table, truncating division, clamp. */
void orc_stage_apply(const orc_stage* s, const uint8_t* pat, uint8_t* out) {
    for (int k = 0; k < s->outputs; ++k) {
        int64_t acc = s->bias;
        for (int i = 0; i < s->pattern; ++i) acc += (int64_t)s->weight[k][i] * pat[i];
        out[k] = clamp_u8(acc / s->divisor);   /* C division truncates toward 0 */
    }
}

/* SPEC's taps as stage tables. */
void orc_default_stages(orc_stage* h, orc_stage* v) {
    memset(h, 0, sizeof *h);
    h->pattern = 8; h->paving = 8; h->origin = 0; h->outputs = 3;
    h->weight[0][0] = 1; h->weight[0][1] = 5;
    h->weight[1][3] = 3; h->weight[1][4] = 3;
    h->weight[2][6] = 5; h->weight[2][7] = 1;
    h->divisor = 6; h->bias = 3;
    memset(v, 0, sizeof *v);
    v->pattern = 9; v->paving = 9; v->origin = 0; v->outputs = 4;
    v->weight[0][0] = 3; v->weight[0][1] = 5;
    v->weight[1][2] = 1; v->weight[1][3] = 7;
    v->weight[2][5] = 7; v->weight[2][6] = 1;
    v->weight[3][7] = 5; v->weight[3][8] = 3;
    v->divisor = 8; v->bias = 4;
}

static int stage_ok(const orc_stage* s) {
    return s && s->pattern >= 1 && s->pattern <= ORC_MAXPAT && s->paving >= 1 &&
           s->outputs >= 1 && s->outputs <= ORC_MAXOUT && s->divisor >= 1;
}

/* ---------------------------------------------------------------------- */
/* O1: tiler executor (SPEC sim.execute)                        */
/* ---------------------------------------------------------------------- */

/* Run one repetitive task: for each r of rep (row-major, or reverse),
 * extract the input pattern, apply the stage body, write the output
 * pattern. */
static void run_task(const uint8_t* in, const orc_tiler* tin,
                     uint8_t* out, const orc_tiler* tout,
                     const int64_t rep[2], const orc_stage* body, int32_t order) {
    uint8_t pat[ORC_MAXPAT], res[ORC_MAXOUT];
    int64_t nr = rep[0] * rep[1];
    for (int64_t q = 0; q < nr; ++q) {
        int64_t lin = order ? (nr - 1 - q) : q;
        int64_t r[2] = { lin / rep[1], lin % rep[1] };
        orc_extract_pattern(in, tin, r, pat);
        orc_stage_apply(body, pat, res);
        orc_write_pattern(out, tout, r, res);
    }
}

/*
 * The downscaler model of PAPER sec. 3.1 for one plane, in SPEC's tiler
 * form:
 *   H task  rep [H, W/Sh]
 *     in  : origin (0, oh), paving [[1,0],[0,Sh]], fitting [[0],[1]], pattern [Ph] on (H, W)
 *     out : origin (0, 0),  paving [[1,0],[0,Qh]], fitting [[0],[1]], pattern [Qh] on (H, Wm)
 *   V task  rep [H/Sv, Wm]
 *     in  : origin (ov, 0), paving [[Sv,0],[0,1]], fitting [[1],[0]], pattern [Pv] on (H, Wm)
 *     out : origin (0, 0),  paving [[Qv,0],[0,1]], fitting [[1],[0]], pattern [Qv] on (Ho, Wm)
 * with Wm = Qh*W/Sh, Ho = Qv*H/Sv.  For CIF luma the H repetition space is
 * [288,44], the paper's yhfk multiplicity.  Mid is u8.
 */
int orc_execute_plane(const uint8_t* in, int32_t W, int32_t H,
                      const orc_stage* h, const orc_stage* v,
                      uint8_t* out, int32_t order) {
    return orc_execute_plane_mid(in, W, H, h, v, NULL, out, order);
}

/* Same as orc_execute_plane; if mid_out is not NULL the intermediate array
 * Mid (H x Qh*W/Sh, the H task's output array) is copied there. */
int orc_execute_plane_mid(const uint8_t* in, int32_t W, int32_t H,
                          const orc_stage* h, const orc_stage* v,
                          uint8_t* mid_out, uint8_t* out, int32_t order) {
    if (!in || !out || !stage_ok(h) || !stage_ok(v) || W < 1 || H < 1) return ORC_EINVAL;
    if (W % h->paving != 0 || H % v->paving != 0) return ORC_ESHAPE;
    int64_t Wm = (int64_t)h->outputs * (W / h->paving);
    int64_t Ho = (int64_t)v->outputs * (H / v->paving);

    orc_tiler hin, hout, vin, vout;
    memset(&hin, 0, sizeof hin); memset(&hout, 0, sizeof hout);
    memset(&vin, 0, sizeof vin); memset(&vout, 0, sizeof vout);

    hin.ndim = 2; hin.shape[0] = H; hin.shape[1] = W;
    hin.origin[0] = 0; hin.origin[1] = h->origin;
    hin.nrep = 2; hin.paving[0][0] = 1; hin.paving[1][1] = h->paving;
    hin.npat = 1; hin.fitting[0][0] = 0; hin.fitting[1][0] = 1; hin.pattern[0] = h->pattern;

    hout.ndim = 2; hout.shape[0] = H; hout.shape[1] = Wm;
    hout.nrep = 2; hout.paving[0][0] = 1; hout.paving[1][1] = h->outputs;
    hout.npat = 1; hout.fitting[1][0] = 1; hout.pattern[0] = h->outputs;

    vin.ndim = 2; vin.shape[0] = H; vin.shape[1] = Wm;
    vin.origin[0] = v->origin; vin.origin[1] = 0;
    vin.nrep = 2; vin.paving[0][0] = v->paving; vin.paving[1][1] = 1;
    vin.npat = 1; vin.fitting[0][0] = 1; vin.fitting[1][0] = 0; vin.pattern[0] = v->pattern;

    vout.ndim = 2; vout.shape[0] = Ho; vout.shape[1] = Wm;
    vout.nrep = 2; vout.paving[0][0] = v->outputs; vout.paving[1][1] = 1;
    vout.npat = 1; vout.fitting[0][0] = 1; vout.pattern[0] = v->outputs;

    uint8_t* mid = (uint8_t*)calloc((size_t)(H * Wm), 1);
    if (!mid) return ORC_ENOMEM;
    int64_t hrep[2] = { H, W / h->paving };
    int64_t vrep[2] = { H / v->paving, Wm };
    run_task(in, &hin, mid, &hout, hrep, h, order);    /* toposort: H before V */
    run_task(mid, &vin, out, &vout, vrep, v, order);
    if (mid_out) memcpy(mid_out, mid, (size_t)(H * Wm));
    free(mid);
    return ORC_OK;
}

/* A general repetitive task (executed as S:517-520): for every
 * repetition index r of rep_shape (row-major, or reverse when order = 1),
 * pattern = extract(in, tin, r); out pattern = body(pattern); write(out,
 * tout, r).  The body is the linear integer stage over the row-major
 * flattened input pattern (body->pattern elements), producing
 * body->outputs elements in the output pattern's row-major order. */
int orc_run_task(const uint8_t* in, const orc_tiler* tin, uint8_t* out,
                 const orc_tiler* tout, int32_t nrep, const int64_t* rep_shape,
                 const orc_stage* body, int32_t order) {
    if (!in || !out || !tiler_ok(tin) || !tiler_ok(tout) || !rep_shape || !body) return ORC_EINVAL;
    if (nrep != tin->nrep || nrep != tout->nrep) return ORC_EINVAL;
    if (pattern_size(tin) != body->pattern || pattern_size(tout) != body->outputs) return ORC_EINVAL;
    if (body->pattern > ORC_MAXPAT || body->outputs > ORC_MAXOUT || body->divisor < 1) return ORC_EINVAL;
    int64_t nr = 1;
    for (int j = 0; j < nrep; ++j) {
        if (rep_shape[j] < 1) return ORC_EINVAL;
        nr *= rep_shape[j];
    }
    uint8_t pat[ORC_MAXPAT], res[ORC_MAXOUT];
    for (int64_t q = 0; q < nr; ++q) {
        int64_t lin = order ? (nr - 1 - q) : q;
        int64_t r[ORC_MAXDIM] = {0};
        for (int j = nrep - 1; j >= 0; --j) { r[j] = lin % rep_shape[j]; lin /= rep_shape[j]; }
        orc_extract_pattern(in, tin, r, pat);
        orc_stage_apply(body, pat, res);
        orc_write_pattern(out, tout, r, res);
    }
    return ORC_OK;
}

/* Plane layout of a frame: Y then plane 1 then plane 2, row-major u8, no
 * headers; 4:2:0 chroma is (W/2, H/2) (SPEC default), 4:4:4
 * is three equal planes (the paper's "24-bit RGB"). */
int orc_plane_dims(int32_t W, int32_t H, int32_t channels, int32_t chroma,
                   int32_t plane, int32_t* pw, int32_t* ph) {
    if (W < 1 || H < 1) return ORC_ESHAPE;
    if (channels != 1 && channels != 3) return ORC_EINVAL;
    if (plane < 0 || plane >= channels) return ORC_EINVAL;
    if (channels == 3 && chroma == 1 && plane > 0) {
        if (W % 2 != 0 || H % 2 != 0) return ORC_ESHAPE;
        *pw = W / 2; *ph = H / 2;
    } else {
        *pw = W; *ph = H;
    }
    return ORC_OK;
}

int orc_execute_frames(const uint8_t* in, int64_t n, int32_t W, int32_t H,
                       int32_t channels, int32_t chroma,
                       const orc_stage* h, const orc_stage* v, uint8_t* out) {
    if (n < 0 || !stage_ok(h) || !stage_ok(v)) return ORC_EINVAL;
    int64_t in_off[3], out_off[3], in_frame = 0, out_frame = 0;
    int32_t pw[3], ph[3];
    for (int p = 0; p < channels; ++p) {
        int rc = orc_plane_dims(W, H, channels, chroma, p, &pw[p], &ph[p]);
        if (rc) return rc;
        if (pw[p] % h->paving || ph[p] % v->paving) return ORC_ESHAPE;
        in_off[p] = in_frame; out_off[p] = out_frame;
        in_frame += (int64_t)pw[p] * ph[p];
        out_frame += ((int64_t)h->outputs * (pw[p] / h->paving)) *
                     ((int64_t)v->outputs * (ph[p] / v->paving));
    }
    for (int64_t f = 0; f < n; ++f)                 /* no inter-frame state */
        for (int p = 0; p < channels; ++p) {
            int rc = orc_execute_plane(in + f * in_frame + in_off[p], pw[p], ph[p], h, v,
                                       out + f * out_frame + out_off[p], 0);
            if (rc) return rc;
        }
    return ORC_OK;
}

/* ---------------------------------------------------------------------- */
/* O2: direct_downscale_oracle                                 */
/* ---------------------------------------------------------------------- */

/* "per plane: apply hfilter_8to3 to each consecutive 8-column packet of
 * each row, then vfilter_9to4 to each consecutive 9-row packet of each
 * column of the intermediate"; non-divisible shape -> error. */
int orc_direct_plane(const uint8_t* in, int32_t W, int32_t H, uint8_t* out) {
    if (!in || !out || W < 1 || H < 1) return ORC_EINVAL;
    if (W % 8 != 0 || H % 9 != 0) return ORC_ESHAPE;
    int32_t Wm = W / 8 * 3;
    uint8_t* mid = (uint8_t*)malloc((size_t)Wm * H);
    if (!mid) return ORC_ENOMEM;
    for (int32_t y = 0; y < H; ++y)
        for (int32_t p = 0; p < W / 8; ++p)
            orc_hfilter_8to3(in + (int64_t)y * W + 8 * p, mid + (int64_t)y * Wm + 3 * p);
    for (int32_t c = 0; c < Wm; ++c)
        for (int32_t g = 0; g < H / 9; ++g) {
            uint8_t col[9], res[4];
            for (int i = 0; i < 9; ++i) col[i] = mid[(int64_t)(9 * g + i) * Wm + c];
            orc_vfilter_9to4(col, res);
            for (int k = 0; k < 4; ++k) out[(int64_t)(4 * g + k) * Wm + c] = res[k];
        }
    free(mid);
    return ORC_OK;
}

int orc_direct_frames(const uint8_t* in, int64_t n, int32_t W, int32_t H,
                      int32_t channels, int32_t chroma, uint8_t* out) {
    if (n < 0) return ORC_EINVAL;
    int64_t in_frame = 0, out_frame = 0, in_off[3], out_off[3];
    int32_t pw[3], ph[3];
    for (int p = 0; p < channels; ++p) {
        int rc = orc_plane_dims(W, H, channels, chroma, p, &pw[p], &ph[p]);
        if (rc) return rc;
        if (pw[p] % 8 || ph[p] % 9) return ORC_ESHAPE;
        in_off[p] = in_frame; out_off[p] = out_frame;
        in_frame += (int64_t)pw[p] * ph[p];
        out_frame += (int64_t)(pw[p] / 8 * 3) * (ph[p] / 9 * 4);
    }
    for (int64_t f = 0; f < n; ++f)
        for (int p = 0; p < channels; ++p) {
            int rc = orc_direct_plane(in + f * in_frame + in_off[p], pw[p], ph[p],
                                      out + f * out_frame + out_off[p]);
            if (rc) return rc;
        }
    return ORC_OK;
}

/* ---------------------------------------------------------------------- */
/* O3: closed form of one output pixel (default taps), brute force          */
/* ---------------------------------------------------------------------- */

/* Output (R, C) of a plane lies in V repetition g = R/4 at pattern slot
 * k = R%4 and H repetition p = C/3 at slot j = C%3.  Its two V taps are the
 * mid rows 9g+a_k, 9g+a_k+1 (a = 0,2,5,7) with weights wv_k; each
 * mid value is the H output j of packet p on that row, whose two taps are
 * columns 8p+b_j, 8p+b_j+1 (b = 0,3,6) with weights wh_j. */
int orc_pixel(const uint8_t* plane, int32_t W, int32_t H, int32_t R, int32_t C) {
    static const int a[4] = { 0, 2, 5, 7 };
    static const int wv[4][2] = { {3, 5}, {1, 7}, {7, 1}, {5, 3} };
    static const int b[3] = { 0, 3, 6 };
    static const int wh[3][2] = { {1, 5}, {3, 3}, {5, 1} };
    if (!plane || W % 8 || H % 9) return ORC_ESHAPE;
    if (R < 0 || C < 0 || R >= H / 9 * 4 || C >= W / 8 * 3) return ORC_EINVAL;
    int g = R / 4, k = R % 4, p = C / 3, j = C % 3;
    int m[2];
    for (int t = 0; t < 2; ++t) {
        int64_t row = 9 * g + a[k] + t;
        const uint8_t* rp = plane + row * W + 8 * p + b[j];
        m[t] = (wh[j][0] * rp[0] + wh[j][1] * rp[1] + 3) / 6;
    }
    return (wv[k][0] * m[0] + wv[k][1] * m[1] + 4) / 8;
}
