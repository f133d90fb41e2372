/*
 * mns_oracle.c -- CPU ORACLE (test infrastructure only; never shipped, never on the product path).
 *
 * A literal fp64 restatement of the reference `mnscodec` hot path
 * (/root/reference/pkg/src/mnscodec, pure Python + numpy) used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference arm
 * as the checker.  Every numeric step follows the reference's own float64
 * evaluation order so that results are bit-identical to it:
 *
 *   - numpy elementwise expressions are evaluated left to right with no FMA
 *     contraction (built with -ffp-contract=off);
 *   - numpy mean / add.reduce use numpy's pairwise summation
 *     (`pw_sum`, restating numpy's pairwise_sum for float64: n<8 sequential,
 *     n<=128 eight strided partial sums, else split at n/2 rounded down to a
 *     multiple of 8);
 *   - BLAS dot products (`d0 @ d0`, `pool @ v`) only ever see exactly
 *     representable dyadic partial sums, so any summation order is exact.
 *
 * Pinned against the reference itself through tests/golden/ (fixtures made
 * by oracle/gen_golden.py, which imports /root/reference in the build
 * container).
 *
 * Image inputs are already padded (pad_to_multiple, image.py:123-132, is done
 * by the Python wrapper with numpy's edge mode).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../include/mns_record.h"

#define EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------ helpers */

static inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* numpy pairwise_sum_DOUBLE (numpy/_core/src/umath/loops_utils.h.src) restated. */
static double pw_sum(const double *a, long n) {
    if (n < 8) {
        double res = 0.0;
        for (long i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        long i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        long n2 = n / 2;
        n2 -= n2 % 8;
        return pw_sum(a, n2) + pw_sum(a + n2, n - n2);
    }
}

/* image.py:174-187 co_domain_rect: origin of the 2*size domain sharing the range centre. */
static inline void co_domain(int x, int y, int size, int W, int H, int *dx, int *dy) {
    int d = 2 * size;
    *dx = clampi(x - size / 2, 0, W - d);
    *dy = clampi(y - size / 2, 0, H - d);
}

/* image.py:160-171 downsample_mean2 on a uint8 raster:
 * (a[0::2,0::2] + a[0::2,1::2] + a[1::2,0::2] + a[1::2,1::2]) * 0.25, row-major output. */
static void downsample_u8(const uint8_t *img, int W, int dx, int dy, int size, double *out) {
    for (int i = 0; i < size; i++)
        for (int j = 0; j < size; j++) {
            const uint8_t *p = img + (size_t)(dy + 2 * i) * W + (dx + 2 * j);
            double a = p[0], b = p[1], c = p[W], d = p[W + 1];
            out[i * size + j] = (((a + b) + c) + d) * 0.25;
        }
}

static void downsample_f64(const double *img, int W, int dx, int dy, int size, double *out) {
    for (int i = 0; i < size; i++)
        for (int j = 0; j < size; j++) {
            const double *p = img + (size_t)(dy + 2 * i) * W + (dx + 2 * j);
            out[i * size + j] = (((p[0] + p[1]) + p[W]) + p[W + 1]) * 0.25;
        }
}

/* image.py:146-150 block_pixels */
static void block_u8(const uint8_t *img, int W, int x, int y, int size, double *out) {
    for (int i = 0; i < size; i++)
        for (int j = 0; j < size; j++) out[i * size + j] = img[(size_t)(y + i) * W + (x + j)];
}

/* transform.py:46-53 quantize_contrast */
static int quantize_contrast(double s) {
    double c = s < -1.0 ? -1.0 : (s > 1.0 ? 1.0 : s);
    int k = (int)floor((c + 1.0) * 4.0);
    return k < 7 ? k : 7;
}

/* transform.py:56-60 dequantize_contrast */
static inline double dequantize_contrast(int code) { return -0.875 + 0.25 * code; }

/* encoder.py:47-49 round_to_int */
static inline int round_to_int(double v) { return (int)floor(v + 0.5); }

/* transform.py:23-43 fit_affine -> s (o = r.mean() is returned through *o). */
static double fit_affine_s(const double *r, const double *d, int n, double *o_out) {
    double o = pw_sum(r, n) / n;
    double dm = pw_sum(d, n) / n;
    double denom = 0.0, num = 0.0;
    for (int i = 0; i < n; i++) {
        double d0 = d[i] - dm;
        denom += d0 * d0; /* exact: dyadic partial sums */
    }
    *o_out = o;
    if (denom == 0.0) return 0.0;
    for (int i = 0; i < n; i++) num += (d[i] - dm) * (r[i] - o); /* exact */
    return num / denom;
}

/* transform.py:69-80 rms_error: sqrt(mean((r - (s*(d - d.mean()) + o))**2)). */
static double rms_error(const double *r, const double *d, int n, double s, double o) {
    double sq[256];
    double dm = pw_sum(d, n) / n;
    for (int i = 0; i < n; i++) {
        double t = s * (d[i] - dm);
        double u = t + o;
        double res = r[i] - u;
        sq[i] = res * res;
    }
    return sqrt(pw_sum(sq, n) / n);
}

/* ------------------------------------------------------------ MNS encoder */

typedef struct {
    double e[3];      /* e1, e2, e3 (encoder.py:56-58) */
    double mean_tol;  /* encoder.py:59 */
    int mns;          /* mode == "mns" (1) or "no_search" (0) */
    int root_level;   /* 1 = reference driver; 2 = "8->4" extension: roots forced to split once */
    int n_iso;        /* 0 / 1 = the reference; 8 = extension: phase 1 also tries the 8 isometries */
} orc_enc_cfg;

static const double CONTRAST_SETS[4][2] = {{0, 0}, {0.2, 0.5}, {0.4, 0.65}, {0.5, 0.9}}; /* encoder.py:36 */
static const int DELTA_LIMIT[4] = {0, 15, 31, 31};                                   /* encoder.py:39-44 */

static inline int iso_src(int t, int i, int j, int B);

/* encoder.py:145-166 try_phase1.  Isometry extension (cfg->n_iso = 8): the same fit on each
 * d_t(i, j) = d(src_t(i, j)), the first smallest rms wins (strict '<' over t), t goes in the record. */
static int try_phase1(const uint8_t *img, int W, int H, int x, int y, int size, int level, const orc_enc_cfg *cfg,
                      uint64_t *rec, double *rms_out) {
    double d[256], dt[256], r[256], o;
    int dx, dy, n = size * size, n_iso = cfg->n_iso > 1 ? cfg->n_iso : 1;
    co_domain(x, y, size, W, H, &dx, &dy);
    downsample_u8(img, W, dx, dy, size, d);
    block_u8(img, W, x, y, size, r);
    double best = INFINITY;
    int bcode = 0, bob = 0, bt = 0;
    for (int t = 0; t < n_iso; t++) {
        for (int k = 0; k < n; k++) dt[k] = t ? d[iso_src(t, k / size, k % size, size)] : d[k];
        double s = fit_affine_s(r, dt, n, &o);
        int code = quantize_contrast(s);
        int ob = round_to_int(o);
        double rms = rms_error(r, dt, n, dequantize_contrast(code), (double)ob);
        if (rms < best || t == 0) {
            best = rms;
            bcode = code;
            bob = ob;
            bt = t;
        }
    }
    if (rms_out) *rms_out = best;
    if (level == 4 || best <= cfg->e[level - 1]) {
        *rec = mns_rec_phase1(x, y, level, bob, bcode) | ((uint64_t)bt << MNS_REC_ISO_SHIFT);
        return 1;
    }
    return 0;
}

static double block_mean_u8(const uint8_t *img, int W, int x, int y, int size) {
    double r[256];
    block_u8(img, W, x, y, size, r);
    return pw_sum(r, size * size) / (size * size);
}

/* encoder.py:169-212 try_phase2 */
static int try_phase2(const uint8_t *img, int W, int H, int x, int y, int size, int level, const orc_enc_cfg *cfg,
                      uint64_t *rec, double *rms_out) {
    int h = size / 2;
    int qx[4] = {x, x + h, x, x + h}, qy[4] = {y, y, y + h, y + h}; /* image.py:25-33 TL,TR,BL,BR */
    double o_mean = block_mean_u8(img, W, x, y, size);
    double qm[4];
    double worst_gap = 0.0;
    for (int k = 0; k < 4; k++) {
        qm[k] = block_mean_u8(img, W, qx[k], qy[k], h);
        double g = fabs(qm[k] - o_mean);
        if (g > worst_gap) worst_gap = g;
    }
    if (rms_out) *rms_out = INFINITY;
    if (worst_gap > cfg->mean_tol) return 0;
    int ob = round_to_int(o_mean);
    int dl[3];
    for (int k = 0; k < 3; k++) dl[k] = round_to_int(qm[k] - o_mean);
    for (int k = 0; k < 3; k++)
        if (abs(dl[k]) > DELTA_LIMIT[level]) return 0;
    int implied = ob - (dl[0] + dl[1] + dl[2]);
    if (implied < 0 || implied > 255) return 0;
    int targets[4] = {ob + dl[0], ob + dl[1], ob + dl[2], implied};
    double s_lo = CONTRAST_SETS[level][0], s_hi = CONTRAST_SETS[level][1];
    double tol = cfg->e[level - 1];
    int bits = 0;
    double worst = 0.0;
    for (int k = 0; k < 4; k++) {
        double d[64], r[64];
        int dx, dy;
        co_domain(qx[k], qy[k], h, W, H, &dx, &dy);
        downsample_u8(img, W, dx, dy, h, d);
        block_u8(img, W, qx[k], qy[k], h, r);
        double rlo = rms_error(r, d, h * h, s_lo, (double)targets[k]);
        double rhi = rms_error(r, d, h * h, s_hi, (double)targets[k]);
        int bit = rlo <= rhi ? 0 : 1;
        double rms = bit ? rhi : rlo;
        if (rms > tol) return 0;
        bits |= bit << k;
        if (rms > worst) worst = rms;
    }
    if (rms_out) *rms_out = worst;
    *rec = mns_rec_phase2(x, y, level, ob, dl[0], dl[1], dl[2], bits);
    return 1;
}

typedef struct {
    const uint8_t *img;
    int W, H, min_dim;
    const orc_enc_cfg *cfg;
    uint64_t *out;
    int count;
} visit_ctx;

/* encoder.py:229-239 visit */
static void visit(visit_ctx *c, int x, int y, int size, int level) {
    uint64_t rec;
    int ok = 0;
    if (2 * size <= c->min_dim) {
        ok = try_phase1(c->img, c->W, c->H, x, y, size, level, c->cfg, &rec, NULL);
        if (!ok && c->cfg->mns) ok = try_phase2(c->img, c->W, c->H, x, y, size, level, c->cfg, &rec, NULL);
    }
    if (ok) {
        c->out[c->count++] = rec;
        return;
    }
    int h = size / 2;
    visit(c, x, y, h, level + 1);
    visit(c, x + h, y, h, level + 1);
    visit(c, x, y + h, h, level + 1);
    visit(c, x + h, y + h, h, level + 1);
}

/* encoder.py:215-246 encode_quadtree over an already padded raster (W, H multiples of 16).
 * Roots in raster order; records in DFS order.  root_counts (optional, n_roots entries)
 * receives the per-root leaf counts.  Returns the number of records, or -1 if cap is too small. */
EXPORT int64_t orc_encode_quadtree(const uint8_t *img, int W, int H, const orc_enc_cfg *cfg, uint64_t *out,
                                   int64_t cap, int32_t *root_counts, int nthreads) {
    int rw = W / 16, rh = H / 16;
    int64_t nroots = (int64_t)rw * rh;
    int32_t *counts = (int32_t *)malloc(sizeof(int32_t) * (size_t)nroots);
    int min_dim = W < H ? W : H;
    int64_t total = 0;
    if (nthreads < 1) nthreads = 1;
    /* Batches of root rows are encoded in parallel into a scratch of 64 records per root
     * (a root holds at most 64 leaves), then appended in raster order. */
    int rows_per_batch = (int)((1 << 22) / (64 * (int64_t)rw));
    if (rows_per_batch < 1) rows_per_batch = 1;
    if (rows_per_batch > rh) rows_per_batch = rh;
    uint64_t *scratch = (uint64_t *)malloc(sizeof(uint64_t) * 64 * (size_t)rw * rows_per_batch);
    for (int r0 = 0; r0 < rh; r0 += rows_per_batch) {
        int r1 = r0 + rows_per_batch < rh ? r0 + rows_per_batch : rh;
        int64_t nb = (int64_t)(r1 - r0) * rw;
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads)
        for (int64_t i = 0; i < nb; i++) {
            int64_t root = (int64_t)r0 * rw + i;
            int ry = (int)(root / rw), rx = (int)(root % rw);
            visit_ctx c = {img, W, H, min_dim, cfg, scratch + 64 * i, 0};
            if (cfg->root_level <= 1) {
                visit(&c, rx * 16, ry * 16, 16, 1);
            } else {
                visit(&c, rx * 16, ry * 16, 8, 2);
                visit(&c, rx * 16 + 8, ry * 16, 8, 2);
                visit(&c, rx * 16, ry * 16 + 8, 8, 2);
                visit(&c, rx * 16 + 8, ry * 16 + 8, 8, 2);
            }
            counts[root] = c.count;
        }
        for (int64_t i = 0; i < nb; i++) {
            int64_t root = (int64_t)r0 * rw + i;
            int cnt = counts[root];
            if (total + cnt > cap) {
                free(counts);
                free(scratch);
                return -1;
            }
            memcpy(out + total, scratch + 64 * i, sizeof(uint64_t) * cnt);
            total += cnt;
        }
    }
    if (root_counts) memcpy(root_counts, counts, sizeof(int32_t) * (size_t)nroots);
    free(counts);
    free(scratch);
    return total;
}

/* Single-node entry points (try_phase1 / try_phase2 parity).  Return 1 with *rec set on accept. */
EXPORT int orc_try_phase1(const uint8_t *img, int W, int H, int x, int y, int size, int level,
                          const orc_enc_cfg *cfg, uint64_t *rec, double *rms) {
    return try_phase1(img, W, H, x, y, size, level, cfg, rec, rms);
}
EXPORT int orc_try_phase2(const uint8_t *img, int W, int H, int x, int y, int size, int level,
                          const orc_enc_cfg *cfg, uint64_t *rec, double *rms) {
    return try_phase2(img, W, H, x, y, size, level, cfg, rec, rms);
}

/* ------------------------------------------------------------------ decoder */

/* One painted unit: destination square, domain origin (domain side = 2*size), map (s, o). */
typedef struct {
    int32_t x, y, size, dx, dy;
    double s, o;
} orc_unit;

/* decoder.py:48-62: expand transform-code records into painted units
 * (1 per phase-1 leaf, 4 per phase-2 leaf).  Returns unit count. */
EXPORT int64_t orc_records_to_units(const uint64_t *rec, int64_t n, int W, int H, orc_unit *u) {
    int64_t k = 0;
    for (int64_t i = 0; i < n; i++) {
        uint64_t r = rec[i];
        int x = (int)((r >> MNS_REC_X_SHIFT) & 0x7FFF) * 2, y = (int)((r >> MNS_REC_Y_SHIFT) & 0x7FFF) * 2;
        int level = (int)((r >> MNS_REC_LEVEL_SHIFT) & 3) + 1;
        int size = 32 >> level;
        int ob = (int)((r >> MNS_REC_O_SHIFT) & 0xFF);
        if (!((r >> MNS_REC_PHASE2_SHIFT) & 1)) {
            int code = (int)((r >> MNS_REC_PAYLOAD_SHIFT) & 7), iso = (int)((r >> MNS_REC_ISO_SHIFT) & 7);
            orc_unit v = {x, y, size | (iso << 8), 0, 0, dequantize_contrast(code), (double)ob};  /* side | iso << 8 */
            co_domain(x, y, size, W, H, &v.dx, &v.dy);
            u[k++] = v;
        } else {
            int d[3];
            for (int j = 0; j < 3; j++) {
                int f = (int)((r >> (41 + 6 * j)) & 63);
                d[j] = f >= 32 ? f - 64 : f;
            }
            int bits = (int)((r >> 59) & 15);
            int targets[4] = {ob + d[0], ob + d[1], ob + d[2], ob - (d[0] + d[1] + d[2])};
            int h = size / 2;
            int qx[4] = {x, x + h, x, x + h}, qy[4] = {y, y, y + h, y + h};
            for (int q = 0; q < 4; q++) {
                orc_unit v = {qx[q], qy[q], h, 0, 0, CONTRAST_SETS[level][(bits >> q) & 1], (double)targets[q]};
                co_domain(qx[q], qy[q], h, W, H, &v.dx, &v.dy);
                u[k++] = v;
            }
        }
    }
    return k;
}

/* decoder.py:32-34 _paint + transform.py:63-66 apply_map */
static void paint(double *out, const double *cur, int W, const orc_unit *u) {
    double d0[256], d[256] = {0};
    int size = u->size & 255, iso = u->size >> 8, n = size * size; /* size = side | isometry << 8 */
    downsample_f64(cur, W, u->dx, u->dy, size, d0);
    /* isometry extension: the transformed domain d_t(i, j) = d(src_t(i, j)), then apply_map on it */
    for (int k = 0; k < n; k++) d[k] = iso ? d0[iso_src(iso, k / size, k % size, size)] : d0[k];
    double dm = pw_sum(d, n) / n;
    for (int i = 0; i < size; i++)
        for (int j = 0; j < size; j++) {
            double v = u->s * (d[i * size + j] - dm) + u->o;
            v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
            out[(size_t)(u->y + i) * W + (u->x + j)] = v;
        }
}

/* decoder.py:37-63 decode_step: one Jacobi sweep cur -> out. */
EXPORT void orc_decode_step(const orc_unit *u, int64_t nu, int W, int H, const double *cur, double *out,
                            int nthreads) {
    (void)H;
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (int64_t i = 0; i < nu; i++) paint(out, cur, W, &u[i]);
}

/* decoder.py:66-77 decode: flat start, <= max_iters sweeps, early stop on max|delta| < stop_delta,
 * clip(floor(x + 0.5)) -> uint8 over the padded raster (caller crops).  raster (W*H doubles,
 * optional) receives the final float raster.  Returns sweeps run. */
EXPORT int orc_decode(const orc_unit *u, int64_t nu, int W, int H, int max_iters, double stop_delta,
                      double initial_value, uint8_t *out_u8, double *raster, int nthreads) {
    size_t np_ = (size_t)W * H;
    double *cur = (double *)malloc(sizeof(double) * np_);
    double *nxt = (double *)malloc(sizeof(double) * np_);
    int it = 0;
    if (nthreads < 1) nthreads = 1;
    for (size_t i = 0; i < np_; i++) cur[i] = initial_value;
    for (it = 0; it < max_iters;) {
        orc_decode_step(u, nu, W, H, cur, nxt, nthreads);
        double delta = 0.0;
#pragma omp parallel for reduction(max : delta) num_threads(nthreads)
        for (size_t i = 0; i < np_; i++) {
            double g = fabs(nxt[i] - cur[i]);
            if (g > delta) delta = g;
        }
        double *t = cur;
        cur = nxt;
        nxt = t;
        it++;
        if (delta < stop_delta) break;
    }
    for (size_t i = 0; i < np_; i++) {
        double v = floor(cur[i] + 0.5);
        v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
        out_u8[i] = (uint8_t)v;
    }
    if (raster) memcpy(raster, cur, sizeof(double) * np_);
    free(cur);
    free(nxt);
    return it;
}

/* ------------------------------------------------------- search baselines */

/* Isometry t of a B x B block (extension; the reference has none):
 * d_t(i, j) = d(src_t(i, j)).  t = 0 is the identity (the reference's only map). */
static inline int iso_src(int t, int i, int j, int B) {
    switch (t) {
    case 0: return i * B + j;                         /* identity            */
    case 1: return i * B + (B - 1 - j);               /* mirror columns      */
    case 2: return (B - 1 - i) * B + j;               /* mirror rows         */
    case 3: return (B - 1 - i) * B + (B - 1 - j);     /* rotate 180          */
    case 4: return j * B + i;                         /* transpose           */
    case 5: return (B - 1 - j) * B + i;               /* rotate 90 clockwise */
    case 6: return j * B + (B - 1 - i);               /* rotate 90 ccw       */
    default: return (B - 1 - j) * B + (B - 1 - i);    /* anti-transpose      */
    }
}

/* encoder.py:249-309 encode_full_search restated for a subset of ranges (range ids in raster
 * order over the B-padded raster).  Domain pool: every 2B x 2B block on a stride-`step`
 * lattice, raster order.  n_iso = 1 reproduces the reference; n_iso = 8 extends the pool with
 * isometries (index order: domain-major, then isometry), ties to the lowest (domain, iso).
 * Outputs per listed range: domain index, isometry, o_byte, s_code. */
EXPORT int orc_full_search(const uint8_t *img, int W, int H, int B, int step, int n_iso, const int32_t *range_ids,
                           int64_t n_ranges, int32_t *out_dom, int8_t *out_iso, uint8_t *out_o, uint8_t *out_code,
                           int nthreads) {
    int D2 = 2 * B, n = B * B;
    int ndx = (W - D2) / step + 1, ndy = (H - D2) / step + 1;
    int64_t ndom = (int64_t)ndx * ndy;
    /* pool[k][dom] (k-major so the per-range sweep vectorises across domains without
     * reassociating any single dot product; all partial sums are exact anyway). */
    double *pool = (double *)malloc(sizeof(double) * (size_t)n * ndom);
    double *denom = (double *)malloc(sizeof(double) * ndom);
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (int64_t dI = 0; dI < ndom; dI++) {
        int x = (int)(dI % ndx) * step, y = (int)(dI / ndx) * step;
        double v[256], acc = 0.0;
        /* sums2 = a[:-1,:-1] + a[:-1,1:] + a[1:,:-1] + a[1:,1:]; pool row = sums2[y::2, x::2] * 0.25 */
        for (int i = 0; i < B; i++)
            for (int j = 0; j < B; j++) {
                const uint8_t *p = img + (size_t)(y + 2 * i) * W + (x + 2 * j);
                double a = p[0], b = p[1], c = p[W], d = p[W + 1];
                v[i * B + j] = (((a + b) + c) + d) * 0.25;
            }
        double m = pw_sum(v, n) / n; /* pool.mean(axis=1): exact (quarter-integer sums) */
        for (int k = 0; k < n; k++) {
            double p0 = v[k] - m;
            pool[(size_t)k * ndom + dI] = p0;
            acc += p0 * p0; /* einsum: exact */
        }
        denom[dI] = acc;
    }
#pragma omp parallel num_threads(nthreads)
    {
        double *cross = (double *)malloc(sizeof(double) * ndom);
#pragma omp for schedule(dynamic, 1)
        for (int64_t ri = 0; ri < n_ranges; ri++) {
            int rid = range_ids[ri];
            int rpr = W / B;
            int rx = (rid % rpr) * B, ry = (rid / rpr) * B;
            double r[256], rc[256], rr = 0.0;
            block_u8(img, W, rx, ry, B, r);
            double rmean = pw_sum(r, n) / n;
            int ob = round_to_int(rmean);
            for (int k = 0; k < n; k++) {
                double t = r[k] - (double)ob;
                rr += t * t; /* rr @ rr: exact */
            }
            double best = INFINITY;
            int64_t best_idx = 0;
            int best_code = 0;
            for (int t = 0; t < n_iso; t++) {
                /* cross_t[dom] = sum_k pool_t[dom][k] (r_k - mean r) with pool_t[dom][k] = pool[dom][src_t(k)];
                 * evaluated as sum_m pool[dom][m] rc[inv_t(m)] -- exact, so the order is immaterial. */
                for (int k = 0; k < n; k++) rc[iso_src(t, k / B, k % B, B)] = r[k] - rmean;
                for (int64_t dI = 0; dI < ndom; dI++) cross[dI] = 0.0;
                for (int k = 0; k < n; k++) {
                    const double *pk = pool + (size_t)k * ndom;
                    double c = rc[k];
                    for (int64_t dI = 0; dI < ndom; dI++) cross[dI] += pk[dI] * c;
                }
                for (int64_t dI = 0; dI < ndom; dI++) {
                    double dn = denom[dI];
                    double code;
                    if (dn > 0.0) {
                        double s = cross[dI] / dn;
                        s = s < -1.0 ? -1.0 : (s > 1.0 ? 1.0 : s);
                        code = floor((s + 1.0) * 4.0);
                        if (code > 7.0) code = 7.0;
                    } else {
                        code = 4.0;
                    }
                    double sq = -0.875 + 0.25 * code;
                    double sse = rr - 2.0 * sq * cross[dI] + sq * sq * dn;
                    int64_t idx = dI * n_iso + t;
                    if (sse < best || (sse == best && idx < best_idx)) {
                        best = sse;
                        best_idx = idx;
                        best_code = (int)code;
                    }
                }
            }
            out_dom[ri] = (int32_t)(best_idx / n_iso);
            out_iso[ri] = (int8_t)(best_idx % n_iso);
            out_o[ri] = (uint8_t)ob;
            out_code[ri] = (uint8_t)best_code;
        }
        free(cross);
    }
    free(pool);
    free(denom);
    return 0;
}

/* encoder.py:312-347 encode_local_search restated with a radius parameter (reference: 4 ->
 * 81 candidates; radius 32 is the extension) and an isometry count (reference: 1; 8 is the
 * extension: candidate t of a domain is d_t(i,j) = d(src_t(i,j)), as in orc_full_search).  Over the
 * 8-padded raster, 8x8 ranges in raster order; candidates = co-centred 16x16 domain translated by
 * (dy, dx) in [-R, R]^2, dy outer, each clamped, then the isometries; strict '<' keeps the first
 * best.  Outputs per range: domain x, y, isometry, o, code. */
EXPORT int orc_local_search(const uint8_t *img, int W, int H, int radius, int n_iso, int32_t *out_dx,
                            int32_t *out_dy, int8_t *out_iso, uint8_t *out_o, uint8_t *out_code, int nthreads) {
    int rpr = W / 8;
    int64_t nr = (int64_t)rpr * (H / 8);
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 4) num_threads(nthreads)
    for (int64_t ri = 0; ri < nr; ri++) {
        int rx = (int)(ri % rpr) * 8, ry = (int)(ri / rpr) * 8;
        double r[64], d[64], dt[64], o_fit;
        block_u8(img, W, rx, ry, 8, r);
        int bx, by;
        co_domain(rx, ry, 8, W, H, &bx, &by);
        int ob = round_to_int(pw_sum(r, 64) / 64);
        double best_rms = INFINITY;
        int best_x = bx, best_y = by, best_code = 0, best_t = 0;
        for (int dy = -radius; dy <= radius; dy++)
            for (int dx = -radius; dx <= radius; dx++) {
                int cx = clampi(bx + dx, 0, W - 16), cy = clampi(by + dy, 0, H - 16);
                downsample_u8(img, W, cx, cy, 8, d);
                for (int t = 0; t < n_iso; t++) {
                    for (int k = 0; k < 64; k++) dt[k] = d[iso_src(t, k / 8, k % 8, 8)];
                    int code = quantize_contrast(fit_affine_s(r, dt, 64, &o_fit));
                    double rms = rms_error(r, dt, 64, dequantize_contrast(code), (double)ob);
                    if (rms < best_rms) {
                        best_rms = rms;
                        best_x = cx;
                        best_y = cy;
                        best_code = code;
                        best_t = t;
                    }
                }
            }
        out_dx[ri] = best_x;
        out_dy[ri] = best_y;
        out_iso[ri] = (int8_t)best_t;
        out_o[ri] = (uint8_t)ob;
        out_code[ri] = (uint8_t)best_code;
    }
    return 0;
}
