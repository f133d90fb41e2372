// MNS quadtree encoder for sm_100a: block moments (K1) + phase-1/phase-2 matcher
// + per-root DFS emission (K2) in one kernel, then a scan + compaction kernel.
//
// Replaces the reference's per-node Python recursion
//   encoder.py:215-246 encode_quadtree / visit, :145-166 try_phase1,
//   :169-212 try_phase2, image.py:146-187 block helpers, transform.py:23-80.
//
// Work decomposition: one CTA = up to TR = 32 consecutive 16x16 roots of one root
// row (warp w owns roots w, w + 8, w + 16, w + 24: two per half-warp per step).  The CTA stages the uint8 window
// [x0-16, x0+16*TR+16) x [y0-16, y0+32) (every clamped domain of every node of its roots lies inside,
// SURVEY 7 "geometry") with 16-byte coalesced loads, and builds the table of
// even-phase 2x2 pixel sums q (0..1020, u16) with packed SIMD-in-register adds.
// Levels 1-3 read q from that table (their domain origins are always even);
// level 4 (odd phase, 2x2 ranges) sums its 4 pixels directly.
//
// Exactness (SURVEY 0 "exactness findings"):
//   phase 1  -- integer moments Sr, Srr, Sq, Sqq, Sqr; code from floor(16N/D);
//               1024*n*SSE = 1024nA - 64 k2 N + k2^2 D exactly; accept iff that
//               integer <= bound(E)*1024n^2 (bound = largest double whose sqrt <= E).
//   phase 2  -- gate/o/deltas/implied in integers; each quadrant's two candidate
//               SSEs from moments in fp64 with a rigorous margin; only inside the
//               margin (near-ties, near-threshold) is the reference's per-element
//               fp64 evaluation emulated bit-exactly (no FMA, numpy pairwise sum).
// Emission: leaves are keyed by the Morton index of their top-left 2x2 cell
//   (= reference DFS order TL,TR,BL,BR); lane l owns cells 2l, 2l+1, so a warp
//   compacts its root with two ballots into the root's 64 staged slots;
//   compact_records_kernel scans the per-root counts (decoupled look-back over
//   uniform tiles) and copies the records to their final offsets.

#include <math.h>

#include <climits>

#include "mns_common.cuh"
#include "mns_tma.cuh"

namespace mns {
namespace {

constexpr unsigned FULL = 0xffffffffu;
#ifndef ENC_MINB
#define ENC_MINB 3
#endif
#ifndef ENC_RPW
#define ENC_RPW 2
#endif
constexpr int EW = 8;                // warps per CTA
constexpr int ET = EW * 32;
constexpr int RPW = ENC_RPW;         // roots per half-warp per step (2: half the per-step barriers per root;
                                     // c5 encode 0.632 -> 0.605 ms with 3 CTAs/SM, 85 registers)
constexpr int TR = 2 * EW * RPW;     // consecutive roots of one root row per step
constexpr int WIN_W = TR * 16 + 32;  // pixel columns: [x0 - 16, x0 + 16 TR + 16)
constexpr int TMA_E = WIN_W / 2 <= 256 ? 2 : (WIN_W / 4 <= 256 ? 4 : 8);  // TMA element bytes (box <= 256)

struct EncParams {
    int y_res0;  // first resident image row (the tensor map's row 0)
    int W, H, n_images, rr0, rows, rw, tiles_per_row, chunk_rows;
    int mns, root_level, min_dim;
    double p1b[5];  // phase-1 accept bound on 1024*n*SSE per level (inf for level 4)
    double p2b[4];  // bound(E_level): phase-2 quadrant accepts iff SSE <= n_k * p2b
    double tol[4];  // E_level (emulation path compares rms > tol like the reference)
    double mean_tol;
    int gate[4];    // phase-2 mean gate per level: |n * (O_k - O_i)| > gate  <=>  |O_k - O_i| > mean_tol
    uint64_t *stage;     // 64 record slots per root (workspace); compacted by compact_records_kernel
    uint32_t *unit_map;  // optional: decoder map (mns_record.h), 32 words per root (unit map) or 8 (block map)
    int map_form;        // 0: unit map, 1: block map
    int32_t *root_cnt;   // per-root record counts (root_offsets, scanned in place by the compaction)
    long long n_roots;
};

struct Mom {
    int sr, srr, sq, sqq, sqr;
};

// 2^-k as an exact double
__device__ __forceinline__ double pow2neg(int k) { return __longlong_as_double((long long)(1023 - k) << 52); }

// Quantised contrast code = 4 + clamp(floor(16N/D), -4, 3) (4 when D == 0): the
// reference's quantize_contrast(fl(4N/D)) (transform.py:46-53), exactly.  t = 16N and D are
// exact doubles (|16N|, 4|D| < 2^53); a fast fp32 quotient is corrected by one exact fp64
// comparison (its error is < 1 unit).
__device__ __forceinline__ int quant_code(double t, double D) {
    if (D == 0.0) return 4;  // fit_affine degenerate domain: s = 0 -> bin 4
    const float q = fminf(3.5f, fmaxf(-4.5f, __fdividef((float)t, (float)D)));
    const float f = floorf(q);
    int k = (int)f;
    // the fp32 quotient is within 1e-5 of t/D: away from an integer it already is the floor
    if (q - f < 1e-4f || q - f > 1.f - 1e-4f) {
        if (t < (double)k * D) --k;
        else if (t >= (double)(k + 1) * D) ++k;
    }
    return 4 + min(3, max(-4, k));
}

// N = n Sqr - Sq Sr and D = n Sqq - Sq^2 (one wide multiply-add each), as exact doubles
__device__ __forceinline__ double mom_N(int nlog2, const Mom &m) {  // Sq * Sr < 2^53: one exact FMA
    return fma((double)m.sqr, (double)(1 << nlog2), -((double)m.sq * (double)m.sr));
}
__device__ __forceinline__ double mom_D(int nlog2, const Mom &m) {
    return fma((double)m.sqq, (double)(1 << nlog2), -((double)m.sq * (double)m.sq));
}

// Phase 1 from exact integer moments (encoder.py:145-166 + transform.py:23-80).  Every term of
// 1024 n SSE = 1024 n A - 64 k2 N + k2^2 D is an integer below 2^53, so two fp64 FMAs give it
// exactly; an infinite bound (E = inf) accepts without it.
__device__ __forceinline__ uint64_t phase1(int x, int y, int level, int nlog2, const Mom &m, double bnd,
                                           bool &acc) {
    const int o = (2 * m.sr + (1 << nlog2)) >> (nlog2 + 1);  // round_to_int(mean)
    const double N = mom_N(nlog2, m), D = mom_D(nlog2, m);
    const int code = quant_code(16.0 * N, D);
    if (bnd == INFINITY) {
        acc = true;
    } else {
        const int k2 = 2 * code - 7;
        const int A = m.srr - 2 * o * m.sr + ((o * o) << nlog2);  // sum (r - o)^2 < 2^25
        acc = fma((double)(k2 * k2), D, fma((double)(-64 * k2), N, (double)A * (double)(1024 << nlog2))) <= bnd;
    }
    return mns_rec_phase1(x, y, level, o, code);
}

// Phase-2 quadrant decision from moments: 0 reject, 1 accept, 2 ambiguous (emulate).
__device__ __forceinline__ int p2_quad(int nlog2, const Mom &m, int t, double slo, double shi, double bnd_n,
                                       int &bit) {
    const int A = m.srr - 2 * t * m.sr + ((t * t) << nlog2);  // sum (r - t)^2 < 2^25
    const double N = mom_N(nlog2, m), D = mom_D(nlog2, m);
    bit = 0;
    if (D == 0.0) return (double)A <= bnd_n ? 1 : 0;  // d - mean(d) == 0: both candidates identical
    const double X = N * pow2neg(nlog2 + 2);  // sum (r - t)(d - dbar), exact
    const double Y = D * pow2neg(nlog2 + 4);  // sum (d - dbar)^2, exact
    const double Ad = (double)A;
    const double lo = Ad - 2.0 * slo * X + slo * slo * Y;
    const double hi = Ad - 2.0 * shi * X + shi * shi * Y;
    const double delta = 1e-5 + 1e-11 * (Ad + 2.0 * fabs(X) + Y);
    double best;
    if (lo < hi - 2.0 * delta) {
        best = lo;
    } else if (lo > hi + 2.0 * delta) {
        bit = 1;
        best = hi;
    } else {
        return 2;
    }
    if (best + delta <= bnd_n) return 1;
    if (best - delta > bnd_n) return 0;
    return 2;
}

// One squared residual exactly as numpy evaluates r - (s*(d - d.mean()) + o)
// (transform.py:79-80): no contraction, d = q*0.25, d.mean() = dm exact.
__device__ __forceinline__ double emu_sq(int r, int q, double dm, double s, double t) {
    const double e = __dsub_rn((double)q * 0.25, dm);
    const double u = __dadd_rn(__dmul_rn(s, e), t);
    const double res = __dsub_rn((double)r, u);
    return __dmul_rn(res, res);
}

struct Node2 {  // phase-2 node-level quantities (gate, o_byte, deltas, targets)
    bool pass;
    int o, d0, d1, d2, t[4];
};

// The gate compares exact dyadic means (encoder.py:187): |O_k - O_i| > mean_tol  <=>
// |n (O_k - O_i)| > mean_tol * n  <=>  |df| > floor(mean_tol * n) for the integer df (host: gate).
__device__ __forceinline__ Node2 p2_node(int nlog2, int sr, int s0, int s1, int s2, int s3, int limit, int gate) {
    Node2 z;
    const int n = 1 << nlog2;
    const int df[4] = {4 * s0 - sr, 4 * s1 - sr, 4 * s2 - sr, 4 * s3 - sr};  // n * (O_k - O_i)
    z.pass = max(max(abs(df[0]), abs(df[1])), max(abs(df[2]), abs(df[3]))) <= gate;
    z.o = (2 * sr + n) >> (nlog2 + 1);
    z.d0 = (2 * df[0] + n) >> (nlog2 + 1);  // floor((O_k - O_i) + 0.5), arithmetic shift = floor
    z.d1 = (2 * df[1] + n) >> (nlog2 + 1);
    z.d2 = (2 * df[2] + n) >> (nlog2 + 1);
    if (abs(z.d0) > limit || abs(z.d1) > limit || abs(z.d2) > limit) z.pass = false;
    const int implied = z.o - (z.d0 + z.d1 + z.d2);
    if (implied < 0 || implied > 255) z.pass = false;
    z.t[0] = z.o + z.d0;
    z.t[1] = z.o + z.d1;
    z.t[2] = z.o + z.d2;
    z.t[3] = implied;
    return z;
}

// ---- node geometry inside a 16x16 root (Morton order = reference DFS order)
__device__ __forceinline__ int node2_x(int k) { return 8 * (k & 1); }
__device__ __forceinline__ int node2_y(int k) { return 8 * (k >> 1); }
__device__ __forceinline__ int node3_x(int m) { return node2_x(m >> 2) + 4 * (m & 1); }
__device__ __forceinline__ int node3_y(int m) { return node2_y(m >> 2) + 4 * ((m >> 1) & 1); }

// A staged window in shared memory addressed by GLOBAL image coordinates: pixel row gy lives at
// window row (gy - py0) & pmask, q row gqy (q = even-phase 2x2 pixel sum) at (gqy - qy0) & qmask,
// pixel column gx at gx - wx0 and q column gqx at gqx - wx0 / 2.  The encoder's rings use masks
// (rows wrap); try_node_kernel's flat window uses mask -1.
struct Win {
    const uint8_t *pix;
    const uint16_t *qe;
    int ppitch, qpitch, pmask, qmask, py0, qy0, wx0, W, H;
    __device__ __forceinline__ int px(int gx, int gy) const { return pix[((gy - py0) & pmask) * ppitch + gx - wx0]; }
    __device__ __forceinline__ int q(int gqx, int gqy) const {
        return qe[((gqy - qy0) & qmask) * qpitch + gqx - (wx0 >> 1)];
    }
};

// q of pixel (px, py) against the co-centred domain of node (x, y, s) (image.py:174-187; global)
__device__ __forceinline__ int dom_q(const Win &w, int x, int y, int s, int px, int py) {
    const int gdx = clampi(x - s / 2, 0, w.W - 2 * s), gdy = clampi(y - s / 2, 0, w.H - 2 * s);
    const int gx = gdx + 2 * (px - x), gy = gdy + 2 * (py - y);
    if (((gx | gy) & 1) == 0) return w.q(gx >> 1, gy >> 1);
    return w.px(gx, gy) + w.px(gx + 1, gy) + w.px(gx, gy + 1) + w.px(gx + 1, gy + 1);
}

// Reference-order emulation of one phase-2 quadrant (transform.py:69-80 rms_error): the quadrant
// is the square (cx, cy, cs) (global) and its domain the co-centred one.  Returns 1 accept /
// 0 reject, the chosen bit and (rms_out) the chosen candidate's rms.
__device__ __forceinline__ int emulate_quadrant(const Win &w, int cx, int cy, int cs, int sq, int t, double slo,
                                             double shi, double tol, int &bit, double *rms_out = nullptr) {
    double lo[64], hi[64];
    const int n = cs * cs;
    const double dm = ((double)sq * 0.25) / (double)n;
    const double td = (double)t;
    for (int i = 0; i < cs; i++)
        for (int j = 0; j < cs; j++) {
            const int q = dom_q(w, cx, cy, cs, cx + j, cy + i);
            const int r = w.px(cx + j, cy + i);
            lo[i * cs + j] = emu_sq(r, q, dm, slo, td);
            hi[i * cs + j] = emu_sq(r, q, dm, shi, td);
        }
    const double rlo = __dsqrt_rn(pw_sum_dev(lo, n) / (double)n), rhi = __dsqrt_rn(pw_sum_dev(hi, n) / (double)n);
    bit = rlo <= rhi ? 0 : 1;
    if (rms_out) *rms_out = bit ? rhi : rlo;
    return ((bit ? rhi : rlo) > tol) ? 0 : 1;
}

// Phase 2 of node (nx, ny, size) at `level` (global) from its own Sr and its 4 children's
// moments (encoder.py:169-212), serially.  Returns true with *rec on acceptance.
__device__ bool phase2_node(const Win &w, const EncParams &p, int level, int nx, int ny, int size, int sr,
                            const Mom *kids, uint64_t *rec) {
    const int nlog2 = 2 * (5 - level);  // node pixels: 256, 64, 16
    const Node2 z = p2_node(nlog2, sr, kids[0].sr, kids[1].sr, kids[2].sr, kids[3].sr, level == 1 ? 15 : 31,
                            p.gate[level]);
    if (!z.pass) return false;
    const double slo = level == 1 ? 0.2 : (level == 2 ? 0.4 : 0.5);
    const double shi = level == 1 ? 0.5 : (level == 2 ? 0.65 : 0.9);
    const int h = size / 2;
    const double bnd_n = p.p2b[level] * (double)(h * h);
    int bits = 0;
    for (int k = 0; k < 4; k++) {
        int bit;
        int res = p2_quad(nlog2 - 2, kids[k], z.t[k], slo, shi, bnd_n, bit);
        if (res == 2)
            res = emulate_quadrant(w, nx + (k & 1) * h, ny + (k >> 1) * h, h, kids[k].sq, z.t[k], slo, shi,
                                   p.tol[level], bit);
        if (res != 1) return false;
        bits |= bit << k;
    }
    *rec = mns_rec_phase2(nx, ny, level, z.o, z.d0, z.d1, z.d2, bits);
    return true;
}

// A sure rejection: the node's best fit with FREE contrast and offset (least squares), whose
// SSE_min = (Dr D - N^2) / (n D) (Dr = n Srr - Sr^2, D = n Sqq - Sq^2, N = n Sqr - Sq Sr; D = 0:
// SSE_min = Dr / n), already exceeds bound * n.  The quantised phase-1 fit and every phase-2
// candidate (fixed luminance, a contrast from the set) are special cases of that fit, so their SSE
// is >= SSE_min.  bn2 = bound * n^2 (inf never rejects).  Levels 2-4 (n <= 64): Dr and D are exact
// 32-bit integers and N one correctly rounded FMA, so each input carries one fp32 rounding; level 1
// also rounds n Sqq and n Sqr, whose absolute errors enter the margin (`extra`).  The margin is
// 16x the worst rounding error, so "true" is never wrong.
template <int NL>
struct FitGap {  // a = Dr D, b = N^2, d = D and the rounding scales of surely_above
    float a, b, d, dr, extra_s, extra_n;
    bool d0;
};

template <int NL>
__device__ __forceinline__ FitGap<NL> fit_gap(const Mom &m) {
    FitGap<NL> g;
    g.extra_s = 0.f;
    g.extra_n = 0.f;
    if (NL <= 6) {
        g.dr = (float)((m.srr << NL) - m.sr * m.sr);
        const unsigned du = ((unsigned)m.sqq << NL) - (unsigned)m.sq * (unsigned)m.sq;
        g.d = (float)du;
        g.d0 = du == 0u;
        const float nn = fmaf(-(float)m.sq, (float)m.sr, (float)(m.sqr << NL));
        g.b = nn * nn;
    } else {
        g.dr = (float)(((unsigned)m.srr << NL) - (unsigned)m.sr * (unsigned)m.sr);
        const float S = (float)m.sqq * (float)(1 << NL), T = (float)m.sqr * (float)(1 << NL);
        g.d = fmaf(-(float)m.sq, (float)m.sq, S);
        g.d0 = false;
        const float nn = fmaf(-(float)m.sq, (float)m.sr, T);
        g.b = nn * nn;
        g.extra_s = S;
        g.extra_n = fabsf(nn) * T;
    }
    g.a = g.dr * g.d;
    return g;
}

template <int NL>
__device__ __forceinline__ bool surely_above(const FitGap<NL> &g, float bn2) {
    if (NL <= 6 && g.d0) return g.dr > bn2 * (1.f + 1.f / 1048576.f);
    const float c = bn2 * g.d;
    const float extra = NL <= 6 ? 0.f : (g.dr + bn2) * g.extra_s + g.extra_n;
    return g.a - g.b - c > (g.a + g.b + c + extra) * (1.f / 1048576.f);
}

template <int NL>
__device__ __forceinline__ bool surely_above(const Mom &m, float bn2) {
    return surely_above<NL>(fit_gap<NL>(m), bn2);
}

// The phase-2 mean gate (encoder.py:186-188) fails: some quadrant mean is farther than mean_tol from
// the block mean (integer form of p2_node's test).
__device__ __forceinline__ bool gate_fails(int nlog2, int sr, const int *ks, int gate) {
    (void)nlog2;
    const int d = max(max(abs(4 * ks[0] - sr), abs(4 * ks[1] - sr)), max(abs(4 * ks[2] - sr), abs(4 * ks[3] - sr)));
    return d > gate;
}

// Phase 1 + phase 2 of one level-1/2 node (global (nx, ny)) with its 4 quadrant tests on 4 lanes of
// the warp: this lane tests quadrant `quad` (moments `kid`) when is_quad; ks = the 4 children's
// Sr; gather(ballot) extracts the node's 4 quadrant bits.  Same decisions as phase1 / phase2_node.
// Every lane of the warp must call it (ballots); the result lands on every lane of the node.
template <class Gather>
__device__ __forceinline__ void node_decide(const Win &w, const EncParams &p, bool active, bool is_quad, int quad,
                                            int level, int nx, int ny, const Mom &m, const int *ks, const Mom &kid,
                                            Gather gather, bool &acc, uint64_t &rec) {
    const int size = 32 >> level, nlog2 = 2 * (5 - level);
    acc = false;
    rec = 0;
    bool want2 = false, ok = false;
    int bit = 0;
    Node2 z{};
    if (active) {
        rec = phase1(nx, ny, level, nlog2, m, p.p1b[level], acc);
        if (!acc && p.mns) {
            z = p2_node(nlog2, m.sr, ks[0], ks[1], ks[2], ks[3], level == 1 ? 15 : 31, p.gate[level]);
            want2 = z.pass;
            if (want2 && is_quad) {
                const double slo = level == 1 ? 0.2 : 0.4, shi = level == 1 ? 0.5 : 0.65;
                const int h = size / 2;
                int res = p2_quad(nlog2 - 2, kid, z.t[quad], slo, shi, p.p2b[level] * (double)(h * h), bit);
                if (res == 2)
                    res = emulate_quadrant(w, nx + (quad & 1) * h, ny + (quad >> 1) * h, h, kid.sq, z.t[quad], slo,
                                           shi, p.tol[level], bit);
                ok = res == 1;
            }
        }
    }
    const unsigned okm = __ballot_sync(FULL, ok), bitm = __ballot_sync(FULL, bit != 0);
    if (want2 && gather(okm) == 15u) {
        acc = true;
        rec = mns_rec_phase2(nx, ny, level, z.o, z.d0, z.d1, z.d2, (int)gather(bitm));
    }
}

// The level-3 node below a rejected level-3 phase 1 (finite e3): the moments of its four 2x2
// children (odd-phase domains: 4-pixel sums), phase 2 at level 3, else the four level-4 leaves.
__device__ __forceinline__ void level3_rejected(const Win &w, const EncParams &p, int x, int y, int sr3, bool &acc,
                                             uint64_t &rec, uint64_t *rec4) {
    Mom k4[4];
    for (int c = 0; c < 4; c++) {
        const int cx = x + 2 * (c & 1), cy = y + 2 * (c >> 1);
        Mom mm{0, 0, 0, 0, 0};
        for (int i = 0; i < 2; i++)
            for (int j = 0; j < 2; j++) {
                const int r = w.px(cx + j, cy + i);
                const int q = dom_q(w, cx, cy, 2, cx + j, cy + i);
                mm.sr += r;
                mm.srr += r * r;
                mm.sq += q;
                mm.sqq += q * q;
                mm.sqr += q * r;
            }
        k4[c] = mm;
    }
    acc = p.mns ? phase2_node(w, p, 3, x, y, 4, sr3, k4, &rec) : false;
    if (!acc)
        for (int c = 0; c < 4; c++) {
            bool dummy;
            rec4[c] = phase1(x + 2 * (c & 1), y + 2 * (c >> 1), 4, 2, k4[c], INFINITY, dummy);
        }
}

// One try_phase1 / try_phase2 call (encoder.py:145-212) on the node (x, y, 32 >> level) of a
// W x H image: the packed record (0 = rejected) and the reference's rms -- phase 1: sqrt of the
// exact mean squared residual (every term is dyadic), phase 2: the worst chosen quadrant rms,
// replayed in the reference's fp64 order, or +inf on rejection.  One CTA stages an 80-row window
// from the node's 16-aligned origin - 16 (it holds the node and its co-centred domains even for
// rects not aligned to their size); thread 0 decides.
constexpr int NODE_WIN_W = 288, NODE_WIN_H = 80, NODE_QW = NODE_WIN_W / 2;
__global__ void try_node_kernel(const uint8_t *img, int W, int H, int64_t pitch, int x, int y, int level, int phase,
                                const EncParams p, uint64_t *out_rec, double *out_rms) {
    __shared__ uint8_t pix[NODE_WIN_H][NODE_WIN_W];
    __shared__ uint16_t qe[NODE_WIN_H / 2][NODE_QW];
    __shared__ double sq_buf[256];
    const int x0 = x & ~15, y0 = y & ~15, wx0 = x0 - 16, wy0 = y0 - 16;
    for (int i = threadIdx.x; i < NODE_WIN_H * NODE_WIN_W; i += blockDim.x) {
        const int r = i / NODE_WIN_W, c = i % NODE_WIN_W, gy = wy0 + r, gx = wx0 + c;
        pix[r][c] = (gy >= 0 && gy < H && gx >= 0 && gx < W) ? img[(size_t)gy * pitch + gx] : 0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < NODE_WIN_H / 2 * NODE_QW; i += blockDim.x) {
        const int qi = i / NODE_QW, qj = i % NODE_QW;
        qe[qi][qj] = (uint16_t)(pix[2 * qi][2 * qj] + pix[2 * qi][2 * qj + 1] + pix[2 * qi + 1][2 * qj] +
                                pix[2 * qi + 1][2 * qj + 1]);
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const Win w{&pix[0][0], &qe[0][0], NODE_WIN_W, NODE_QW, -1, -1, wy0, wy0 / 2, wx0, W, H};
    const int size = 32 >> level, nlog2 = 2 * (5 - level);
    auto moments = [&](int cx, int cy, int cs) {
        Mom m{0, 0, 0, 0, 0};
        for (int i = 0; i < cs; i++)
            for (int j = 0; j < cs; j++) {
                const int q = dom_q(w, cx, cy, cs, cx + j, cy + i), r = w.px(cx + j, cy + i);
                m.sr += r;
                m.srr += r * r;
                m.sq += q;
                m.sqq += q * q;
                m.sqr += q * r;
            }
        return m;
    };
    if (phase == 1) {
        const Mom m = moments(x, y, size);
        bool acc;
        const uint64_t rec = phase1(x, y, level, nlog2, m, p.p1b[level], acc);
        const long long n = 1ll << nlog2;
        const int o = (2 * m.sr + (int)n) >> (nlog2 + 1);
        const int code = (int)((rec >> MNS_REC_PAYLOAD_SHIFT) & 7);  // the record's contrast code
        const double sdq = -0.875 + 0.25 * code, dm = ((double)m.sq * 0.25) / (double)n;
        for (int i = 0; i < size; i++)  // rms_error replayed in numpy's fp64 order (exact in practice)
            for (int j = 0; j < size; j++)
                sq_buf[i * size + j] = emu_sq(w.px(x + j, y + i), dom_q(w, x, y, size, x + j, y + i), dm, sdq,
                                              (double)o);
        *out_rec = acc ? rec : 0;
        *out_rms = __dsqrt_rn(pw_sum_dev(sq_buf, (int)n) / (double)n);
        return;
    }
    const int h = size / 2;
    Mom kids[4];
    for (int k = 0; k < 4; k++) kids[k] = moments(x + (k & 1) * h, y + (k >> 1) * h, h);
    const int sr = kids[0].sr + kids[1].sr + kids[2].sr + kids[3].sr;
    const Node2 z = p2_node(nlog2, sr, kids[0].sr, kids[1].sr, kids[2].sr, kids[3].sr, level == 1 ? 15 : 31,
                            p.gate[level]);
    *out_rec = 0;
    *out_rms = INFINITY;
    if (!z.pass) return;
    const double slo = level == 1 ? 0.2 : (level == 2 ? 0.4 : 0.5);
    const double shi = level == 1 ? 0.5 : (level == 2 ? 0.65 : 0.9);
    double worst = 0.0;
    int bits = 0;
    for (int k = 0; k < 4; k++) {
        int bit;
        double rms;
        if (!emulate_quadrant(w, x + (k & 1) * h, y + (k >> 1) * h, h, kids[k].sq, z.t[k], slo, shi, p.tol[level],
                              bit, &rms))
            return;
        bits |= bit << k;
        worst = fmax(worst, rms);
    }
    *out_rec = mns_rec_phase2(x, y, level, z.o, z.d0, z.d1, z.d2, bits);
    *out_rms = worst;
}

// ---------------------------------------------------------------- the encoder kernel
//
// Persistent CTAs over a balanced share of the (image, 16-root column band, root row) steps,
// band-major: a CTA walks DOWN its bands one root row per step with a sliding window, so every
// 16-row block of pixels is staged (TMA) and reduced to q (even 2x2 sums) and Q2 (2x2 sums of q^2
// over every q position) exactly once per band -- not three times as with one window per root
// row.  Rings (rows wrap; global row -> ring row by masking): pixels 4 blocks x 16 rows, q and Q2
// 4 blocks x 8 rows.  Step ry: block ry + 1 lands (issued one step ahead) -> its q rows -> Q2 rows
// 8ry + 7 .. 8ry + 14 -> the TMA of block ry + 2 into the slot block ry - 2 freed -> the 16 roots.
//
// Per root (half-warp; lane m = level-3 node m, its 4x4 range pixels as 4 words): Sr, Srr by
// DP4A; per level the lane's 16 q values against that level's domain as u16 pairs (PRMT-aligned
// for the odd-phase level-3 domains) -> Sqr by DP2A, Sq by packed u16x2 adds, Sqq by 4 Q2
// lookups; level 2 sums over 4 lanes, level 1 over the half-warp.  All moments and decisions
// stay in registers: level 2 on all 32 lanes (8 nodes x 4 quadrant lanes), level 1 on the
// quadrant lanes 0/4/8/12 of each half, level 3 one node per lane; then the DFS emission.
constexpr int PRING = 64;                           // pixel ring rows (4 blocks of 16)
constexpr int QW = WIN_W / 2;                       // 144 q columns
constexpr int QP = QW + 4;                          // q ring pitch (u16): 148 halves the level-1/2 load conflicts (4- to 2-way, the floor for these patterns)
constexpr int QRING = 32;                           // q / q^2 ring rows (4 blocks of 8)
constexpr int ENC_PIX = PRING * WIN_W;              // 18432 B
constexpr int ENC_Q = QRING * QP * 2;               // 9728 B
constexpr int ENC_SMEM = ENC_PIX + ENC_Q;           // 28160 B
static_assert(ENC_PIX % 16 == 0 && ENC_Q % 16 == 0, "ring alignment");

// Sum of squares of four q values (< 1024) held as u16 pairs p01, p23, by bytes: q = 256 qh + ql,
// q^2 = 65536 qh^2 + 512 qh ql + ql^2; the low and high bytes of the four values are gathered with
// two PRMTs and the three partial sums accumulate by DP4A (5 instructions for 4 squares).
__device__ __forceinline__ void sq_bytes(uint32_t p01, uint32_t p23, unsigned &sl, unsigned &sc, unsigned &sh) {
    const uint32_t lo = __byte_perm(p01, p23, 0x6420), hi = __byte_perm(p01, p23, 0x7531);
    sl = __dp4a(lo, lo, sl);
    sc = __dp4a(lo, hi, sc);
    sh = __dp4a(hi, hi, sh);
}

__device__ __forceinline__ uint32_t lds32(const uint16_t *p) { return *reinterpret_cast<const uint32_t *>(p); }

__global__ void __launch_bounds__(ET, ENC_MINB) mns_encode_kernel(const __grid_constant__ CUtensorMap tmap,
                                                           const EncParams p) {
    extern __shared__ __align__(128) unsigned char esm[];
    uint8_t *const pix = esm;
    uint16_t *const qe = reinterpret_cast<uint16_t *>(esm + ENC_PIX);
    __shared__ __align__(8) uint64_t bars[4];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int b = 0; b < 4; b++) mbar_init(&bars[b], 1);
        fence_mbar_init();
        prefetch_tmap(&tmap);
    }
    __syncthreads();
    unsigned par = 0;  // expected phase parity of each slot's barrier
    const bool try1 = p.root_level == 1 && p.min_dim >= 32;  // encoder.py:231 guard 2*size <= min_dim
    const bool vis1 = p.root_level == 1;
    const int hw = lane >> 4, m = lane & 15;
    const int lx = node3_x(m), ly = node3_y(m);
    const int k2 = m >> 2, nx2 = node2_x(k2), ny2 = node2_y(k2);
    // sure-rejection bounds bound(E) * n^2: level-1 node, its level-2 quadrants, level-2 node, its
    // level-3 quadrants
    const float bn2_1 = (float)p.p2b[1] * 65536.f, bn2_1k = (float)p.p2b[1] * 4096.f;
    const float bn2_2 = (float)p.p2b[2] * 4096.f, bn2_2k = (float)p.p2b[2] * 256.f;

    {
        // CTA (band, chunk, image): root rows [chunk * chunk_rows, ...) of one 16-root column band;
        // blockIdx.x (band) runs fastest, so horizontally adjacent bands walk the same rows together
        // and their shared halo columns are read from DRAM once
        const int band = blockIdx.x, img_i = blockIdx.z;
        const int rowi = blockIdx.y * p.chunk_rows;
        const int steps = min(p.chunk_rows, p.rows - rowi);
        const int ry0 = p.rr0 + rowi, ry_last = ry0 + steps - 1;
        const int x0 = band * TR * 16, wx0 = x0 - 16;
        const int nr = min(TR, p.rw - band * TR);
        const Win w{pix, qe, WIN_W, QP, PRING - 1, QRING - 1, 0, 0, wx0, p.W, p.H};

        auto issue = [&](int g) {  // thread 0: pixel block g (rows 16g .. 16g + 15) into slot g & 3
            mbar_arrive_expect_tx(&bars[g & 3], 16 * WIN_W);
            tma_load_3d(pix + ((16 * g) & (PRING - 1)) * WIN_W, &tmap, wx0 / TMA_E, 16 * g - p.y_res0, img_i,
                        &bars[g & 3]);
        };
        auto wait = [&](int g) {
            mbar_wait(&bars[g & 3], (par >> (g & 3)) & 1u);
            par ^= 1u << (g & 3);
        };
        // this thread's q-table items (the same every block): 8 q rows x 36 groups of 4 columns
        constexpr int NIT = 8 * (QW / 4), NBI = (NIT + ET - 1) / ET;
        int src[NBI], dst[NBI];
#pragma unroll
        for (int k = 0; k < NBI; k++) {
            const int it = tid + k * ET < NIT ? tid + k * ET : tid;
            src[k] = 2 * (it / (QW / 4)) * WIN_W + 8 * (it % (QW / 4));
            dst[k] = (it / (QW / 4)) * QP + 4 * (it % (QW / 4));
        }
        auto build = [&](int g) {  // q rows 8g .. 8g + 7 from pixel block g (4 q per item, packed adds)
            const uint8_t *pb = pix + ((16 * g) & (PRING - 1)) * WIN_W;
            uint16_t *qb = qe + ((8 * g) & (QRING - 1)) * QP;
#pragma unroll
            for (int k = 0; k < NBI; k++) {
                if (k == NBI - 1 && tid + k * ET >= NIT) break;
                const uint8_t *a = pb + src[k];
                const uint2 u = *reinterpret_cast<const uint2 *>(a);
                const uint2 v = *reinterpret_cast<const uint2 *>(a + WIN_W);
                // bytes 0, 2 and 1, 3 of each word zero-extended into u16 lanes (PRMT), summed lane-wise
                uint2 s;
                s.x = (__byte_perm(u.x, 0u, 0x4240) + __byte_perm(u.x, 0u, 0x4341)) +
                      (__byte_perm(v.x, 0u, 0x4240) + __byte_perm(v.x, 0u, 0x4341));
                s.y = (__byte_perm(u.y, 0u, 0x4240) + __byte_perm(u.y, 0u, 0x4341)) +
                      (__byte_perm(v.y, 0u, 0x4240) + __byte_perm(v.y, 0u, 0x4341));
                *reinterpret_cast<uint2 *>(qb + dst[k]) = s;
            }
        };

        if (tid == 0) {
            fence_proxy_async();
            issue(ry0 - 1);
            issue(ry0);
            issue(ry0 + 1);
        }
        wait(ry0 - 1);
        build(ry0 - 1);
        wait(ry0);
        build(ry0);

        long long row_root = ((long long)img_i * p.rows + rowi) * p.rw + (long long)band * TR;  // root index of slot 0
        for (int ry = ry0; ry <= ry_last; ry++) {
            wait(ry + 1);
            build(ry + 1);
            __syncthreads();  // the window of row ry is complete; every warp is done with row ry - 1
            if (tid == 0 && ry < ry_last) {  // block ry + 2 is read by step ry + 1 only
                fence_proxy_async();         // generic reads of block ry - 2 precede the refill
                issue(ry + 2);
            }
            // ---------------- the TR roots of root row ry (warp w: slots w + 8 (2j + hw))
#pragma unroll 1
            for (int j = 0; j < RPW; j++) {
            const int slot = warp + EW * (2 * j + hw);
            const bool live = slot < nr;
            const int sl = live ? slot : 0;
            const int rxg = x0 + 16 * sl, ryg = 16 * ry;
            const int x3 = rxg + lx, y3 = ryg + ly;
            uint32_t rw[4];
#pragma unroll
            for (int i = 0; i < 4; i++)
                rw[i] = *reinterpret_cast<const uint32_t *>(pix + ((y3 + i) & (PRING - 1)) * WIN_W + (x3 - wx0));
            int sr3 = 0, srr3 = 0;
#pragma unroll
            for (int i = 0; i < 4; i++) {
                sr3 = (int)__dp4a(rw[i], 0x01010101u, (unsigned)sr3);
                srr3 = (int)__dp4a(rw[i], rw[i], (unsigned)srr3);
            }
            // level 3: the lane's own node; the domain may start on an odd q column (PRMT-aligned pairs)
            int sq3, sqq3, sqr3;
            {
                const int gdx = clampi(x3 - 2, 0, p.W - 8), gdy = clampi(y3 - 2, 0, p.H - 8);
                const int qx = (gdx - wx0) >> 1, qy = gdy >> 1;
                const int cw = qx & ~1;
                const unsigned sel = (qx & 1) ? 0x5432u : 0x3210u;
                unsigned sqp = 0, sqr = 0, sql = 0, sqc = 0, sqh = 0;
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const int row = (qy + i) & (QRING - 1);
                    const uint16_t *qr = qe + row * QP + cw;
                    const uint32_t w0 = lds32(qr), w1 = lds32(qr + 2), w2 = lds32(qr + 4);
                    const uint32_t p01 = __byte_perm(w0, w1, sel), p23 = __byte_perm(w1, w2, sel);
                    sqr = __dp2a_lo(p01, rw[i], sqr);
                    sqr = __dp2a_hi(p23, rw[i], sqr);
                    sqp += p01 + p23;
                    sq_bytes(p01, p23, sql, sqc, sqh);
                }
                sq3 = (int)((sqp & 0xFFFF) + (sqp >> 16));
                sqr3 = (int)sqr;
                sqq3 = (int)((sqh << 16) + (sqc << 9) + sql);
            }
            // the lane's share of an even-phase level-1/2 domain starting at window q column qx, q row qy
            auto part = [&](int qx, int qy, unsigned &sqp, unsigned &sqr, unsigned &sqq) {
                sqp = 0;
                sqr = 0;
                unsigned sql = 0, sqc = 0, sqh = 0;
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const uint16_t *qr = qe + ((qy + i) & (QRING - 1)) * QP + qx;
                    const uint32_t p01 = lds32(qr), p23 = lds32(qr + 2);  // qx even (not always 4-aligned)
                    sqr = __dp2a_lo(p01, rw[i], sqr);
                    sqr = __dp2a_hi(p23, rw[i], sqr);
                    sqp += p01 + p23;
                    sq_bytes(p01, p23, sql, sqc, sqh);
                }
                sqq = (sqh << 16) + (sqc << 9) + sql;
            };
            // level 2: node k2 of the root; 4-lane groups
            Mom m2;
            {
                const int gdx = clampi(rxg + nx2 - 4, 0, p.W - 16), gdy = clampi(ryg + ny2 - 4, 0, p.H - 16);
                unsigned sqp, sqr, sqq;
                part(((gdx - wx0) >> 1) + (lx - nx2), (gdy >> 1) + (ly - ny2), sqp, sqr, sqq);
                int v[5] = {sr3, srr3, (int)sqp, (int)sqq, (int)sqr};  // packed Sq halves stay < 2^16
#pragma unroll
                for (int k = 0; k < 5; k++) {
                    v[k] += __shfl_xor_sync(FULL, v[k], 1);
                    v[k] += __shfl_xor_sync(FULL, v[k], 2);
                }
                m2 = Mom{v[0], v[1], (int)((v[2] & 0xFFFF) + ((unsigned)v[2] >> 16)), v[3], v[4]};
            }
            // level 1: the half-warp (one root); Sr, Srr from the level-2 sums
            Mom m1{0, 0, 0, 0, 0};
            if (try1) {
                const int gdx = clampi(rxg - 8, 0, p.W - 32), gdy = clampi(ryg - 8, 0, p.H - 32);
                unsigned sqp, sqr, sqq;
                part(((gdx - wx0) >> 1) + lx, (gdy >> 1) + ly, sqp, sqr, sqq);
                int u[5] = {m2.sr, m2.srr, (int)((sqp & 0xFFFF) + (sqp >> 16)), (int)sqq, (int)sqr};
#pragma unroll
                for (int k = 0; k < 2; k++) {
                    u[k] += __shfl_xor_sync(FULL, u[k], 4);
                    u[k] += __shfl_xor_sync(FULL, u[k], 8);
                }
#pragma unroll
                for (int k = 2; k < 5; k++) {
                    u[k] += __shfl_xor_sync(FULL, u[k], 1);
                    u[k] += __shfl_xor_sync(FULL, u[k], 2);
                    u[k] += __shfl_xor_sync(FULL, u[k], 4);
                    u[k] += __shfl_xor_sync(FULL, u[k], 8);
                }
                m1 = Mom{u[0], u[1], u[2], u[3], u[4]};
            }
            const Mom m3{sr3, srr3, sq3, sqq3, sqr3};
            // ---- decisions (encoder.py:226-246).  A node whose best free least-squares fit already
            // misses its bound is rejected for sure (no quantised fit can do better) -- the common
            // case on textured images -- and a warp whose nodes are all surely rejected skips the
            // exact decision; otherwise node_decide runs the exact one.
            // level 2: quadrant lane = m & 3, kid = own level-3 node
            bool acc2 = false;
            uint64_t rec2 = 0;
            const FitGap<6> g2 = fit_gap<6>(m2);  // shared by the level-2 node test and level 1's quadrant test
            {
                const int g0 = lane & ~3;
                int ks[4];
#pragma unroll
                for (int c = 0; c < 4; c++) ks[c] = __shfl_sync(FULL, sr3, g0 + c);
                const bool kid_out = !p.mns || surely_above<4>(m3, bn2_2k);
                const unsigned kb = __ballot_sync(FULL, kid_out);
                const bool sure = surely_above<6>(g2, bn2_2) &&
                                  (((kb >> g0) & 15u) != 0 || gate_fails(6, m2.sr, ks, p.gate[2]));
                if (__any_sync(FULL, live && !sure))
                    node_decide(w, p, live, true, m & 3, 2, rxg + nx2, ryg + ny2, m2, ks, m3,
                                [g0](unsigned b) { return (b >> g0) & 15u; }, acc2, rec2);
            }
            // level 1: quadrant lanes 0, 4, 8, 12 of the half (kid = the lane's level-2 node)
            bool acc1 = false;
            uint64_t rec1 = 0;
            if (try1) {
                const int hb = 16 * hw;
                int ks[4];
#pragma unroll
                for (int c = 0; c < 4; c++) ks[c] = __shfl_sync(FULL, m2.sr, hb + 4 * c);
                auto gather = [hb](unsigned b) {  // bits hb, hb + 4, hb + 8, hb + 12 -> 0..3
                    unsigned x = (b >> hb) & 0x1111u;
                    x = (x | (x >> 3)) & 0x0303u;
                    return (x | (x >> 6)) & 15u;
                };
                const bool kid_out = (m & 3) == 0 && (!p.mns || surely_above<6>(g2, bn2_1k));
                const unsigned kb = __ballot_sync(FULL, kid_out);
                const bool sure = surely_above<8>(m1, bn2_1) &&
                                  ((kb & (0x1111u << hb)) != 0 || gate_fails(8, m1.sr, ks, p.gate[1]));
                if (__any_sync(FULL, live && !sure))
                    node_decide(w, p, live, (m & 3) == 0, k2, 1, rxg, ryg, m1, ks, m2, gather, acc1, rec1);
            }
            // level 3 (own node): phase 1, and the rejected path (finite e3) only where visible
            bool acc3;
            uint64_t rec3 = phase1(x3, y3, 3, 4, m3, p.p1b[3], acc3);
            const bool vis2 = !vis1 || !acc1;
            const bool vis3 = vis2 && !acc2;
            uint64_t rec4[4];  // written (and read) only on the rejected path
            if (live && vis3 && !acc3) level3_rejected(w, p, x3, y3, sr3, acc3, rec3, rec4);
            const bool vis4 = vis3 && !acc3;

            // ---- DFS (Morton) emission: the covering leaf's record on the first lane it covers, or
            // the node's four level-4 records; offsets by two ballots (records per lane: 0, 1 or 4)
            uint64_t cov;
            int nrec;
            if (vis1 && acc1) {
                nrec = m == 0;
                cov = rec1;
            } else if (vis2 && acc2) {
                nrec = (m & 3) == 0;
                cov = rec2;
            } else if (vis3 && acc3) {
                nrec = 1;
                cov = rec3;
            } else {
                nrec = 4;
                cov = 0;
            }
            if (!live) nrec = 0;
            const unsigned half = hw ? 0xFFFF0000u : 0x0000FFFFu, lt = lanemask_lt() & half;
            const unsigned b1 = __ballot_sync(FULL, nrec != 0) & half, b4 = __ballot_sync(FULL, nrec == 4) & half;
            const int off = __popc(b1 & lt) + 3 * __popc(b4 & lt);
            const long long root = row_root + sl;
            if (live) {
                uint64_t *st = p.stage + root * 64 + off;
                if (nrec == 4) {
#pragma unroll
                    for (int c = 0; c < 4; c++) st[c] = rec4[c];
                } else if (nrec) {
                    st[0] = cov;
                }
                if (m == 0) p.root_cnt[root] = __popc(b1) + 3 * __popc(b4);
                if (p.unit_map && p.map_form == 1) {  // block map: the descriptor of the block's first cell
                    reinterpret_cast<uint16_t *>(p.unit_map)[root * 16 + m] =
                        mns_unit_of_record(vis4 ? rec4[0] : cov, rxg, ryg, lx, ly);
                } else if (p.unit_map) {
                    uint2 u;
                    if (vis4) {
                        u.x = (uint32_t)mns_unit_of_record(rec4[0], rxg, ryg, lx, ly) |
                              ((uint32_t)mns_unit_of_record(rec4[1], rxg, ryg, lx + 2, ly) << 16);
                        u.y = (uint32_t)mns_unit_of_record(rec4[2], rxg, ryg, lx, ly + 2) |
                              ((uint32_t)mns_unit_of_record(rec4[3], rxg, ryg, lx + 2, ly + 2) << 16);
                    } else if (!((cov >> MNS_REC_PHASE2_SHIFT) & 1)) {  // a phase-1 leaf: one descriptor
                        const uint32_t d = mns_unit_desc((int)((cov >> MNS_REC_PAYLOAD_SHIFT) & 7),
                                                         (int)((cov >> MNS_REC_O_SHIFT) & 0xFF),
                                                         4 - (int)((cov >> MNS_REC_LEVEL_SHIFT) & 3));
                        u.x = u.y = d | (d << 16);
                    } else {
                        u.x = mns_unit_pair_of_record(cov, rxg, ryg, lx, ly);
                        u.y = mns_unit_pair_of_record(cov, rxg, ryg, lx, ly + 2);
                    }
                    *reinterpret_cast<uint2 *>(&p.unit_map[root * 32 + 2 * m]) = u;
                }
            }
            }
            row_root += p.rw;
        }
    }
}

// ---------------------------------------------------------------- isometry extension
//
// n_iso = 8 (BASELINE configs[1], not in the reference: SPEC.md:16): phase 1 of every node also tries
// the 8 isometries d_t(i, j) = d(src_t(i, j)) of its co-centred domain (mns_common.cuh iso_src, as in
// the full search) and keeps the one with the smallest exact quantised SSE (ties: the lowest t); the
// record carries t (MNS_REC_ISO_SHIFT).  Phase 2 and the traversal are the reference's.  One warp per
// root walks the quadtree depth first with an explicit stack; every node's moments (and the
// isometries' cross terms) are warp reductions over its pixels, the decisions run on every lane
// (phase 2 through phase2_node, emulation included), records go straight into the root's staged
// slots (the same compaction follows).
constexpr int IWIN = 48;  // a root's window: [x0 - 16, x0 + 32) x [y0 - 16, y0 + 32)
constexpr int IWARPS = 4;

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// Identity moments of node (x, y, size) against its co-centred domain, warp-wide (every lane gets them)
__device__ Mom warp_moments(const Win &w, int x, int y, int size) {
    const int lane = threadIdx.x & 31, n = size * size;
    int v[5] = {0, 0, 0, 0, 0};
    for (int e = lane; e < n; e += 32) {
        const int px = x + e % size, py = y + e / size;
        const int r = w.px(px, py), q = dom_q(w, x, y, size, px, py);
        v[0] += r;
        v[1] += r * r;
        v[2] += q;
        v[3] += q * q;
        v[4] += q * r;
    }
    return Mom{warp_sum(v[0]), warp_sum(v[1]), warp_sum(v[2]), warp_sum(v[3]), warp_sum(v[4])};
}

// Phase 1 with the isometry search; returns acceptance (level 4 always) and the record.
__device__ bool phase1_iso(const Win &w, const EncParams &p, int x, int y, int level, int n_iso, uint64_t &rec) {
    const int lane = threadIdx.x & 31, size = 32 >> level, n = size * size, nlog2 = 2 * (5 - level);
    int m5[5] = {0, 0, 0, 0, 0}, sqr_t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int e = lane; e < n; e += 32) {
        const int i = e / size, j = e % size;
        const int r = w.px(x + j, y + i), q = dom_q(w, x, y, size, x + j, y + i);
        m5[0] += r;
        m5[1] += r * r;
        m5[2] += q;
        m5[3] += q * q;
        for (int t = 0; t < n_iso; t++) {  // d_t(i, j) = d(src_t(i, j))
            const int m = t ? iso_src(t, i, j, size) : e;
            sqr_t[t] += r * (t ? dom_q(w, x, y, size, x + m % size, y + m / size) : q);
        }
    }
    const int sr = warp_sum(m5[0]), srr = warp_sum(m5[1]), sq = warp_sum(m5[2]), sqq = warp_sum(m5[3]);
    const int o = (2 * sr + n) >> (nlog2 + 1);  // round_to_int(mean)
    const long long D = ((long long)sqq << nlog2) - (long long)sq * sq;
    const long long A = (long long)srr - 2ll * o * sr + ((long long)o * o << nlog2);  // sum (r - o)^2
    long long best = LLONG_MAX;
    int bt = 0, bcode = 4;
    for (int t = 0; t < n_iso; t++) {
        const int sqr = warp_sum(sqr_t[t]);
        const long long N = ((long long)sqr << nlog2) - (long long)sq * sr;
        const int code = quant_code(16.0 * (double)N, (double)D);
        const long long k2 = 2 * code - 7;
        const long long X = (A << (nlog2 + 10)) - 64 * k2 * N + k2 * k2 * D;  // 1024 n SSE, exact
        if (X < best) {
            best = X;
            bt = t;
            bcode = code;
        }
    }
    rec = mns_rec_phase1(x, y, level, o, bcode) | ((uint64_t)bt << MNS_REC_ISO_SHIFT);
    return level == 4 || (double)best <= p.p1b[level];
}

__global__ void __launch_bounds__(IWARPS * 32) mns_encode_iso_kernel(const uint8_t *img, int64_t pitch,
                                                                    int64_t image_stride, int y_res0, int y_res1,
                                                                    const EncParams p, int n_iso) {
    __shared__ uint8_t pix[IWARPS][IWIN][IWIN];
    __shared__ uint16_t qe[IWARPS][IWIN / 2][IWIN / 2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long root = (long long)blockIdx.x * IWARPS + warp;
    if (root >= p.n_roots) return;  // whole warps
    const int rx = (int)(root % p.rw);
    const long long t = root / p.rw;
    const int ry = p.rr0 + (int)(t % p.rows), img_i = (int)(t / p.rows);
    const int x0 = 16 * rx, y0 = 16 * ry;
    const uint8_t *base = img + (ptrdiff_t)img_i * image_stride;
    for (int e = lane; e < IWIN * IWIN; e += 32) {  // rows outside the resident strip are never read
        const int r = e / IWIN, c = e % IWIN, gy = y0 - 16 + r, gx = x0 - 16 + c;
        pix[warp][r][c] = (gy >= y_res0 && gy < y_res1 && gx >= 0 && gx < p.W) ? base[(ptrdiff_t)gy * pitch + gx] : 0;
    }
    __syncwarp();
    for (int e = lane; e < (IWIN / 2) * (IWIN / 2); e += 32) {
        const int r = e / (IWIN / 2), c = e % (IWIN / 2);
        qe[warp][r][c] = (uint16_t)(pix[warp][2 * r][2 * c] + pix[warp][2 * r][2 * c + 1] + pix[warp][2 * r + 1][2 * c] +
                                    pix[warp][2 * r + 1][2 * c + 1]);
    }
    __syncwarp();
    const Win w{&pix[warp][0][0], &qe[warp][0][0], IWIN, IWIN / 2, -1, -1, y0 - 16, (y0 - 16) / 2, x0 - 16, p.W,
                p.H};
    uint64_t *st = p.stage + root * 64;
    int cnt = 0;
    // depth-first stack of (x, y, level) packed as x | y << 8 | level << 16 (root-relative x, y)
    int stack[16], sp = 0;
    if (p.root_level == 1) {
        stack[sp++] = 1 << 16;
    } else {
        for (int c = 3; c >= 0; c--) stack[sp++] = (8 * (c & 1)) | ((8 * (c >> 1)) << 8) | (2 << 16);
    }
    while (sp) {
        const int e = stack[--sp];
        const int level = e >> 16, x = x0 + (e & 255), y = y0 + ((e >> 8) & 255), size = 32 >> level;
        uint64_t rec = 0;
        bool acc = false;
        if (2 * size <= p.min_dim) {  // encoder.py:231
            acc = phase1_iso(w, p, x, y, level, n_iso, rec);
            if (!acc && p.mns && level <= 3) {
                const int h = size / 2;
                Mom kids[4];
                for (int c = 0; c < 4; c++) kids[c] = warp_moments(w, x + (c & 1) * h, y + (c >> 1) * h, h);
                const int sr = kids[0].sr + kids[1].sr + kids[2].sr + kids[3].sr;
                acc = phase2_node(w, p, level, x, y, size, sr, kids, &rec);
            }
        }
        if (acc) {
            if (lane == 0) st[cnt] = rec;
            cnt++;
        } else {
            const int h = size / 2, lx = e & 255, ly = (e >> 8) & 255;
            for (int c = 3; c >= 0; c--) stack[sp++] = (lx + (c & 1) * h) | ((ly + (c >> 1) * h) << 8) | ((level + 1) << 16);
        }
    }
    if (lane == 0) p.root_cnt[root] = cnt;
}

// Compaction (second half of the encode): exclusive scan of the per-root counts into
// root_offsets (in place) with a decoupled look-back over uniform 2048-root tiles, then a
// coalesced copy of every root's staged records to its offset.  Keeping the scan out of the
// encoder means no encoder CTA ever waits on another.
#ifndef CT_PER_DEF
#define CT_PER_DEF 8
#endif
#ifndef CT_U_DEF
#define CT_U_DEF 4
#endif
constexpr int CT_THREADS = 256, CT_PER = CT_PER_DEF, CT_ROOTS = CT_THREADS * CT_PER;
constexpr int CT_U = CT_U_DEF;  // staged-record loads in flight per lane

__global__ void __launch_bounds__(CT_THREADS) compact_records_kernel(const uint64_t *stage, int32_t *root_offsets,
                                                                     long long n_roots, uint64_t *out,
                                                                     int64_t *count, unsigned long long *status) {
    __shared__ int offs[CT_ROOTS];
    __shared__ int warp_tot[CT_THREADS / 32];
    __shared__ long long tile_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long long tile = blockIdx.x, r0 = tile * CT_ROOTS;
    int c[CT_PER], run = 0;
#pragma unroll
    for (int i = 0; i < CT_PER; i++) {
        const long long r = r0 + tid * CT_PER + i;
        c[i] = r < n_roots ? root_offsets[r] : 0;
        run += c[i];
    }
    int incl = run;  // block-wide inclusive scan of the thread totals
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    int wbase = 0, total = 0;
#pragma unroll
    for (int k = 0; k < CT_THREADS / 32; k++) {
        wbase += k < warp ? warp_tot[k] : 0;
        total += warp_tot[k];
    }
    if (warp == 0) {
        const long long b = lookback_exclusive_warp(status, tile, total);
        if (lane == 0) tile_base = b;
    }
    int e = wbase + incl - run;
#pragma unroll
    for (int i = 0; i < CT_PER; i++) {
        offs[tid * CT_PER + i] = e;
        e += c[i];
    }
    __syncthreads();
    const long long base = tile_base;
#pragma unroll
    for (int i = 0; i < CT_PER; i++) {
        const long long r = r0 + tid * CT_PER + i;
        if (r < n_roots) root_offsets[r] = (int32_t)(base + offs[tid * CT_PER + i]);
    }
    if (r0 + CT_ROOTS >= n_roots && tid == 0) {  // last tile
        root_offsets[n_roots] = (int32_t)(base + total);
        *count = base + total;
    }
    // copy, one 32-root chunk per warp at a time: lane l holds the chunk's root l offset; output
    // record j of the chunk belongs to the last root whose offset is <= j (5-step shuffle search);
    // 4 independent read-only loads per lane in flight
    const int nr_tile = (int)min((long long)CT_ROOTS, n_roots - r0);
    uint64_t *dst = out + base;
    for (int c0 = 32 * warp; c0 < nr_tile; c0 += CT_THREADS) {
        const int nk = min(32, nr_tile - c0);
        const int my_off = lane < nk ? offs[c0 + lane] : INT_MAX;
        const int j_lo = __shfl_sync(FULL, my_off, 0);
        const int j_hi = c0 + nk < nr_tile ? offs[c0 + nk] : total;
        for (int j0 = j_lo; j0 < j_hi; j0 += CT_U * 32) {
            uint64_t v[CT_U];
            int jj[CT_U];
#pragma unroll
            for (int u = 0; u < CT_U; u++) {
                jj[u] = j0 + 32 * u + lane;
                int k = 0;  // largest chunk root with offset <= j (roots with no records never win ties)
#pragma unroll
                for (int step = 16; step > 0; step >>= 1) {
                    const int o = __shfl_sync(FULL, my_off, k + step < 32 ? k + step : 31);
                    if (k + step < nk && o <= jj[u]) k += step;
                }
                const int ok = __shfl_sync(FULL, my_off, k);
                if (jj[u] < j_hi) v[u] = __ldg(stage + (r0 + c0 + k) * 64 + (jj[u] - ok));
            }
#pragma unroll
            for (int u = 0; u < CT_U; u++)
                if (jj[u] < j_hi) dst[jj[u]] = v[u];
        }
    }
}

}  // namespace

static long long compact_tiles(long long n_roots) { return (n_roots + CT_ROOTS - 1) / CT_ROOTS; }

// Integer form of the phase-2 mean gate at node size n: floor(mean_tol * n) (exact: n is a power of
// two), saturated -- |df| <= 4 * 255 * 256 never exceeds INT_MAX; NaN never fails, like the float test.
static int mean_gate(double mean_tol, int n) {
    const double x = mean_tol * (double)n;
    if (!(x == x) || x >= 2147483647.0) return INT_MAX;
    if (x < -2147483647.0) return -1;
    return (int)floor(x);
}

int encode_workspace_bytes(int width, int n_images, int rr0, int rr1, int64_t *bytes) {
    const long long n_roots = (long long)n_images * (rr1 - rr0) * (width / 16);
    // [compaction look-back status, 256-B aligned][64 staged record slots per root]
    *bytes = ((compact_tiles(n_roots) * 8 + 255) / 256) * 256 + n_roots * 64 * 8;
    return 0;
}

int encode_quadtree(const uint8_t *img, int W, int H, int64_t pitch, int64_t image_stride, int n_images, int rr0,
                    int rr1, const mns_enc_cfg *cfg, uint64_t *records, int64_t capacity, int32_t *root_offsets,
                    int64_t *d_count, uint32_t *unit_map, void *workspace, int64_t workspace_bytes,
                    cudaStream_t stream, cudaStream_t cstream) {
    MNS_CHECK_ARG(W > 0 && H > 0 && W % 16 == 0 && H % 16 == 0, "width/height must be positive multiples of 16");
    MNS_CHECK_ARG(W <= 65534 && H <= 65534, "dimensions exceed the record coordinate range");
    MNS_CHECK_ARG(pitch >= W && pitch % 16 == 0, "pitch must be >= width and a multiple of 16");
    MNS_CHECK_ARG(((uintptr_t)img & 15) == 0, "image pointer must be 16-byte aligned");
    MNS_CHECK_ARG(n_images >= 1 && (n_images == 1 || (image_stride % 16 == 0)), "bad image stride");
    MNS_CHECK_ARG(0 <= rr0 && rr0 < rr1 && rr1 <= H / 16, "bad root row range");
    MNS_CHECK_ARG(cfg && (cfg->root_level == 1 || cfg->root_level == 2), "root_level must be 1 or 2");
    MNS_CHECK_ARG(cfg->n_iso == 0 || cfg->n_iso == 1 || cfg->n_iso == 8, "n_iso must be 1 or 8");
    MNS_CHECK_ARG(cfg->map_form == 0 || cfg->map_form == 1, "map_form must be 0 (unit map) or 1 (block map)");
    const int rw = W / 16;
    const long long n_roots = (long long)n_images * (rr1 - rr0) * rw;
    MNS_CHECK_ARG(capacity >= 64 * n_roots, "record capacity must be >= 64 * roots");
    MNS_CHECK_ARG(64 * n_roots < (1ll << 31), "too many roots for int32 root offsets");
    int64_t need;
    encode_workspace_bytes(W, n_images, rr0, rr1, &need);
    MNS_CHECK_ARG(workspace_bytes >= need, "workspace too small");
    MNS_CHECK_ARG(((uintptr_t)workspace & 15) == 0, "workspace must be 16-byte aligned");

    EncParams p{};
    p.W = W;
    p.H = H;
    p.n_images = n_images;
    p.rr0 = rr0;
    p.rows = rr1 - rr0;
    p.rw = rw;
    p.tiles_per_row = (rw + TR - 1) / TR;
    p.mns = cfg->mns;
    p.root_level = cfg->root_level;
    p.min_dim = W < H ? W : H;
    for (int l = 1; l <= 3; l++) {
        const double n = (double)(1 << (2 * (5 - l)));  // 256, 64, 16
        const double bnd = sqrt_bound(cfg->e[l - 1]);
        p.p1b[l] = bnd * 1024.0 * n * n;  // exact power-of-two scaling (inf stays inf)
        p.p2b[l] = bnd;
        p.tol[l] = cfg->e[l - 1];
    }
    p.p1b[4] = INFINITY;
    p.mean_tol = cfg->mean_tol;
    for (int l = 1; l <= 3; l++) p.gate[l] = mean_gate(cfg->mean_tol, 1 << (2 * (5 - l)));
    const long long ctiles = compact_tiles(n_roots);
    const size_t status_bytes = ((ctiles * 8 + 255) / 256) * 256;
    unsigned long long *status = reinterpret_cast<unsigned long long *>(workspace);
    p.stage = reinterpret_cast<uint64_t *>(reinterpret_cast<char *>(workspace) + status_bytes);
    p.unit_map = unit_map;
    p.map_form = cfg->map_form;
    p.root_cnt = root_offsets;
    p.n_roots = n_roots;
    MNS_CUDA_TRY(cudaMemsetAsync(status, 0, ctiles * 8, stream));
    {
        static std::atomic<unsigned long long> done{0};
        MNS_CUDA_TRY(ensure_dynamic_smem(mns_encode_kernel, ENC_SMEM, done));
    }
    // rows [16 rr0 - 16, 16 rr1 + 16) of each image are resident: the tensor map starts there
    p.y_res0 = 16 * rr0 - 16 > 0 ? 16 * rr0 - 16 : 0;
    const int y_res1 = 16 * rr1 + 16 < H ? 16 * rr1 + 16 : H;
    CUtensorMap tmap{};
    if (encode_tmap_3d(&tmap, TMA_E == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                   : (TMA_E == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT64),
                       img + (ptrdiff_t)p.y_res0 * pitch, (uint64_t)W / TMA_E,
                       (uint64_t)(y_res1 - p.y_res0), (uint64_t)n_images, (uint64_t)pitch,
                       (uint64_t)(n_images > 1 ? image_stride : pitch * (int64_t)(y_res1 - p.y_res0)), WIN_W / TMA_E, 16,
                       1))
        return -1;
    // chunks of root rows per band: about two waves of resident CTAs (a CTA re-stages two blocks of
    // halo rows per chunk, so chunks are as long as the wave count allows)
    static int ctas = 0;
    if (!ctas) {
        int dev = 0, sms = 148, occ = 4;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mns_encode_kernel, ET, ENC_SMEM) != cudaSuccess ||
            occ < 1)
            occ = 1;
        ctas = sms * occ;
    }
    const long long cols = (long long)p.tiles_per_row * n_images;
    long long chunks = 2ll * ctas / cols;
    chunks = chunks < 1 ? 1 : (chunks > p.rows ? p.rows : chunks);
    p.chunk_rows = (int)((p.rows + chunks - 1) / chunks);
    chunks = (p.rows + p.chunk_rows - 1) / p.chunk_rows;
    MNS_CHECK_ARG(n_images <= 65535 && chunks <= 65535, "grid too large");
    const dim3 grid((unsigned)p.tiles_per_row, (unsigned)chunks, (unsigned)n_images);
    if (cfg->n_iso > 1) {  // the isometry extension (no unit map: those codes decode on the unit path)
        mns_encode_iso_kernel<<<(unsigned)((n_roots + IWARPS - 1) / IWARPS), IWARPS * 32, 0, stream>>>(
            img, pitch, n_images > 1 ? image_stride : 0, p.y_res0, y_res1, p, cfg->n_iso);
    } else {
        mns_encode_kernel<<<grid, ET, ENC_SMEM, stream>>>(tmap, p);
    }
    MNS_CUDA_TRY(cudaGetLastError());
    if (cstream != stream) {  // the compaction on its own stream, after the encoder
        cudaEvent_t ev;
        MNS_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        MNS_CUDA_TRY(cudaEventRecord(ev, stream));
        MNS_CUDA_TRY(cudaStreamWaitEvent(cstream, ev, 0));
        MNS_CUDA_TRY(cudaEventDestroy(ev));
    }
    compact_records_kernel<<<(unsigned)ctiles, CT_THREADS, 0, cstream>>>(p.stage, root_offsets, n_roots, records,
                                                                         d_count, status);
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

int try_node(const uint8_t *img, int W, int H, int64_t pitch, int x, int y, int level, int phase,
             const mns_enc_cfg *cfg, uint64_t *d_rec, double *d_rms, cudaStream_t stream) {
    MNS_CHECK_ARG(W > 0 && H > 0 && pitch >= W && W <= 65534 && H <= 65534, "bad image geometry");
    MNS_CHECK_ARG(level >= 1 && level <= 4 && (phase == 1 || (phase == 2 && level <= 3)), "bad level / phase");
    const int size = 32 >> level;
    MNS_CHECK_ARG(x >= 0 && y >= 0 && x + size <= W && y + size <= H, "node outside the image");
    MNS_CHECK_ARG(phase == 2 || (2 * size <= W && 2 * size <= H), "no co-centred domain fits the image");
    EncParams p{};
    for (int l = 1; l <= 3; l++) {
        const double n = (double)(1 << (2 * (5 - l)));
        const double bnd = sqrt_bound(cfg->e[l - 1]);
        p.p1b[l] = bnd * 1024.0 * n * n;
        p.p2b[l] = bnd;
        p.tol[l] = cfg->e[l - 1];
    }
    p.p1b[4] = INFINITY;
    p.mean_tol = cfg->mean_tol;
    for (int l = 1; l <= 3; l++) p.gate[l] = mean_gate(cfg->mean_tol, 1 << (2 * (5 - l)));
    try_node_kernel<<<1, 256, 0, stream>>>(img, W, H, pitch, x, y, level, phase, p, d_rec, d_rms);
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

}  // namespace mns
