// MNS quadtree encoder for sm_100a: block moments (K1) + phase-1/phase-2 matcher
// + per-root DFS emission (K2) in one kernel, then a scan + compaction kernel.
//
// Replaces the reference's per-node Python recursion
//   encoder.py:215-246 encode_quadtree / visit, :145-166 try_phase1,
//   :169-212 try_phase2, image.py:146-187 block helpers, transform.py:23-80.
//
// Work decomposition: one CTA = up to TR = 16 consecutive 16x16 roots of one root
// row (warp w owns roots w and w + 8).  The CTA stages the uint8 window
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
constexpr int EW = 8;                // warps per CTA
constexpr int ET = EW * 32;
constexpr int RPW = 2;               // roots encoded by each warp per tile (in turn)
constexpr int TR = EW * RPW;         // 16 consecutive roots of one root row per tile
static_assert(RPW == 2, "the warp-local decision rounds map two roots onto one warp");
constexpr int WIN_W = TR * 16 + 32;  // 544
constexpr int WIN_H = 48;
constexpr int QE_WL = WIN_W / 2;     // 272 q columns
constexpr int QE_W = QE_WL + 4;      // row stride 276: K1c's lanes read rows 2 apart, 4 banks apart
constexpr int QE_H = WIN_H / 2;      // 24

struct EncParams {
    int y_res0;  // first resident image row (the tensor map's row 0)
    int W, H, n_images, rr0, rows, rw, tiles_per_row;
    int mns, root_level, min_dim;
    double p1b[5];  // phase-1 accept bound on 1024*n*SSE per level (inf for level 4)
    double p2b[4];  // bound(E_level): phase-2 quadrant accepts iff SSE <= n_k * p2b
    double tol[4];  // E_level (emulation path compares rms > tol like the reference)
    double mean_tol;
    int gate[4];    // phase-2 mean gate per level: |n * (O_k - O_i)| > gate  <=>  |O_k - O_i| > mean_tol
    uint64_t *stage;     // 64 record slots per root (workspace); compacted by compact_records_kernel
    uint32_t *unit_map;  // optional: decoder unit map (mns_record.h), 32 words per root
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
__device__ __forceinline__ int node4_x(int c) { return node3_x(c >> 2) + 2 * (c & 1); }
__device__ __forceinline__ int node4_y(int c) { return node3_y(c >> 2) + 2 * ((c >> 1) & 1); }

// Shared-memory layout of one tile (TR roots); moments and decisions are per node.
struct TileSmem {
    Mom m1[TR];
    Mom m2[TR][4];
    Mom m3[TR][16];
    int sr4[TR][64], srr4[TR][64];  // level-4 range sums (q moments are computed lazily)
    uint64_t rec1[TR], rec2[TR][4], rec3[TR][16], rec4[TR][64];
    uint8_t acc1[TR], acc2[TR][4], acc3[TR][16];
};
constexpr int TILE_SMEM = ((int)sizeof(TileSmem) + 127) / 128 * 128;  // the TMA window follows, 128-B aligned
constexpr int ENC_SMEM = WIN_H * WIN_W + QE_H * QE_W * 2 + TILE_SMEM + 64;

struct Win {  // the staged window and the tile/image geometry a decision thread needs
    const uint8_t (*pix)[WIN_W];
    const uint16_t (*qe)[QE_W];
    int x0, y0, wx0, wy0, W, H;
};

// q of pixel (py, px) (root-relative) against the co-centred domain of node (nx, ny, s) of root slot
__device__ __forceinline__ int dom_q(const Win &w, int slot, int nx, int ny, int s, int px, int py) {
    const int rxg = w.x0 + 16 * slot, ryg = w.y0;
    const int gdx = clampi(rxg + nx - s / 2, 0, w.W - 2 * s), gdy = clampi(ryg + ny - s / 2, 0, w.H - 2 * s);
    const int wx = gdx - w.wx0 + 2 * (px - nx), wy = gdy - w.wy0 + 2 * (py - ny);
    if (((wx | wy) & 1) == 0) return w.qe[wy >> 1][wx >> 1];
    const uint8_t *pp = &w.pix[wy][wx];
    return (int)pp[0] + pp[1] + pp[WIN_W] + pp[WIN_W + 1];
}

__device__ __forceinline__ int pixel(const Win &w, int slot, int px, int py) {
    return w.pix[16 + py][16 + 16 * slot + px];
}

// Reference-order emulation of one phase-2 quadrant (transform.py:69-80 rms_error) -- the
// quadrant is the child (cx, cy, cs) of a node at `level`; the domain is the child's own.
// Returns 1 accept / 0 reject, the chosen bit and (rms_out) the chosen candidate's rms.
__device__ int emulate_quadrant(const Win &w, int slot, int cx, int cy, int cs, const Mom &m, int t, double slo,
                                double shi, double tol, int &bit, double *rms_out = nullptr) {
    double lo[64], hi[64];
    const int n = cs * cs;
    const double dm = ((double)m.sq * 0.25) / (double)n;
    const double td = (double)t;
    for (int i = 0; i < cs; i++)
        for (int j = 0; j < cs; j++) {
            const int q = dom_q(w, slot, cx, cy, cs, cx + j, cy + i);
            const int r = pixel(w, slot, cx + j, cy + i);
            lo[i * cs + j] = emu_sq(r, q, dm, slo, td);
            hi[i * cs + j] = emu_sq(r, q, dm, shi, td);
        }
    const double rlo = __dsqrt_rn(pw_sum_dev(lo, n) / (double)n), rhi = __dsqrt_rn(pw_sum_dev(hi, n) / (double)n);
    bit = rlo <= rhi ? 0 : 1;
    if (rms_out) *rms_out = bit ? rhi : rlo;
    return ((bit ? rhi : rlo) > tol) ? 0 : 1;
}

// Phase 2 of node (nx, ny, size) at `level` from its own Sr and its 4 children's moments
// (encoder.py:169-212).  Returns true with *rec on acceptance.
__device__ bool phase2_node(const Win &w, const EncParams &p, int slot, int level, int nx, int ny, int size, int sr,
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
            res = emulate_quadrant(w, slot, nx + (k & 1) * h, ny + (k >> 1) * h, h, kids[k], z.t[k], slo, shi,
                                   p.tol[level], bit);
        if (res != 1) return false;
        bits |= bit << k;
    }
    *rec = mns_rec_phase2(w.x0 + 16 * slot + nx, w.y0 + ny, level, z.o, z.d0, z.d1, z.d2, bits);
    return true;
}

// Phase 1 + phase 2 of one level-1/2 node with its 4 quadrants on 4 consecutive lanes (lane & 3 =
// quadrant): same decisions as phase1 / phase2_node, the fp64 quadrant tests in parallel.  Every
// lane of the warp must call it (ballots); lanes with !live take no part.  Returns the record on
// the group's quadrant-0 lane via acc / rec.
__device__ __forceinline__ void node_quad_lanes(const Win &w, const EncParams &p, bool live, int slot, int level,
                                                int nx, int ny, const Mom &m, const Mom *kids, bool try_node,
                                                bool &acc, uint64_t &rec) {
    const int lane = threadIdx.x & 31, quad = lane & 3;
    const int size = 32 >> level, nlog2 = 2 * (5 - level);
    acc = false;
    rec = 0;
    bool want2 = false, ok = false;
    int bit = 0;
    Node2 z{};
    if (live && try_node) {
        rec = phase1(w.x0 + 16 * slot + nx, w.y0 + ny, level, nlog2, m, p.p1b[level], acc);
        if (!acc && p.mns) {
            z = p2_node(nlog2, m.sr, kids[0].sr, kids[1].sr, kids[2].sr, kids[3].sr, level == 1 ? 15 : 31,
                        p.gate[level]);
            want2 = z.pass;
            if (want2) {
                const double slo = level == 1 ? 0.2 : 0.4, shi = level == 1 ? 0.5 : 0.65;
                const int h = size / 2;
                int res = p2_quad(nlog2 - 2, kids[quad], z.t[quad], slo, shi, p.p2b[level] * (double)(h * h), bit);
                if (res == 2)
                    res = emulate_quadrant(w, slot, nx + (quad & 1) * h, ny + (quad >> 1) * h, h, kids[quad],
                                           z.t[quad], slo, shi, p.tol[level], bit);
                ok = res == 1;
            }
        }
    }
    const unsigned okm = __ballot_sync(FULL, ok), bitm = __ballot_sync(FULL, bit != 0);
    const int g = lane & ~3;
    if (want2 && ((okm >> g) & 15u) == 15u) {
        acc = true;
        rec = mns_rec_phase2(w.x0 + 16 * slot + nx, w.y0 + ny, level, z.o, z.d0, z.d1, z.d2, (int)((bitm >> g) & 15u));
    }
}

// One try_phase1 / try_phase2 call (encoder.py:145-212) on the node (x, y, 32 >> level) of a
// W x H image: the packed record (0 = rejected) and the reference's rms -- phase 1: sqrt of the
// exact mean squared residual (every term is dyadic), phase 2: the worst chosen quadrant rms,
// replayed in the reference's fp64 order, or +inf on rejection.  One CTA stages an 80-row window
// from the node's 16-aligned origin - 16 (it holds the node and its co-centred domains even for
// rects not aligned to their size); thread 0 decides.
constexpr int NODE_WIN_H = 80;
__global__ void try_node_kernel(const uint8_t *img, int W, int H, int64_t pitch, int x, int y, int level, int phase,
                                const EncParams p, uint64_t *out_rec, double *out_rms) {
    __shared__ uint8_t pix[NODE_WIN_H][WIN_W];
    __shared__ uint16_t qe[NODE_WIN_H / 2][QE_W];
    __shared__ double sq_buf[256];
    const int x0 = x & ~15, y0 = y & ~15, wx0 = x0 - 16, wy0 = y0 - 16;
    for (int i = threadIdx.x; i < NODE_WIN_H * WIN_W; i += blockDim.x) {
        const int r = i / WIN_W, c = i % WIN_W, gy = wy0 + r, gx = wx0 + c;
        pix[r][c] = (gy >= 0 && gy < H && gx >= 0 && gx < W) ? img[(size_t)gy * pitch + gx] : 0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < NODE_WIN_H / 2 * QE_WL; i += blockDim.x) {
        const int qi = i / QE_WL, qj = i % QE_WL;
        qe[qi][qj] = (uint16_t)(pix[2 * qi][2 * qj] + pix[2 * qi][2 * qj + 1] + pix[2 * qi + 1][2 * qj] +
                                pix[2 * qi + 1][2 * qj + 1]);
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const Win w{pix, qe, x0, y0, wx0, wy0, W, H};
    const int size = 32 >> level, nx = x - x0, ny = y - y0, nlog2 = 2 * (5 - level);
    auto moments = [&](int cx, int cy, int cs) {
        Mom m{0, 0, 0, 0, 0};
        for (int i = 0; i < cs; i++)
            for (int j = 0; j < cs; j++) {
                const int q = dom_q(w, 0, cx, cy, cs, cx + j, cy + i), r = pixel(w, 0, cx + j, cy + i);
                m.sr += r;
                m.srr += r * r;
                m.sq += q;
                m.sqq += q * q;
                m.sqr += q * r;
            }
        return m;
    };
    if (phase == 1) {
        const Mom m = moments(nx, ny, size);
        bool acc;
        const uint64_t rec = phase1(x, y, level, nlog2, m, p.p1b[level], acc);
        const long long n = 1ll << nlog2;
        const int o = (2 * m.sr + (int)n) >> (nlog2 + 1);
        const int code = (int)((rec >> MNS_REC_PAYLOAD_SHIFT) & 7);  // the record's contrast code
        const double sdq = -0.875 + 0.25 * code, dm = ((double)m.sq * 0.25) / (double)n;
        for (int i = 0; i < size; i++)  // rms_error replayed in numpy's fp64 order (exact in practice)
            for (int j = 0; j < size; j++)
                sq_buf[i * size + j] = emu_sq(pixel(w, 0, nx + j, ny + i), dom_q(w, 0, nx, ny, size, nx + j, ny + i),
                                              dm, sdq, (double)o);
        *out_rec = acc ? rec : 0;
        *out_rms = __dsqrt_rn(pw_sum_dev(sq_buf, (int)n) / (double)n);
        return;
    }
    const int h = size / 2;
    Mom kids[4];
    for (int k = 0; k < 4; k++) kids[k] = moments(nx + (k & 1) * h, ny + (k >> 1) * h, h);
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
        if (!emulate_quadrant(w, 0, nx + (k & 1) * h, ny + (k >> 1) * h, h, kids[k], z.t[k], slo, shi, p.tol[level], bit,
                              &rms))
            return;
        bits |= bit << k;
        worst = fmax(worst, rms);
    }
    *out_rec = mns_rec_phase2(x, y, level, z.o, z.d0, z.d1, z.d2, bits);
    *out_rms = worst;
}

__global__ void __launch_bounds__(ET, 4) mns_encode_kernel(const __grid_constant__ CUtensorMap tmap,
                                                           const EncParams p) {
    extern __shared__ __align__(128) unsigned char esm[];
    TileSmem &ts = *reinterpret_cast<TileSmem *>(esm);
    uint8_t(*pix)[WIN_W] = reinterpret_cast<uint8_t(*)[WIN_W]>(esm + TILE_SMEM);
    uint16_t(*qe)[QE_W] = reinterpret_cast<uint16_t(*)[QE_W]>(esm + TILE_SMEM + WIN_H * WIN_W);
    __shared__ __align__(8) uint64_t wbar;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int img_i = blockIdx.z;
    const int ry = p.rr0 + blockIdx.y;
    const int rx0 = blockIdx.x * TR;
    const int nr = min(TR, p.rw - rx0);
    const int x0 = rx0 * 16, y0 = ry * 16;
    const int wx0 = x0 - 16, wy0 = y0 - 16;
    const Win w{pix, qe, x0, y0, wx0, wy0, p.W, p.H};

    // ---- K1a: stage the pixel window with one TMA box (the image viewed as u16 pairs, so a
    // 288-byte window row is one 144-element box row; out-of-image bytes are zero-filled)
    if (tid == 0) {
        mbar_init(&wbar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(&wbar, WIN_H * WIN_W);
        tma_load_3d(&pix[0][0], &tmap, wx0 / 2, wy0 - p.y_res0, img_i, &wbar);
    }
    __syncthreads();
    mbar_wait(&wbar, 0);
    // ---- K1b: even-phase 2x2 sums, 4 per thread-step via packed u16x2 adds
    for (int c = tid; c < QE_H * (QE_WL / 4); c += ET) {
        const int qi = c / (QE_WL / 4), qj = (c % (QE_WL / 4)) * 4;
        const uint2 a = *reinterpret_cast<const uint2 *>(&pix[2 * qi][2 * qj]);
        const uint2 b = *reinterpret_cast<const uint2 *>(&pix[2 * qi + 1][2 * qj]);
        // bytes 0, 2 and 1, 3 of each word zero-extended into u16 lanes (PRMT), summed lane-wise
        uint2 s;
        s.x = (__byte_perm(a.x, 0u, 0x4240) + __byte_perm(a.x, 0u, 0x4341)) +
              (__byte_perm(b.x, 0u, 0x4240) + __byte_perm(b.x, 0u, 0x4341));
        s.y = (__byte_perm(a.y, 0u, 0x4240) + __byte_perm(a.y, 0u, 0x4341)) +
              (__byte_perm(b.y, 0u, 0x4240) + __byte_perm(b.y, 0u, 0x4341));
        *reinterpret_cast<uint2 *>(&qe[qi][qj]) = s;
    }
    __syncthreads();

    const bool try1 = p.root_level == 1 && p.min_dim >= 32;  // encoder.py:231 guard 2*size <= min_dim
    // ---- K1c: block moments of every level-1..3 node.  Lane = one 4x4 level-3 node (16 pixels);
    // half-warps take the warp's two roots (slots warp, warp + EW) in one pass.  Level-2 sums over 4
    // lanes, level-1 sums over the half-warp (its Sr, Srr from the level-2 partials).
    {
        const int hw = lane >> 4, m = lane & 15;
        const int slot = warp + EW * hw;
        const bool live = slot < nr;
        const int sl = live ? slot : 0;
        const int lx = node3_x(m), ly = node3_y(m);
        int r[16];
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const uint32_t wd = *reinterpret_cast<const uint32_t *>(&pix[16 + ly + i][16 + 16 * sl + lx]);
#pragma unroll
            for (int j = 0; j < 4; j++) r[4 * i + j] = (wd >> (8 * j)) & 0xFF;
        }
        // 2x2 cell sums (level-4 ranges, Morton order inside the node) and the node's Sr, Srr
        int sr3 = 0, srr3 = 0;
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const int i0 = 2 * (c >> 1), j0 = 2 * (c & 1);
            const int a0 = r[4 * i0 + j0], a1 = r[4 * i0 + j0 + 1], a2 = r[4 * i0 + 4 + j0], a3 = r[4 * i0 + 5 + j0];
            const int cs = a0 + a1 + a2 + a3, css = a0 * a0 + a1 * a1 + a2 * a2 + a3 * a3;
            if (live) {
                ts.sr4[slot][4 * m + c] = cs;
                ts.srr4[slot][4 * m + c] = css;
            }
            sr3 += cs;
            srr3 += css;
        }
        // q-moments of the lane's 16 pixels against the domain of node (nx, ny, s)
        auto part = [&](int nx, int ny, int s, int &sq, int &sqq, int &sqr) {
            const int gdx = clampi(x0 + 16 * sl + nx - s / 2, 0, p.W - 2 * s);
            const int gdy = clampi(y0 + ny - s / 2, 0, p.H - 2 * s);
            const uint16_t *qp = &qe[(gdy - wy0) / 2 + (ly - ny)][(gdx - wx0) / 2 + (lx - nx)];
            sq = sqq = sqr = 0;
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int q = qp[i * QE_W + j];
                    sq += q;
                    sqq += q * q;
                    sqr += q * r[4 * i + j];
                }
        };
        int sq, sqq, sqr;
        part(lx, ly, 4, sq, sqq, sqr);  // level 3: the lane is the node
        if (live) ts.m3[slot][m] = Mom{sr3, srr3, sq, sqq, sqr};
        // level 2 (4-lane groups)
        const int k2 = m >> 2;
        int v[5] = {sr3, srr3, 0, 0, 0};
        part(node2_x(k2), node2_y(k2), 8, v[2], v[3], v[4]);
#pragma unroll
        for (int k = 0; k < 5; k++) {
            v[k] += __shfl_xor_sync(FULL, v[k], 1);
            v[k] += __shfl_xor_sync(FULL, v[k], 2);
        }
        if (live && (m & 3) == 0) ts.m2[slot][k2] = Mom{v[0], v[1], v[2], v[3], v[4]};
        // level 1 (half-warp): Sr, Srr from the level-2 sums, the q-moments from the lanes
        int u[5] = {v[0], v[1], 0, 0, 0};
        if (try1) part(0, 0, 16, u[2], u[3], u[4]);
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
        if (live && m == 0) ts.m1[slot] = Mom{u[0], u[1], u[2], u[3], u[4]};
    }
    __syncwarp();

    // ---- K2: decisions.  Round 1 (warp-local: warp w owns root slots w, w + EW): the 8 level-2
    // nodes of its roots x 4 quadrant lanes (a node is decided whether or not a parent accepts --
    // the emission's visibility flags discard covered decisions); round 2 (warp-local): the level-3
    // nodes not covered by a level-2 leaf (and the level-4 quartets below them), one per lane;
    // round 3 (CTA-wide, warps 0-1): the level-1 roots.
    const bool mns = p.mns != 0;
    {  // round 1: the 8 level-2 nodes of this warp's two roots x 4 quadrant lanes
        const int node = lane >> 2, s = warp + EW * (node >> 2), k = node & 3;
        const bool live = s < nr;
        const int sc = live ? s : 0;
        bool acc;
        uint64_t rec;
        node_quad_lanes(w, p, live, sc, 2, node2_x(k), node2_y(k), ts.m2[sc][k], &ts.m3[sc][4 * k], true, acc, rec);
        if (live && (lane & 3) == 0) {
            ts.acc2[s][k] = acc;
            ts.rec2[s][k] = rec;
        }
    }
    __syncwarp();
    {
        const int s = warp + EW * (lane >> 4), m = lane & 15;
        if (s < nr) {
            const bool vis = !ts.acc2[s][m >> 2];  // a level-1 acceptance is applied at the emission
            bool acc = false;
            uint64_t rec = 0;
            if (vis) {
                const int nx = node3_x(m), ny = node3_y(m);
                rec = phase1(x0 + 16 * s + nx, y0 + ny, 3, 4, ts.m3[s][m], p.p1b[3], acc);
                if (!acc) {  // level-4 moments (odd-phase domains) of the 4 children, then phase 2 / split
                    Mom k4[4];
                    for (int c = 0; c < 4; c++) {
                        const int cx = nx + 2 * (c & 1), cy = ny + 2 * (c >> 1);
                        Mom mm{ts.sr4[s][4 * m + c], ts.srr4[s][4 * m + c], 0, 0, 0};
                        for (int i = 0; i < 2; i++)
                            for (int j = 0; j < 2; j++) {
                                const int q = dom_q(w, s, cx, cy, 2, cx + j, cy + i);
                                mm.sq += q;
                                mm.sqq += q * q;
                                mm.sqr += q * pixel(w, s, cx + j, cy + i);
                            }
                        k4[c] = mm;
                    }
                    if (mns) acc = phase2_node(w, p, s, 3, nx, ny, 4, ts.m3[s][m].sr, k4, &rec);
                    if (!acc)
                        for (int c = 0; c < 4; c++) {
                            bool dummy;
                            ts.rec4[s][4 * m + c] = phase1(x0 + 16 * s + nx + 2 * (c & 1), y0 + ny + 2 * (c >> 1), 4,
                                                           2, k4[c], INFINITY, dummy);
                        }
                }
            }
            ts.acc3[s][m] = acc;
            ts.rec3[s][m] = rec;
        }
    }
    // round 3: the level-1 roots of the whole tile, 16 roots x 4 quadrant lanes on warps 0-1 (every
    // lane busy, instead of 8 lanes of every warp); the other warps wait at the emission barrier
    __syncthreads();
    if (warp < 2) {
        const int s = 8 * warp + (lane >> 2);
        const bool live = s < nr;
        const int sc = live ? s : 0;
        bool acc;
        uint64_t rec;
        node_quad_lanes(w, p, live, sc, 1, 0, 0, ts.m1[sc], ts.m2[sc], try1, acc, rec);
        if (live && (lane & 3) == 0) {
            ts.acc1[s] = acc;
            ts.rec1[s] = rec;
        }
    }
    __syncthreads();

    // ---- K2b: DFS (Morton) emission.  Half-warps take the warp's two roots in one pass; lane m
    // owns level-3 node m (cells 4m..4m+3): the covering leaf's record on the first lane it covers,
    // or the node's four level-4 records; offsets by two ballots (records per lane: 0, 1 or 4).
    {
        const int hw = lane >> 4, m = lane & 15, a = m >> 2;
        const int slot = warp + EW * hw;
        const bool live = slot < nr;
        const int sl = live ? slot : 0;
        const bool vis1 = p.root_level == 1;
        const bool acc1 = ts.acc1[sl];
        const bool vis2 = !vis1 || !acc1;
        const bool acc2 = ts.acc2[sl][a];
        const bool vis3 = vis2 && !acc2;
        const bool acc3 = ts.acc3[sl][m];
        const bool vis4 = vis3 && !acc3;
        uint64_t cov;
        int nrec;
        if (vis1 && acc1) {
            nrec = m == 0;
            cov = ts.rec1[sl];
        } else if (vis2 && acc2) {
            nrec = (m & 3) == 0;
            cov = ts.rec2[sl][a];
        } else if (vis3 && acc3) {
            nrec = 1;
            cov = ts.rec3[sl][m];
        } else {
            nrec = 4;
            cov = ts.rec4[sl][4 * m];
        }
        if (!live) nrec = 0;
        const unsigned half = hw ? 0xFFFF0000u : 0x0000FFFFu, lt = lanemask_lt() & half;
        const unsigned b1 = __ballot_sync(FULL, nrec != 0) & half, b4 = __ballot_sync(FULL, nrec == 4) & half;
        const int off = __popc(b1 & lt) + 3 * __popc(b4 & lt);
        const long long root = (long long)img_i * p.rows * p.rw + (long long)(ry - p.rr0) * p.rw + rx0 + sl;
        if (live) {
            uint64_t *st = p.stage + root * 64 + off;
            if (nrec == 4) {
#pragma unroll
                for (int c = 0; c < 4; c++) st[c] = ts.rec4[sl][4 * m + c];
            } else if (nrec) {
                st[0] = cov;
            }
            if (m == 0) p.root_cnt[root] = __popc(b1) + 3 * __popc(b4);
            if (p.unit_map) {
                const int rxg = x0 + 16 * sl, lx = node3_x(m), ly = node3_y(m);
                uint2 u;
                if (vis4) {
                    u.x = (uint32_t)mns_unit_of_record(ts.rec4[sl][4 * m], rxg, y0, lx, ly) |
                          ((uint32_t)mns_unit_of_record(ts.rec4[sl][4 * m + 1], rxg, y0, lx + 2, ly) << 16);
                    u.y = (uint32_t)mns_unit_of_record(ts.rec4[sl][4 * m + 2], rxg, y0, lx, ly + 2) |
                          ((uint32_t)mns_unit_of_record(ts.rec4[sl][4 * m + 3], rxg, y0, lx + 2, ly + 2) << 16);
                } else {
                    u.x = mns_unit_pair_of_record(cov, rxg, y0, lx, ly);
                    u.y = mns_unit_pair_of_record(cov, rxg, y0, lx, ly + 2);
                }
                *reinterpret_cast<uint2 *>(&p.unit_map[root * 32 + 2 * m]) = u;
            }
        }
    }
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
    MNS_CHECK_ARG(n_images <= 65535 && p.rows <= 65535, "grid too large");
    CUtensorMap tmap{};
    if (encode_tmap_3d(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT16, img + (ptrdiff_t)p.y_res0 * pitch, (uint64_t)W / 2,
                       (uint64_t)(y_res1 - p.y_res0), (uint64_t)n_images, (uint64_t)pitch,
                       (uint64_t)(n_images > 1 ? image_stride : pitch * (int64_t)(y_res1 - p.y_res0)), WIN_W / 2,
                       WIN_H, 1))
        return -1;
    const dim3 grid((unsigned)p.tiles_per_row, (unsigned)p.rows, (unsigned)n_images);
    mns_encode_kernel<<<grid, ET, ENC_SMEM, stream>>>(tmap, p);
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
