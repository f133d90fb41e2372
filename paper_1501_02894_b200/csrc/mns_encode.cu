// MNS quadtree encoder for sm_100a: block moments (K1) + phase-1/phase-2 matcher
// with DFS compaction (K2) in ONE single-pass kernel.
//
// Replaces the reference's per-node Python recursion
//   encoder.py:215-246 encode_quadtree / visit, :145-166 try_phase1,
//   :169-212 try_phase2, image.py:146-187 block helpers, transform.py:23-80.
//
// Work decomposition: one CTA = up to 8 consecutive 16x16 roots of one root row
// (one warp per root).  The CTA stages the uint8 window [x0-16, x0+144) x
// [y0-16, y0+32) (every clamped domain of every node of its roots lies inside,
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
//   compacts its root with two ballots; CTAs chain with a decoupled look-back.

#include <math.h>

#include "mns_common.cuh"

namespace mns {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int EW = 8;                // warps per CTA
constexpr int ET = EW * 32;
constexpr int RPW = 4;               // roots encoded by each warp per tile (in turn)
constexpr int TR = EW * RPW;         // 32 consecutive roots of one root row per tile
constexpr int WIN_W = TR * 16 + 32;  // 544
constexpr int WIN_H = 48;
constexpr int QE_W = WIN_W / 2;      // 272
constexpr int QE_H = WIN_H / 2;      // 24
constexpr int ENC_SMEM = WIN_H * WIN_W + QE_H * QE_W * 2 + EW * 2 * 64 * 8 + TR * 64 * 8;

struct EncParams {
    const uint8_t *img;
    int64_t pitch, image_stride;
    int W, H, n_images, rr0, rows, rw, tiles_per_row;
    int mns, root_level, min_dim;
    double p1b[5];  // phase-1 accept bound on 1024*n*SSE per level (inf for level 4)
    double p2b[4];  // bound(E_level): phase-2 quadrant accepts iff SSE <= n_k * p2b
    double tol[4];  // E_level (emulation path compares rms > tol like the reference)
    double mean_tol;
    uint64_t *out;
    uint32_t *unit_map;  // optional: decoder unit map (mns_record.h), 32 words per root
    int32_t *root_offsets;
    int64_t *count;
    unsigned long long *status;
    long long n_tiles, n_roots;
};

struct Mom {
    int sr, srr, sq, sqq, sqr;
};

__device__ __forceinline__ int xsum(int v, int G) {
    for (int o = 1; o < G; o <<= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// 2^-k as an exact double
__device__ __forceinline__ double pow2neg(int k) { return __longlong_as_double((long long)(1023 - k) << 52); }

// Quantised contrast code = 4 + clamp(floor(16N/D), -4, 3) (4 when D == 0): the
// reference's quantize_contrast(fl(4N/D)) (transform.py:46-53), exactly.  A fast
// fp32 quotient is corrected by one exact int64 comparison (its error is < 1 unit).
__device__ __forceinline__ int quant_code(long long N, long long D) {
    if (D == 0) return 4;  // fit_affine degenerate domain: s = 0 -> bin 4
    const long long t = 16 * N;
    int k = (int)floorf(fminf(3.f, fmaxf(-4.f, __fdividef((float)t, (float)D))));
    if (k > -4 && t < (long long)k * D) --k;
    else if (k < 3 && t >= (long long)(k + 1) * D) ++k;
    return 4 + k;
}

// Phase 1 from exact integer moments (encoder.py:145-166 + transform.py:23-80).
__device__ __forceinline__ uint64_t phase1(int x, int y, int level, int nlog2, const Mom &m, double bnd,
                                           bool &acc) {
    const long long n = 1ll << nlog2;
    const int o = (2 * m.sr + (int)n) >> (nlog2 + 1);  // round_to_int(mean)
    const long long N = n * m.sqr - (long long)m.sq * m.sr;
    const long long D = n * m.sqq - (long long)m.sq * m.sq;
    const int code = quant_code(N, D);
    const long long k2 = 2 * code - 7;
    const long long A = (long long)m.srr - 2ll * o * m.sr + n * o * o;
    const long long X = 1024ll * n * A - 64ll * k2 * N + k2 * k2 * D;
    acc = (double)X <= bnd;
    return mns_rec_phase1(x, y, level, o, code);
}

// Phase-2 quadrant decision from moments: 0 reject, 1 accept, 2 ambiguous (emulate).
__device__ __forceinline__ int p2_quad(int nlog2, const Mom &m, int t, double slo, double shi, double bnd_n,
                                       int &bit) {
    const long long n = 1ll << nlog2;
    const long long A = (long long)m.srr - 2ll * t * m.sr + n * t * t;
    const long long N = n * m.sqr - (long long)m.sq * m.sr;
    const long long D = n * m.sqq - (long long)m.sq * m.sq;
    bit = 0;
    if (D == 0) return (double)A <= bnd_n ? 1 : 0;  // d - mean(d) == 0: both candidates identical
    const double X = (double)N * pow2neg(nlog2 + 2);  // sum (r - t)(d - dbar), exact
    const double Y = (double)D * pow2neg(nlog2 + 4);  // sum (d - dbar)^2, exact
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

__device__ __forceinline__ Node2 p2_node(int nlog2, int sr, int s0, int s1, int s2, int s3, int limit,
                                         double mean_tol) {
    Node2 z;
    const int n = 1 << nlog2;
    const int df[4] = {4 * s0 - sr, 4 * s1 - sr, 4 * s2 - sr, 4 * s3 - sr};  // n * (O_k - O_i)
    z.pass = true;
    for (int k = 0; k < 4; k++)
        if ((double)abs(df[k]) > mean_tol * (double)n) z.pass = false;  // encoder.py:187
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

__global__ void __launch_bounds__(ET, 3) mns_encode_kernel(const EncParams p) {
    extern __shared__ __align__(16) unsigned char esm[];
    uint64_t(*stage)[64] = reinterpret_cast<uint64_t(*)[64]>(esm);  // per-root records, DFS order
    double(*scratch)[2][64] = reinterpret_cast<double(*)[2][64]>(esm + TR * 64 * 8);
    uint8_t(*pix)[WIN_W] = reinterpret_cast<uint8_t(*)[WIN_W]>(esm + TR * 64 * 8 + EW * 2 * 64 * 8);
    uint16_t(*qe)[QE_W] =
        reinterpret_cast<uint16_t(*)[QE_W]>(esm + TR * 64 * 8 + EW * 2 * 64 * 8 + WIN_H * WIN_W);
    __shared__ int root_cnt[TR];
    __shared__ long long root_base[TR];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long long tile = blockIdx.x;
    const int per_img = p.rows * p.tiles_per_row;
    const int img_i = (int)(tile / per_img);
    const int rem = (int)(tile % per_img);
    const int ry = p.rr0 + rem / p.tiles_per_row;
    const int rx0 = (rem % p.tiles_per_row) * TR;
    const int nr = min(TR, p.rw - rx0);
    const uint8_t *img = p.img + (size_t)img_i * p.image_stride;
    const int x0 = rx0 * 16, y0 = ry * 16;
    const int wx0 = x0 - 16, wy0 = y0 - 16;

    // ---- K1a: stage the pixel window (16-byte coalesced loads, zero outside the image)
    constexpr int CH = WIN_W / 16;
    for (int c = tid; c < WIN_H * CH; c += ET) {
        const int wr = c / CH, wc = (c % CH) * 16;
        const int gy = wy0 + wr, gx = wx0 + wc;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (gy >= 0 && gy < p.H && gx >= 0 && gx < p.W)
            v = __ldg(reinterpret_cast<const uint4 *>(img + (size_t)gy * p.pitch + gx));
        *reinterpret_cast<uint4 *>(&pix[wr][wc]) = v;
    }
    __syncthreads();
    // ---- K1b: even-phase 2x2 sums, 4 per thread-step via packed u16x2 adds
    for (int c = tid; c < QE_H * (QE_W / 4); c += ET) {
        const int qi = c / (QE_W / 4), qj = (c % (QE_W / 4)) * 4;
        const uint2 a = *reinterpret_cast<const uint2 *>(&pix[2 * qi][2 * qj]);
        const uint2 b = *reinterpret_cast<const uint2 *>(&pix[2 * qi + 1][2 * qj]);
        uint2 s;
        s.x = (a.x & 0x00FF00FFu) + ((a.x >> 8) & 0x00FF00FFu) + (b.x & 0x00FF00FFu) + ((b.x >> 8) & 0x00FF00FFu);
        s.y = (a.y & 0x00FF00FFu) + ((a.y >> 8) & 0x00FF00FFu) + (b.y & 0x00FF00FFu) + ((b.y >> 8) & 0x00FF00FFu);
        *reinterpret_cast<uint2 *>(&qe[qi][qj]) = s;
    }
    __syncthreads();

    // ---- each warp encodes roots warp, warp + 8, ... of the tile: K1c moments + K2 decisions
    for (int rr = 0; rr < RPW; rr++) {
    const int slot = rr * EW + warp;
    if (slot >= nr) break;
    uint64_t recA = 0, recB = 0;
    bool hasA = false, hasB = false;
    uint32_t umap = 0;
    {
        const int rxg = x0 + slot * 16, ryg = y0;
        const int wrx = 16 + slot * 16, wry = 16;
        const int a = lane >> 3, b = (lane >> 1) & 3, c = lane & 1;
        const int ax = (a & 1) * 8, ay = (a >> 1) * 8, bx = (b & 1) * 4, by = (b >> 1) * 4;
        const int lx = ax + bx, ly = ay + by + 2 * c;  // lane's 2x4 pixel block (root-relative)
        const int W = p.W, H = p.H;

        int r[8];
        {
            const uint32_t w0 = *reinterpret_cast<const uint32_t *>(&pix[wry + ly][wrx + lx]);
            const uint32_t w1 = *reinterpret_cast<const uint32_t *>(&pix[wry + ly + 1][wrx + lx]);
#pragma unroll
            for (int j = 0; j < 4; j++) {
                r[j] = (w0 >> (8 * j)) & 0xFF;
                r[4 + j] = (w1 >> (8 * j)) & 0xFF;
            }
        }
        Mom m4L, m4R;
        m4L.sr = r[0] + r[1] + r[4] + r[5];
        m4R.sr = r[2] + r[3] + r[6] + r[7];
        m4L.srr = r[0] * r[0] + r[1] * r[1] + r[4] * r[4] + r[5] * r[5];
        m4R.srr = r[2] * r[2] + r[3] * r[3] + r[6] * r[6] + r[7] * r[7];
        Mom m3, m2, m1;  // range sums of the lane's level-3 / level-2 / level-1 node
        m3.sr = m4L.sr + m4R.sr;
        m3.srr = m4L.srr + m4R.srr;
        m3.sr += __shfl_xor_sync(FULL, m3.sr, 1);
        m3.srr += __shfl_xor_sync(FULL, m3.srr, 1);
        m2.sr = m3.sr + __shfl_xor_sync(FULL, m3.sr, 2);
        m2.srr = m3.srr + __shfl_xor_sync(FULL, m3.srr, 2);
        m2.sr += __shfl_xor_sync(FULL, m2.sr, 4);
        m2.srr += __shfl_xor_sync(FULL, m2.srr, 4);
        m1.sr = m2.sr + __shfl_xor_sync(FULL, m2.sr, 8);
        m1.srr = m2.srr + __shfl_xor_sync(FULL, m2.srr, 8);
        m1.sr += __shfl_xor_sync(FULL, m1.sr, 16);
        m1.srr += __shfl_xor_sync(FULL, m1.srr, 16);

        // even-phase moments of this lane's 8 pixels against the domain of node (nx, ny, s)
        auto even_moments = [&](int nx, int ny, int s, Mom &m) {
            const int gdx = clampi(rxg + nx - s / 2, 0, W - 2 * s);
            const int gdy = clampi(ryg + ny - s / 2, 0, H - 2 * s);
            const int qr = (gdy - wy0) / 2 + (ly - ny), qc = (gdx - wx0) / 2 + (lx - nx);
            int sq = 0, sqq = 0, sqr = 0;
#pragma unroll
            for (int i = 0; i < 2; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int q = qe[qr + i][qc + j];
                    sq += q;
                    sqq += q * q;
                    sqr += q * r[4 * i + j];
                }
            m.sq = sq;
            m.sqq = sqq;
            m.sqr = sqr;
        };
        auto even_q = [&](int nx, int ny, int s, int i, int j) -> int {
            const int gdx = clampi(rxg + nx - s / 2, 0, W - 2 * s);
            const int gdy = clampi(ryg + ny - s / 2, 0, H - 2 * s);
            return qe[(gdy - wy0) / 2 + (ly - ny) + i][(gdx - wx0) / 2 + (lx - nx) + j];
        };
        // level-4 node at (nx, ly): 2x2 range, 4x4 domain (odd phase in the interior)
        auto l4_q = [&](int nx, int i, int j) -> int {
            const int gdx = clampi(rxg + nx - 1, 0, W - 4), gdy = clampi(ryg + ly - 1, 0, H - 4);
            const uint8_t *pp = &pix[gdy - wy0 + 2 * i][gdx - wx0 + 2 * j];
            return (int)pp[0] + pp[1] + pp[WIN_W] + pp[WIN_W + 1];
        };
        auto l4_moments = [&](int nx, int ro, Mom &m) {
            int sq = 0, sqq = 0, sqr = 0;
#pragma unroll
            for (int i = 0; i < 2; i++)
#pragma unroll
                for (int j = 0; j < 2; j++) {
                    const int q = l4_q(nx, i, j);
                    sq += q;
                    sqq += q * q;
                    sqr += q * r[4 * i + ro + j];
                }
            m.sq = sq;
            m.sqq = sqq;
            m.sqr = sqr;
        };

        const bool mns = p.mns != 0;
        const bool vis1 = p.root_level == 1;
        const bool try1 = vis1 && p.min_dim >= 32;  // encoder.py:231 guard 2*size <= min_dim
        bool acc1 = false;
        uint64_t rec1 = 0;
        if (try1) {
            even_moments(0, 0, 16, m1);
            m1.sq = xsum(m1.sq, 32);
            m1.sqq = xsum(m1.sqq, 32);
            m1.sqr = xsum(m1.sqr, 32);
            rec1 = phase1(rxg, ryg, 1, 8, m1, p.p1b[1], acc1);
        }
        // level-2 moments: needed unless the root was accepted by phase 1
        if (!acc1) {
            even_moments(ax, ay, 8, m2);
            m2.sq = xsum(m2.sq, 8);
            m2.sqq = xsum(m2.sqq, 8);
            m2.sqr = xsum(m2.sqr, 8);
        }
        // ---- phase 2 at level 1 (node = root, quadrants = level-2 nodes)
        if (try1 && !acc1 && mns) {
            const Node2 z = p2_node(8, m1.sr, __shfl_sync(FULL, m2.sr, 0), __shfl_sync(FULL, m2.sr, 8),
                                    __shfl_sync(FULL, m2.sr, 16), __shfl_sync(FULL, m2.sr, 24), 15, p.mean_tol);
            if (z.pass) {  // warp-uniform
                int bit;
                int res = p2_quad(6, m2, z.t[a], 0.2, 0.5, p.p2b[1] * 64.0, bit);
                unsigned amb = __ballot_sync(FULL, res == 2 && (lane & 7) == 0);
                while (amb) {
                    const int g = __ffs(amb) - 1;
                    amb &= amb - 1;
                    if ((lane >> 3) == (g >> 3)) {
                        const double dm = ((double)m2.sq * 0.25) / 64.0;
                        const double t = (double)z.t[a];
#pragma unroll
                        for (int i = 0; i < 2; i++)
#pragma unroll
                            for (int j = 0; j < 4; j++) {
                                const int q = even_q(ax, ay, 8, i, j);
                                const int idx = (by + 2 * c + i) * 8 + bx + j;
                                scratch[warp][0][idx] = emu_sq(r[4 * i + j], q, dm, 0.2, t);
                                scratch[warp][1][idx] = emu_sq(r[4 * i + j], q, dm, 0.5, t);
                            }
                    }
                    __syncwarp();
                    int rr = 0, bb = 0;
                    if (lane == g) {
                        const double rlo = __dsqrt_rn(pw_sum_dev(scratch[warp][0], 64) / 64.0);
                        const double rhi = __dsqrt_rn(pw_sum_dev(scratch[warp][1], 64) / 64.0);
                        bb = rlo <= rhi ? 0 : 1;
                        rr = ((bb ? rhi : rlo) > p.tol[1]) ? 0 : 1;
                    }
                    rr = __shfl_sync(FULL, rr, g);
                    bb = __shfl_sync(FULL, bb, g);
                    if ((lane >> 3) == (g >> 3)) {
                        res = rr;
                        bit = bb;
                    }
                    __syncwarp();
                }
                if (__all_sync(FULL, res == 1)) {
                    const int bits = __shfl_sync(FULL, bit, 0) | (__shfl_sync(FULL, bit, 8) << 1) |
                                     (__shfl_sync(FULL, bit, 16) << 2) | (__shfl_sync(FULL, bit, 24) << 3);
                    acc1 = true;
                    rec1 = mns_rec_phase2(rxg, ryg, 1, z.o, z.d0, z.d1, z.d2, bits);
                }
            }
        }

        // ---- level 2
        const bool vis2 = vis1 ? !acc1 : true;
        bool acc2 = false;
        uint64_t rec2 = 0;
        if (vis2) rec2 = phase1(rxg + ax, ryg + ay, 2, 6, m2, p.p1b[2], acc2);
        if (__any_sync(FULL, vis2 && !acc2)) {
            even_moments(ax + bx, ay + by, 4, m3);
            m3.sq = xsum(m3.sq, 2);
            m3.sqq = xsum(m3.sqq, 2);
            m3.sqr = xsum(m3.sqr, 2);
        }
        const bool try2p2 = mns && vis2 && !acc2;
        if (__any_sync(FULL, try2p2)) {
            const int gb = lane & ~7;
            const Node2 z = p2_node(6, m2.sr, __shfl_sync(FULL, m3.sr, gb), __shfl_sync(FULL, m3.sr, gb + 2),
                                    __shfl_sync(FULL, m3.sr, gb + 4), __shfl_sync(FULL, m3.sr, gb + 6), 31,
                                    p.mean_tol);
            const bool go = try2p2 && z.pass;
            int bit = 0;
            int res = go ? p2_quad(4, m3, z.t[b], 0.4, 0.65, p.p2b[2] * 16.0, bit) : 0;
            unsigned amb = __ballot_sync(FULL, go && res == 2 && c == 0);
            while (amb) {
                const int g = __ffs(amb) - 1;
                amb &= amb - 1;
                if ((lane >> 1) == (g >> 1)) {
                    const double dm = ((double)m3.sq * 0.25) / 16.0;
                    const double t = (double)z.t[b];
#pragma unroll
                    for (int i = 0; i < 2; i++)
#pragma unroll
                        for (int j = 0; j < 4; j++) {
                            const int q = even_q(ax + bx, ay + by, 4, i, j);
                            const int idx = (2 * c + i) * 4 + j;
                            scratch[warp][0][idx] = emu_sq(r[4 * i + j], q, dm, 0.4, t);
                            scratch[warp][1][idx] = emu_sq(r[4 * i + j], q, dm, 0.65, t);
                        }
                }
                __syncwarp();
                int rr = 0, bb = 0;
                if (lane == g) {
                    const double rlo = __dsqrt_rn(pw_sum_dev(scratch[warp][0], 16) / 16.0);
                    const double rhi = __dsqrt_rn(pw_sum_dev(scratch[warp][1], 16) / 16.0);
                    bb = rlo <= rhi ? 0 : 1;
                    rr = ((bb ? rhi : rlo) > p.tol[2]) ? 0 : 1;
                }
                rr = __shfl_sync(FULL, rr, g);
                bb = __shfl_sync(FULL, bb, g);
                if ((lane >> 1) == (g >> 1)) {
                    res = rr;
                    bit = bb;
                }
                __syncwarp();
            }
            const unsigned okm = __ballot_sync(FULL, res == 1);
            const int bits = __shfl_sync(FULL, bit, gb) | (__shfl_sync(FULL, bit, gb + 2) << 1) |
                             (__shfl_sync(FULL, bit, gb + 4) << 2) | (__shfl_sync(FULL, bit, gb + 6) << 3);
            if (go && ((okm >> gb) & 0xFFu) == 0xFFu) {
                acc2 = true;
                rec2 = mns_rec_phase2(rxg + ax, ryg + ay, 2, z.o, z.d0, z.d1, z.d2, bits);
            }
        }

        // ---- level 3
        const bool vis3 = vis2 && !acc2;
        bool acc3 = false;
        uint64_t rec3 = 0;
        if (vis3) rec3 = phase1(rxg + ax + bx, ryg + ay + by, 3, 4, m3, p.p1b[3], acc3);
        if (__any_sync(FULL, vis3 && !acc3)) {
            l4_moments(lx, 0, m4L);
            l4_moments(lx + 2, 2, m4R);
        }
        const bool try3p2 = mns && vis3 && !acc3;
        if (__any_sync(FULL, try3p2)) {
            const int pb = lane & ~1;
            const Node2 z = p2_node(4, m3.sr, __shfl_sync(FULL, m4L.sr, pb), __shfl_sync(FULL, m4R.sr, pb),
                                    __shfl_sync(FULL, m4L.sr, pb + 1), __shfl_sync(FULL, m4R.sr, pb + 1), 31,
                                    p.mean_tol);
            const bool go = try3p2 && z.pass;
            int bitL = 0, bitR = 0, resL = 0, resR = 0;
            if (go) {
                resL = p2_quad(2, m4L, z.t[2 * c], 0.5, 0.9, p.p2b[3] * 4.0, bitL);
                resR = p2_quad(2, m4R, z.t[2 * c + 1], 0.5, 0.9, p.p2b[3] * 4.0, bitR);
                // in-register emulation for ambiguous 2x2 quadrants (n = 4: sequential sum)
                for (int side = 0; side < 2; side++) {
                    int &res = side ? resR : resL;
                    int &bit = side ? bitR : bitL;
                    if (res != 2) continue;
                    const Mom &m = side ? m4R : m4L;
                    const int nx = lx + 2 * side;
                    const double dm = ((double)m.sq * 0.25) / 4.0;
                    const double t = (double)z.t[2 * c + side];
                    double slo = 0.0, shi = 0.0;
                    for (int i = 0; i < 2; i++)
                        for (int j = 0; j < 2; j++) {
                            const int q = l4_q(nx, i, j);
                            const int rv = r[4 * i + 2 * side + j];
                            slo = __dadd_rn(slo, emu_sq(rv, q, dm, 0.5, t));
                            shi = __dadd_rn(shi, emu_sq(rv, q, dm, 0.9, t));
                        }
                    const double rlo = __dsqrt_rn(slo / 4.0), rhi = __dsqrt_rn(shi / 4.0);
                    bit = rlo <= rhi ? 0 : 1;
                    res = ((bit ? rhi : rlo) > p.tol[3]) ? 0 : 1;
                }
            }
            const bool lane_ok = resL == 1 && resR == 1;
            const int partner_ok = __shfl_xor_sync(FULL, (int)lane_ok, 1);  // every lane must shuffle
            const bool pair_ok = lane_ok && partner_ok;
            int lbits = (bitL << (2 * c)) | (bitR << (2 * c + 1));
            lbits |= __shfl_xor_sync(FULL, lbits, 1);
            if (go && pair_ok) {
                acc3 = true;
                rec3 = mns_rec_phase2(rxg + ax + bx, ryg + ay + by, 3, z.o, z.d0, z.d1, z.d2, lbits);
            }
        }

        // ---- level 4 (always accepts) and emission in Morton (= DFS) order
        const bool vis4 = vis3 && !acc3;
        if (vis1 && acc1) {
            hasA = lane == 0;
            recA = rec1;
        } else if (vis2 && acc2) {
            hasA = (lane & 7) == 0;
            recA = rec2;
        } else if (vis3 && acc3) {
            hasA = c == 0;
            recA = rec3;
        } else if (vis4) {
            bool dummy;
            hasA = hasB = true;
            recA = phase1(rxg + lx, ryg + ly, 4, 2, m4L, INFINITY, dummy);
            recB = phase1(rxg + lx + 2, ryg + ly, 4, 2, m4R, INFINITY, dummy);
        }
        if (p.unit_map) {  // the decoder's per-cell unit map for this lane's two cells
            const uint64_t cov = (vis1 && acc1) ? rec1 : (vis2 && acc2) ? rec2 : (vis3 && acc3) ? rec3 : recA;
            const uint64_t covB = vis4 ? recB : cov;
            umap = (uint32_t)mns_unit_of_record(cov, rxg, ryg, lx, ly) |
                   ((uint32_t)mns_unit_of_record(covB, rxg, ryg, lx + 2, ly) << 16);
        }
    }
    const unsigned bA = __ballot_sync(FULL, hasA), bB = __ballot_sync(FULL, hasB);
    const unsigned lt = lanemask_lt();
    const int offA = __popc(bA & lt) + __popc(bB & lt);
    if (hasA) stage[slot][offA] = recA;
    if (hasB) stage[slot][offA + (hasA ? 1 : 0)] = recB;
    if (lane == 0) root_cnt[slot] = __popc(bA) + __popc(bB);
    if (p.unit_map) {
        const long long root = (long long)img_i * p.rows * p.rw + (long long)(ry - p.rr0) * p.rw + rx0 + slot;
        p.unit_map[root * 32 + lane] = umap;
    }
    }  // roots of this warp
    __syncthreads();
    // ---- one decoupled look-back per 32 roots, then coalesced record copies
    if (warp == 0) {
        long long agg = 0;
        for (int k = 0; k < nr; k++) agg += root_cnt[k];
        const long long base = lookback_exclusive_warp(p.status, tile, agg);
        if (lane == 0) {
            const long long root0 = (long long)img_i * p.rows * p.rw + (long long)(ry - p.rr0) * p.rw + rx0;
            long long run = base;
            for (int k = 0; k < nr; k++) {
                root_base[k] = run;
                p.root_offsets[root0 + k] = (int32_t)run;
                run += root_cnt[k];
            }
            if (tile == p.n_tiles - 1) {
                p.root_offsets[p.n_roots] = (int32_t)run;
                *p.count = run;
            }
        }
    }
    __syncthreads();
    for (int k = warp; k < nr; k += EW) {
        const long long b0 = root_base[k];
        for (int i = lane; i < root_cnt[k]; i += 32) p.out[b0 + i] = stage[k][i];
    }
}

}  // namespace

int encode_workspace_bytes(int width, int n_images, int rr0, int rr1, int64_t *bytes) {
    const int rw = width / 16;
    const long long tiles = (long long)n_images * (rr1 - rr0) * ((rw + TR - 1) / TR);
    *bytes = tiles * 8;
    return 0;
}

int encode_quadtree(const uint8_t *img, int W, int H, int64_t pitch, int64_t image_stride, int n_images, int rr0,
                    int rr1, const mns_enc_cfg *cfg, uint64_t *records, int64_t capacity, int32_t *root_offsets,
                    int64_t *d_count, uint32_t *unit_map, void *workspace, int64_t workspace_bytes,
                    cudaStream_t stream) {
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

    EncParams p{};
    p.img = img;
    p.pitch = pitch;
    p.image_stride = image_stride;
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
    p.out = records;
    p.unit_map = unit_map;
    p.root_offsets = root_offsets;
    p.count = d_count;
    p.status = reinterpret_cast<unsigned long long *>(workspace);
    p.n_tiles = need / 8;
    p.n_roots = n_roots;
    MNS_CUDA_TRY(cudaMemsetAsync(workspace, 0, need, stream));
    static bool attr_set = false;
    if (!attr_set) {
        MNS_CUDA_TRY(cudaFuncSetAttribute(mns_encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ENC_SMEM));
        attr_set = true;
    }
    mns_encode_kernel<<<(unsigned)p.n_tiles, ET, ENC_SMEM, stream>>>(p);
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

}  // namespace mns
