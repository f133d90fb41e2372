// Full-search and local-search baselines (K3) for sm_100a.
//
// Replaces encoder.py:249-309 (encode_full_search) and :312-347
// (encode_local_search).  Exactness: with n = B^2, q = 2x2 pixel sums and
// integer moments, the reference's fp64 SSE is exact and
//     1024*n*SSE = 1024*n*A - 64*k2*N + k2^2*D,  N = n*Sqr - Sq*Sr, D = n*Sqq - Sq^2,
// with k2 = 2*code - 7 the quantised contrast; the quantiser picks the odd k2
// nearest 32N/D, which is the k2 minimising k2^2 D - 64 k2 N.  So the per-range
// argmin over (domain, isometry) with the reference's first-index tie-break is
// the lexicographic minimum of the 64-bit key (val + 2^(63-cb)) << cb | candidate
// (cb = key_cand_bits(n), mns_common.cuh).
//
// This file holds the CUDA-core paths (any B; the local search) and the shared
// domain-pool preparation / finalisation; the tcgen05 tensor-core GEMM for
// B in {4, 8} lives in mns_search_tc.cu.

#include <math.h>
#include <stdlib.h>

#include "mns_common.cuh"

namespace mns {

namespace {

constexpr unsigned FULL = 0xffffffffu;

// min over odd k2 in [-7, 7] of k2^2 D - 64 k2 N (exact, int64)
__device__ __forceinline__ long long best_val(long long N, long long D) {
    if (D == 0) return 0;  // N == 0 whenever D == 0
    const double t = 32.0 * (double)N / (double)D;
    int k = 2 * (int)floor(fmin(8.0, fmax(-8.0, t)) * 0.5) + 1;
    long long best = LLONG_MAX;
#pragma unroll
    for (int dk = -2; dk <= 2; dk += 2) {
        long long k2 = k + dk;
        if (k2 < -7 || k2 > 7) continue;
        const long long v = k2 * k2 * D - 64 * k2 * N;
        best = v < best ? v : best;
    }
    return best;
}

__device__ __forceinline__ int quant_code(long long N, long long D) {
    if (D == 0) return 4;
    double f = floor((double)(16 * N) / (double)D);
    f = fmin(3.0, fmax(-4.0, f));
    return 4 + (int)f;
}

__device__ __forceinline__ unsigned long long make_key(long long val, long long cand) {
    return ((unsigned long long)(val + (1ll << 42)) << 21) | (unsigned long long)cand;
}

// ---- domain pool: q values (u16, n per domain, raster order over the stride lattice), Sq, D.
//      One warp per domain: lanes own consecutive q (coalesced), Sq / Sqq by warp reduction.
__global__ void pool_kernel(const uint8_t *img, int W, int B, int step, int ndx, long long ndom, uint16_t *pool,
                            int32_t *psq, long long *pD) {
    const int n = B * B, lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long d = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); d < ndom; d += warps) {
        const int x = (int)(d % ndx) * step, y = (int)(d / ndx) * step;
        long long sq = 0, sqq = 0;
        for (int k = lane; k < n; k += 32) {
            const uint8_t *p = img + (size_t)(y + 2 * (k / B)) * W + x + 2 * (k % B);
            const int q = p[0] + p[1] + p[W] + p[W + 1];
            pool[d * n + k] = (uint16_t)q;
            sq += q;
            sqq += q * q;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sq += __shfl_xor_sync(FULL, sq, o);
            sqq += __shfl_xor_sync(FULL, sqq, o);
        }
        if (lane == 0) {
            psq[d] = (int32_t)sq;
            pD[d] = n * sqq - sq * sq;
        }
    }
}

// ---- CUDA-core exact full search: CTA = RT ranges x (domain chunk); thread = one domain at a time
template <int B>
__global__ void __launch_bounds__(256) full_search_cc_kernel(const uint8_t *img, int W, int n_iso, int r0, int r1,
                                                             const uint16_t *pool, const int32_t *psq,
                                                             const long long *pD, long long ndom,
                                                             unsigned long long *best) {
    constexpr int n = B * B;
    constexpr int RT = 8;  // ranges per CTA
    __shared__ uint8_t rsh[RT * 8][n];  // (range, iso) rows, permuted range pixels
    __shared__ int rsum[RT * 8];
    const int rpr = W / B;
    const int rbase = r0 + blockIdx.y * RT;
    const int nrows = RT * n_iso;
    for (int k = threadIdx.x; k < nrows * n; k += blockDim.x) {
        const int row = k / n, e = k % n;
        const int ri = rbase + row / n_iso, t = row % n_iso;
        if (ri < r1) {
            const int rx = (ri % rpr) * B, ry = (ri / rpr) * B;
            // row[src_t(e)] = r(e), so sum_m pool[m] * row[m] = sum_e d_t(e) * r(e)
            const int m = iso_src(t, e / B, e % B, B);
            rsh[row][m] = img[(size_t)(ry + e / B) * W + rx + e % B];
        }
    }
    __syncthreads();
    for (int row = threadIdx.x; row < nrows; row += blockDim.x) {
        int s = 0;
        for (int e = 0; e < n; e++) s += rsh[row][e];
        rsum[row] = s;
    }
    __syncthreads();
    unsigned long long local[RT * 8];
    for (int i = 0; i < nrows; i++) local[i] = ~0ull;
    for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < ndom;
         d += (long long)gridDim.x * blockDim.x) {
        constexpr int QN = n <= 64 ? n : 1;
        int q[QN];
        if constexpr (n <= 64) {
#pragma unroll
            for (int e = 0; e < n; e++) q[e] = pool[d * n + e];
        }
        const long long Sq = psq[d], D = pD[d];
        for (int row = 0; row < nrows; row++) {
            if (rbase + row / n_iso >= r1) break;
            int sqr = 0;
            if constexpr (n <= 64) {
#pragma unroll
                for (int e = 0; e < n; e++) sqr += q[e] * rsh[row][e];
            } else {
                for (int e = 0; e < n; e++) sqr += pool[d * n + e] * rsh[row][e];
            }
            const long long N = (long long)n * sqr - Sq * rsum[row];
            const long long v = best_val(N, D);
            const unsigned long long key = make_key_cb(v, d * n_iso + row % n_iso, key_cand_bits(n));
            local[row] = key < local[row] ? key : local[row];
        }
    }
    for (int row = 0; row < nrows; row++) {
        if (rbase + row / n_iso >= r1) break;
        unsigned long long k = local[row];
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long other = __shfl_xor_sync(FULL, k, o);
            k = other < k ? other : k;
        }
        if ((threadIdx.x & 31) == 0) atomicMin(&best[rbase + row / n_iso - r0], k);
    }
}

// merge isometry rows already folded via the key's candidate index; finalise code/o per range
// one warp per range: re-derive o_byte and the contrast code of the winning (domain, isometry)
__global__ void search_finalize_kernel(const uint8_t *img, int W, int B, int n_iso, int r0, int r1,
                                       const unsigned long long *best, const uint16_t *pool,
                                       const int32_t *psq, const long long *pD, int32_t *out_dom, int8_t *out_iso,
                                       uint8_t *out_o, uint8_t *out_code) {
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= r1 - r0) return;
    const int ri = r0 + i, n = B * B, rpr = W / B;
    const int rx = (ri % rpr) * B, ry = (ri / rpr) * B;
    const unsigned long long key = best[i];
    const long long cand = key_cand(key, key_cand_bits(n));
    const long long d = cand / n_iso;
    const int t = (int)(cand % n_iso);
    int sr = 0;
    long long sqr = 0;
    for (int e = lane; e < n; e += 32) {
        const int r = img[(size_t)(ry + e / B) * W + rx + e % B];
        sr += r;
        sqr += (long long)r * pool[d * n + iso_src(t, e / B, e % B, B)];
    }
    sr = __reduce_add_sync(FULL, sr);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sqr += __shfl_xor_sync(FULL, sqr, o);
    if (lane == 0) {
        const long long N = (long long)n * sqr - (long long)psq[d] * sr;
        out_dom[i] = (int32_t)d;
        out_iso[i] = (int8_t)t;
        out_o[i] = (uint8_t)((2 * sr + n) / (2 * n));
        out_code[i] = (uint8_t)quant_code(N, pD[d]);
    }
}

__global__ void fill_u64_kernel(unsigned long long *a, unsigned long long v, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        a[i] = v;
}

// ---- local search: CTA per 8x8 range; stride-1 2x2 sums of the candidate window in smem.
// NI isometries (1 = the reference, 8 = the extension): the range is stored once per isometry,
// permuted (rt[t][src_t(e)] = r(e)), so candidate (c, t)'s cross term is sum_m q_c(m) rt[t][m]; a
// thread keeps its candidate's 64 q values in registers across the isometries.  Winner = the
// lexicographic minimum of (1024 n SSE, c * NI + t): the reference's first strict '<' over the
// (dy, dx) order, then the lowest isometry.
// SEED: score only the candidates on a stride-`sstride` grid of offsets and fold the winner into
// the tensor-core path's keys (val = k2^2 D - 64 k2 N, candidate = domain * NI + t) -- a valid
// seed, every scored candidate being a real one.
template <int R, int NI, bool SEED = false>
__global__ void __launch_bounds__(256) local_search_kernel(const uint8_t *img, int W, int H, int radius,
                                                           int32_t *out_dx, int32_t *out_dy, int8_t *out_iso,
                                                           uint8_t *out_o, uint8_t *out_code,
                                                           unsigned long long *seed_best = nullptr,
                                                           int sstride = 1) {
    constexpr int WS = 16 + 2 * R;  // window side (pixels) covering every clamped candidate
    __shared__ uint16_t s2[WS][WS];
    __shared__ uint8_t pw[WS + 1][WS + 1];
    __shared__ int rt[NI][64];
    __shared__ uint32_t rtp[NI][16];  // rt packed 4 bytes per word (DP2A operands)
    __shared__ unsigned long long wbest[8];
    const int rpr = W / 8;
    const int ri = blockIdx.x;
    const int rx = (ri % rpr) * 8, ry = (ri / rpr) * 8;
    const int bx = clampi(rx - 4, 0, W - 16), by = clampi(ry - 4, 0, H - 16);
    // candidate origins lie in [clamp(b - radius), clamp(b + radius)]
    const int lo_x = clampi(bx - radius, 0, W - 16), lo_y = clampi(by - radius, 0, H - 16);
    const int hi_x = clampi(bx + radius, 0, W - 16), hi_y = clampi(by + radius, 0, H - 16);
    const int ww = hi_x - lo_x + 16, wh = hi_y - lo_y + 16;
    for (int k = threadIdx.x; k < wh * ww; k += blockDim.x) {
        const int i = k / ww, j = k % ww;
        pw[i][j] = img[(size_t)(lo_y + i) * W + lo_x + j];
    }
    for (int k = threadIdx.x; k < NI * 64; k += blockDim.x) {
        const int t = k / 64, e = k % 64;
        rt[t][iso_src(t, e / 8, e % 8, 8)] = img[(size_t)(ry + e / 8) * W + rx + e % 8];
    }
    __syncthreads();
    for (int k = threadIdx.x; k < (wh - 1) * (ww - 1); k += blockDim.x) {
        const int i = k / (ww - 1), j = k % (ww - 1);
        s2[i][j] = (uint16_t)(pw[i][j] + pw[i][j + 1] + pw[i + 1][j] + pw[i + 1][j + 1]);
    }
    for (int k = threadIdx.x; k < NI * 16; k += blockDim.x) {
        const int t = k / 16, w4 = 4 * (k % 16);
        rtp[t][k % 16] = (uint32_t)rt[t][w4] | ((uint32_t)rt[t][w4 + 1] << 8) | ((uint32_t)rt[t][w4 + 2] << 16) |
                         ((uint32_t)rt[t][w4 + 3] << 24);
    }
    __syncthreads();
    int sr = 0, srr = 0;
    for (int e = 0; e < 64; e++) {
        sr += rt[0][e];
        srr += rt[0][e] * rt[0][e];
    }
    const int o = (2 * sr + 64) / 128;
    const long long A = (long long)srr - 2ll * o * sr + 64ll * o * o;
    const int side = 2 * radius + 1;
    const int sside = SEED ? 2 * (radius / sstride) + 1 : side;  // scored grid
    unsigned long long best = ~0ull;
    for (int c = threadIdx.x; c < sside * sside; c += blockDim.x) {
        const int dy = SEED ? (c / sside - radius / sstride) * sstride : c / side - radius;
        const int dx = SEED ? (c % sside - radius / sstride) * sstride : c % side - radius;
        const int cx = clampi(bx + dx, 0, W - 16) - lo_x, cy = clampi(by + dy, 0, H - 16) - lo_y;
        // the candidate's 64 q as 32 u16 pairs (DP2A: two q x r products per instruction)
        uint32_t qp[32];
        int sq = 0, sqq = 0;
#pragma unroll
        for (int i = 0; i < 8; i++)
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
                const uint32_t a = s2[cy + 2 * i][cx + 2 * j], b = s2[cy + 2 * i][cx + 2 * j + 2];
                qp[(8 * i + j) / 2] = __byte_perm(a, b, 0x5410);
                sq += (int)(a + b);
                sqq += (int)(a * a + b * b);
            }
        const long long D = 64ll * sqq - (long long)sq * sq;
#pragma unroll 1
        for (int t = 0; t < NI; t++) {
            unsigned acc = 0;
#pragma unroll
            for (int w4 = 0; w4 < 16; w4++) {
                const uint32_t rw4 = rtp[t][w4];
                acc = __dp2a_lo(qp[2 * w4], rw4, acc);
                acc = __dp2a_hi(qp[2 * w4 + 1], rw4, acc);
            }
            const int sqr = (int)acc;
            const long long N = 64ll * sqr - (long long)sq * sr;
            const long long k2 = 2 * quant_code(N, D) - 7;
            const long long X = 65536ll * A - 64 * k2 * N + k2 * k2 * D;  // 1024 * n * SSE, n = 64
            const unsigned long long key =
                SEED ? make_key_cb(X - 65536ll * A, ((long long)(cy + lo_y) * (W - 15) + cx + lo_x) * NI + t,
                                   key_cand_bits(64))
                     : make_key(X, (long long)c * NI + t);
            best = key < best ? key : best;
        }
    }
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long other = __shfl_xor_sync(FULL, best, off);
        best = other < best ? other : best;
    }
    if ((threadIdx.x & 31) == 0) wbest[threadIdx.x >> 5] = best;
    __syncthreads();
    if (SEED) {
        if (threadIdx.x == 0) {
            for (int w = 0; w < (int)(blockDim.x >> 5); w++) best = wbest[w] < best ? wbest[w] : best;
            atomicMin(&seed_best[ri], best);
        }
        return;
    }
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); w++) best = wbest[w] < best ? wbest[w] : best;
        best = wbest[0] < best ? wbest[0] : best;
        const int cand = (int)(best & ((1ull << 21) - 1));
        const int c = cand / NI, t = cand % NI;
        const int dy = c / side - radius, dx = c % side - radius;
        const int cx = clampi(bx + dx, 0, W - 16), cy = clampi(by + dy, 0, H - 16);
        int sq = 0, sqq = 0, sqr = 0;
        for (int i = 0; i < 8; i++)
            for (int j = 0; j < 8; j++) {
                const int q = s2[cy - lo_y + 2 * i][cx - lo_x + 2 * j];
                sq += q;
                sqq += q * q;
                sqr += q * rt[t][8 * i + j];
            }
        const long long N = 64ll * sqr - (long long)sq * sr, D = 64ll * sqq - (long long)sq * sq;
        out_dx[ri] = cx;
        out_dy[ri] = cy;
        if (out_iso) out_iso[ri] = (int8_t)t;
        out_o[ri] = (uint8_t)o;
        out_code[ri] = (uint8_t)quant_code(N, D);
    }
}

int sm_count_search() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

}  // namespace

struct SearchWs {
    uint16_t *pool;
    int32_t *psq;
    long long *pD;
    unsigned long long *best;
};

static int64_t align256(int64_t v) { return (v + 255) & ~(int64_t)255; }

int64_t search_tc_workspace_bytes(int W, int H, int B, int step, int n_iso);

int search_workspace_bytes(int W, int H, int B, int step, int n_iso, int64_t *bytes) {
    const long long ndx = (W - 2 * B) / step + 1, ndy = (H - 2 * B) / step + 1;
    const long long ndom = ndx * ndy, n = (long long)B * B;
    const long long nranges = (long long)(W / B) * (H / B);
    *bytes = align256(ndom * n * 2) + align256(ndom * 4) + align256(ndom * 8) + align256(nranges * 8);
    if (B <= 8) *bytes += align256(search_tc_workspace_bytes(W, H, B, step, n_iso));
    return 0;
}

int64_t local_search_tc_workspace_bytes(int W, int H, int B, int R, int n_iso);
int local_search_tc(const uint8_t *img, int W, int H, int R, int n_iso, uint16_t *pool, int32_t *psq, long long *pD,
                    long long ndom, unsigned long long *best, void *tc_ws, cudaStream_t st);

int full_search_tc(const uint8_t *img, int W, int H, int B, int step, int n_iso, int r0, int r1,
                   uint16_t *pool, int32_t *psq, long long *pD, long long ndom,
                   unsigned long long *best, void *tc_ws, cudaStream_t st, bool *handled);

// MNS_SEARCH_CUDA_CORES=1 selects the exact CUDA-core path for every B (A/B checks of the tensor-core path).
static bool force_cuda_cores() {
    const char *e = getenv("MNS_SEARCH_CUDA_CORES");
    return e && e[0] == '1';
}

int full_search(const uint8_t *img, int W, int H, int B, int step, int n_iso, int r0, int r1, int32_t *out_dom,
                int8_t *out_iso, uint8_t *out_o, uint8_t *out_code, void *ws, int64_t ws_bytes, cudaStream_t st) {
    MNS_CHECK_ARG(B == 2 || B == 4 || B == 8 || B == 16, "range size must be one of [2, 4, 8, 16]");
    MNS_CHECK_ARG(W % B == 0 && H % B == 0 && W >= 2 * B && H >= 2 * B, "image too small or not B-padded");
    MNS_CHECK_ARG(step >= 1, "full_search_step must be >= 1");
    MNS_CHECK_ARG(n_iso == 1 || n_iso == 8, "n_iso must be 1 or 8");
    const long long nranges = (long long)(W / B) * (H / B);
    MNS_CHECK_ARG(0 <= r0 && r0 <= r1 && r1 <= nranges, "bad range interval");
    int64_t need;
    search_workspace_bytes(W, H, B, step, n_iso, &need);
    MNS_CHECK_ARG(ws_bytes >= need, "workspace too small");
    const long long ndx = (W - 2 * B) / step + 1, ndy = (H - 2 * B) / step + 1, ndom = ndx * ndy;
    MNS_CHECK_ARG(ndom * n_iso < (1ll << key_cand_bits(B * B)), "domain pool too large for the argmin key");
    if (r1 == r0) return 0;
    char *p = (char *)ws;
    SearchWs w;
    const long long n = (long long)B * B;
    w.pool = (uint16_t *)p;
    p += align256(ndom * n * 2);
    w.psq = (int32_t *)p;
    p += align256(ndom * 4);
    w.pD = (long long *)p;
    p += align256(ndom * 8);
    w.best = (unsigned long long *)p;
    p += align256(nranges * 8);
    void *tc_ws = B <= 8 ? (void *)p : nullptr;
    const int sms = sm_count_search();
    fill_u64_kernel<<<64, 256, 0, st>>>(w.best, ~0ull, r1 - r0);
    bool handled = false;
    int rc = 0;
    if (!force_cuda_cores()) rc = full_search_tc(img, W, H, B, step, n_iso, r0, r1, w.pool, w.psq, w.pD, ndom, w.best,
                                               tc_ws, st, &handled);
    if (rc) return rc;
    if (!handled) {
        pool_kernel<<<sms * 16, 256, 0, st>>>(img, W, B, step, (int)ndx, ndom, w.pool, w.psq, w.pD);
        const int tiles = (r1 - r0 + 7) / 8;
        const long long gx = (ndom + 255) / 256;
        dim3 grid((unsigned)(gx < 64 ? gx : 64), (unsigned)tiles);
        switch (B) {
        case 2: full_search_cc_kernel<2><<<grid, 256, 0, st>>>(img, W, n_iso, r0, r1, w.pool, w.psq, w.pD, ndom, w.best); break;
        case 4: full_search_cc_kernel<4><<<grid, 256, 0, st>>>(img, W, n_iso, r0, r1, w.pool, w.psq, w.pD, ndom, w.best); break;
        case 8: full_search_cc_kernel<8><<<grid, 256, 0, st>>>(img, W, n_iso, r0, r1, w.pool, w.psq, w.pD, ndom, w.best); break;
        default: full_search_cc_kernel<16><<<grid, 256, 0, st>>>(img, W, n_iso, r0, r1, w.pool, w.psq, w.pD, ndom, w.best); break;
        }
    }
    search_finalize_kernel<<<(r1 - r0 + 7) / 8, 256, 0, st>>>(img, W, B, n_iso, r0, r1, w.best, w.pool, w.psq, w.pD,
                                                             out_dom, out_iso, out_o, out_code);
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

int local_search(const uint8_t *img, int W, int H, int radius, int n_iso, int32_t *out_dx, int32_t *out_dy,
                 int8_t *out_iso, uint8_t *out_o, uint8_t *out_code, cudaStream_t st);

// winner domain index -> origin (stride 1): dx = d % ndx, dy = d / ndx (in place: out_dx held the index)
__global__ void dom_to_xy_kernel(int32_t *out_dx, int32_t *out_dy, int n, int ndx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int d = out_dx[i];
    out_dx[i] = d % ndx;
    out_dy[i] = d / ndx;
}

int local_search_workspace_bytes(int W, int H, int radius, int n_iso, int64_t *bytes) {
    int64_t base;
    search_workspace_bytes(W, H, 8, 1, n_iso, &base);
    *bytes = base + align256(local_search_tc_workspace_bytes(W, H, 8, radius, n_iso));
    return 0;
}

// Local search through the tensor-core pipeline (windowed full search), exact like the CUDA-core
// kernel (same keys, same finalisation); MNS_LOCAL_CUDA_CORES=1 selects the CUDA-core kernel.
int local_search_ws(const uint8_t *img, int W, int H, int radius, int n_iso, int32_t *out_dx, int32_t *out_dy,
                    int8_t *out_iso, uint8_t *out_o, uint8_t *out_code, void *ws, int64_t ws_bytes, cudaStream_t st) {
    MNS_CHECK_ARG(W >= 16 && H >= 16 && W % 8 == 0 && H % 8 == 0, "local search needs at least a 16x16 image");
    MNS_CHECK_ARG(radius >= 0 && radius <= 32, "radius must be in [0, 32]");
    MNS_CHECK_ARG(n_iso == 1 || n_iso == 8, "n_iso must be 1 or 8");
    const char *e = getenv("MNS_LOCAL_CUDA_CORES");
    if (e && e[0] == '1') return local_search(img, W, H, radius, n_iso, out_dx, out_dy, out_iso, out_o, out_code, st);
    int64_t need;
    local_search_workspace_bytes(W, H, radius, n_iso, &need);
    MNS_CHECK_ARG(ws_bytes >= need, "workspace too small");
    const int B = 8;
    const long long ndx = W - 2 * B + 1, ndy = H - 2 * B + 1, ndom = ndx * ndy, n = 64;
    const long long nranges = (long long)(W / B) * (H / B);
    MNS_CHECK_ARG(ndom * n_iso < (1ll << key_cand_bits(64)), "domain pool too large for the argmin key");
    char *p = (char *)ws;
    SearchWs w;
    w.pool = (uint16_t *)p;
    p += align256(ndom * n * 2);
    w.psq = (int32_t *)p;
    p += align256(ndom * 4);
    w.pD = (long long *)p;
    p += align256(ndom * 8);
    w.best = (unsigned long long *)p;
    p += align256(nranges * 8);
    int64_t fs_base;
    search_workspace_bytes(W, H, B, 1, n_iso, &fs_base);
    void *tc_ws = (char *)ws + fs_base;
    fill_u64_kernel<<<64, 256, 0, st>>>(w.best, ~0ull, nranges);
    if (false) {  // (measured slower: the tensor-core pass is not bound by its rare path) seeds from a grid
        const int nr = (int)nranges;
        if (n_iso == 1)
            local_search_kernel<32, 1, true><<<nr, 256, 0, st>>>(img, W, H, radius, nullptr, nullptr, nullptr, nullptr,
                                                                  nullptr, w.best, 4);
        else
            local_search_kernel<32, 8, true><<<nr, 256, 0, st>>>(img, W, H, radius, nullptr, nullptr, nullptr, nullptr,
                                                                  nullptr, w.best, 4);
    }
    if (int rc = local_search_tc(img, W, H, radius, n_iso, w.pool, w.psq, w.pD, ndom, w.best, tc_ws, st)) return rc;
    search_finalize_kernel<<<(unsigned)((nranges + 7) / 8), 256, 0, st>>>(img, W, B, n_iso, 0, (int)nranges, w.best,
                                                                          w.pool, w.psq, w.pD, out_dx, out_iso,
                                                                          out_o, out_code);
    dom_to_xy_kernel<<<(unsigned)((nranges + 255) / 256), 256, 0, st>>>(out_dx, out_dy, (int)nranges, (int)ndx);
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

int local_search(const uint8_t *img, int W, int H, int radius, int n_iso, int32_t *out_dx, int32_t *out_dy,
                 int8_t *out_iso, uint8_t *out_o, uint8_t *out_code, cudaStream_t st) {
    MNS_CHECK_ARG(W >= 16 && H >= 16 && W % 8 == 0 && H % 8 == 0, "local search needs at least a 16x16 image");
    MNS_CHECK_ARG(radius >= 0 && radius <= 32, "radius must be in [0, 32]");
    MNS_CHECK_ARG(n_iso == 1 || n_iso == 8, "n_iso must be 1 or 8");
    const int nr = (W / 8) * (H / 8);
#define LS_LAUNCH(Rr, NI, T) local_search_kernel<Rr, NI><<<nr, T, 0, st>>>(img, W, H, radius, out_dx, out_dy, out_iso, out_o, out_code)
    if (n_iso == 1) {
        if (radius <= 4) LS_LAUNCH(4, 1, 128);
        else if (radius <= 16) LS_LAUNCH(16, 1, 256);
        else LS_LAUNCH(32, 1, 256);
    } else {
        if (radius <= 4) LS_LAUNCH(4, 8, 128);
        else if (radius <= 16) LS_LAUNCH(16, 8, 256);
        else LS_LAUNCH(32, 8, 256);
    }
#undef LS_LAUNCH
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

}  // namespace mns
