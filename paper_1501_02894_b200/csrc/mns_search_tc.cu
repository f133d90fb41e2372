// tcgen05 tensor-core full search (K3) for B in {2, 4, 8} on sm_100a.
//
// Replaces encoder.py:249-309 (encode_full_search).  rows = (range, isometry) pairs (M, 128 per
// MMA, two M halves per CTA), columns = domains (N = 128 per tile), K = 64 (zero-padded for B < 8).
//
// The GEMM produces, per (row, domain), the quantity the argmin filter needs:
//   x = sum_k (r_k - Sr/n) * (q_k - Sq/n) / sqrt(D) = N / (n sqrt D),   N = n C - Sq Sr,
// with both operands centred and the domain operand scaled by 1/sqrt(D), each rounded once to
// fp16 (FP16 x FP16 -> FP32 UMMA).  The reference's per-domain value is
//   1024 n SSE - 1024 n A = min over odd k2 in [-7, 7] of  k2^2 D - 64 k2 N,
// whose continuous relaxation is -1024 N^2 / D = -1024 n^2 x^2: against the row's running exact
// best V*, an element can only win if |x| >= scl = sqrt(-V*/1024) / n.  The computed x differs
// from the true one by at most e_row = 2^-9 * max_k |r_k - Sr/n| (fp16 rounding of both operands:
// sum_k |q_k - Sq/n| / sqrt(D) <= 1 by Cauchy-Schwarz, so each costs <= 2^-11 max|r_c|; the fp32
// accumulation < 2^-16 of it; a ~2x safety factor on top), a per-ROW constant.  So level 1 is one
// |max| per element against one per-row threshold (FMNMX3 over two elements).  Survivors (voted
// per 16-column group) pass a rigorous fp32 lower bound of the quantised value (level 2); the
// rest are evaluated exactly in int64 from the pooled integer q and the raw range row (level 3)
// and folded into the row's lexicographic (value, index) key, shared across CTAs by atomicMin.
// A prepass over a 1/1024 domain sample, seeded with 5 nearby domains per range, sets the
// thresholds; constant ranges (N == 0 for every domain) take the precomputed argmin of D.
//
// Persistent CTAs (one per SM): CTA b owns a contiguous, equal share of the (M tile, domain tile)
// units in M-major order, so every SM streams the same number of tiles and pays the prologue
// once.  The range operand of consecutive M tiles is double-buffered in shared memory.
//
// Warp roles (20 warps): w0 TMA producer (A per M tile, B tiles through a 4-stage 128B-swizzled
// ring), w1 single-thread MMA issuer (2 M halves x 4 K=16 steps per tile into one of two
// 256-column TMEM accumulators), w2 TMEM allocator, w3 column-constant producer (4-deep ring),
// w4..w19 epilogue: each thread owns one TMEM lane (= one row) and half of the 128 columns; it
// loads its 64 accumulator columns, releases the accumulator, then filters from registers.

#include <cuda_fp16.h>
#include <math.h>

#include "mns_common.cuh"
#include "mns_tma.cuh"

namespace mns {

#ifdef MNS_TC_STATS
__device__ unsigned long long g_tc_stats[4];  // 16-col groups, level-1 group passes, level-2 entries, exact evaluations
#endif

namespace {

constexpr unsigned FULL = 0xffffffffu;
#ifndef TC_BN
#define TC_BN 256
#endif
constexpr int BM = 128, BN = TC_BN, BK = 64;  // MMA tile (M rows, N domains, K)
constexpr int MH = 256 / BN;                  // M halves per CTA (MH * BN = 256 TMEM columns per stage)
#ifndef TC_SAMPLE
#define TC_SAMPLE 1024
#endif
#ifndef TC_POLL
#define TC_POLL 0  // poll the global keys when (t & TC_POLL) == TC_POLL
#endif
#ifndef TC_STAGES
#define TC_STAGES 4
#endif
constexpr int STAGES = TC_STAGES;
#ifndef TC_EPI_WARPS
#define TC_EPI_WARPS 16
#endif
constexpr int EPI_WARP0 = 4, EPI_WARPS = TC_EPI_WARPS;  // 16: each warp 64 columns; 8: all 128
constexpr int NTHREADS = (EPI_WARP0 + EPI_WARPS) * 32;
constexpr int A_BYTES = MH * BM * BK * 2;     // 32 KB per A buffer (two buffers)
constexpr int B_BYTES = BN * BK * 2;          // 16 KB
constexpr int TMEM_COLS = 2 * MH * BN;        // 2 accumulator stages x 2 M halves x 128 columns = 512
constexpr int EPI_COLS = BN * 4 * MH / EPI_WARPS;  // columns per epilogue thread per tile
constexpr int GRP = 16;                       // level-1 vote group (columns)
constexpr int NCB = 4;                        // column-constant ring slots
constexpr int CONST_BYTES = BN * 16;          // per tile: 128 x -Sq, 128 x sqrt_rd(D) (floats), 128 x D (int64)
constexpr int QSIZE = 1024;                   // exact-evaluation queue entries (16 B each)
constexpr int CONST_OFF = 2 * A_BYTES + STAGES * B_BYTES + 512;
constexpr int QUEUE_OFF = CONST_OFF + NCB * CONST_BYTES;
constexpr int STASH_OFF = QUEUE_OFF + QSIZE * 16;  // per epilogue warp: [GRP][32] floats
constexpr int SMEM_BYTES = 1024 + STASH_OFF + EPI_WARPS * GRP * 32 * 4;

struct TcParams {
    int n_rows;          // (r1 - r0) * n_iso
    int n_iso, r0, n;    // n = B*B
    long long ndom;
    int n_dt;            // domain tiles in this launch
    long long n_units;   // M tiles x n_dt
    int dstride;                 // domain of column c of tile t: (t * BN + c) * dstride
    const float2 *consts;        // per 128-domain tile: 128 floats -Sq, then 128 floats sqrt_rd(D)
    const long long *pD;         // exact D
    const uint16_t *pool;        // [ndom][n] pooled q (exact recompute of C)
    const __half *araw;          // [n_rows_pad][BK] raw range rows (r per isometry, exact)
    const int32_t *row_sr;       // [n_rows_pad] Sr of the row's range
    const int32_t *row_flat;     // [n_rows_pad] 1 if the range is constant (N == 0 for every domain)
    const float *row_err;        // [n_rows_pad] e_row
    const unsigned long long *flat_key;  // argmin-D key for constant ranges (full search)
    unsigned long long *best;    // [r1 - r0]
    // local search (encoder.py:312-347 as a windowed GEMM): the (M tile, domain tile) units that meet
    // some row's window, M-major (nullptr: every unit, the full search); their count on the device
    const uint2 *units;
    const int *n_units_dev;
    int local_R;                 // window radius (-1: full search)
    int W, H, B, ndx, ndy;       // geometry of the windows (stride 1: domain index = y * ndx + x)
};


// exact min over odd k2 in [-7, 7] of k2^2 D - 64 k2 N: an fp32 estimate of the vertex
// 32N/D picks the nearest odd k2; it and both odd neighbours are evaluated exactly.
__device__ __forceinline__ long long best_val_exact(long long N, long long D) {
    if (D == 0) return 0;  // N == 0 whenever D == 0
    const float t = __fdividef(32.f * (float)N, (float)D);
    const int k = 2 * (int)floorf(fminf(8.f, fmaxf(-8.f, t)) * 0.5f) + 1;
    long long best = LLONG_MAX;
#pragma unroll
    for (int dk = -2; dk <= 2; dk += 2) {
        const long long k2 = k + dk;
        if (k2 < -7 || k2 > 7) continue;
        const long long v = k2 * k2 * D - 64 * k2 * N;
        best = v < best ? v : best;
    }
    return best;
}

// exact C = sum_k q_k r_k of domain d and range row `row`: the pooled q row (u16) and the raw
// fp16 range row read as 16-byte vectors, all loads issued before the integer dot product
__device__ __noinline__ long long exact_cross(const uint16_t *pool, const __half *araw, int n, long long d, int row) {
    const uint16_t *qd = pool + d * n;
    const __half *ar = araw + (size_t)row * BK;
    long long C = 0;
    if (n == 64) {
        uint4 qv[8], av[8];
#pragma unroll
        for (int i = 0; i < 8; i++) {
            qv[i] = __ldg(reinterpret_cast<const uint4 *>(qd) + i);
            av[i] = __ldg(reinterpret_cast<const uint4 *>(ar) + i);
        }
        int acc = 0;  // < 64 * 1020 * 255 < 2^24
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const uint32_t qw[4] = {qv[i].x, qv[i].y, qv[i].z, qv[i].w};
            const uint32_t aw[4] = {av[i].x, av[i].y, av[i].z, av[i].w};
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const __half2 h = *reinterpret_cast<const __half2 *>(&aw[j]);
                acc += (int)(qw[j] & 0xFFFF) * __half2int_rn(__low2half(h)) +
                       (int)(qw[j] >> 16) * __half2int_rn(__high2half(h));
            }
        }
        return acc;
    }
    for (int k = 0; k < n; k++) C += (long long)qd[k] * (long long)__half2int_rn(ar[k]);
    return C;
}

__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
    // K-major, 128B swizzle: rows of 128 B, 8-row atoms 1024 B apart (SBO), LBO unused (1), version 1
    return (uint64_t)((smem_addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// 32 accumulator columns (no wait)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float *v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// 1D bulk copy global -> shared completing on an mbarrier (size multiple of 16 B)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// mbarrier wait without a suspend-time hint: the try_wait loop never drops into a long
// NANOSLEEP, so a waiter resumes as soon as the phase completes (the MMA <-> epilogue handshake
// sits on the critical path of every tile)
__device__ __forceinline__ void mbar_spin(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// mbarrier wait with a short (~0.2 us) suspend-time hint, for producers that are not on the
// critical path
__device__ __forceinline__ void mbar_wait_ns(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, 200;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// max(|a|, |b|, m): one FMNMX3 with |.| operand modifiers
__device__ __forceinline__ float absmax3(float m, float a, float b) { return fmaxf(m, fmaxf(fabsf(a), fabsf(b))); }

template <bool LOCAL>  // LOCAL: the windowed local search (p.units, p.local_R); else the full search
__global__ void __launch_bounds__(NTHREADS, 1)
    full_search_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          const TcParams p) {
    extern __shared__ __align__(1024) unsigned char tsm_raw[];
    // 1024-B aligned base as an offset from the shared array (keeps shared-space addressing: LDS, not LD.E)
    unsigned char *tsm = tsm_raw + ((1024u - (smem_u32(tsm_raw) & 1023u)) & 1023u);
    unsigned char *sA = tsm;                    // [2][A_BYTES]
    unsigned char *sB = tsm + 2 * A_BYTES;
    uint64_t *bars = reinterpret_cast<uint64_t *>(tsm + 2 * A_BYTES + STAGES * B_BYTES);
    uint64_t *full_bar = bars, *empty_bar = bars + STAGES;
    uint64_t *a_full = bars + 2 * STAGES, *a_empty = bars + 2 * STAGES + 2;
    uint64_t *tfull = bars + 2 * STAGES + 4, *tempty = bars + 2 * STAGES + 6;
    uint32_t *tmem_base_sh = reinterpret_cast<uint32_t *>(bars + 2 * STAGES + 8);
    uint32_t *q_head = tmem_base_sh + 1, *q_tail = tmem_base_sh + 2, *q_done = tmem_base_sh + 3;
    uint64_t *cfull = bars + 2 * STAGES + 12, *cempty = bars + 2 * STAGES + 12 + NCB;  // column-constant ring
    uint32_t *c_issued = tmem_base_sh + 4;  // constant copies issued so far
    unsigned char *queue = tsm + QUEUE_OFF;
    unsigned char *sC = tsm + CONST_OFF;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // this CTA's contiguous share of the (M tile, domain tile) units, M-major
    const long long n_units = LOCAL ? (long long)*p.n_units_dev : p.n_units;
    const long long u0 = n_units * blockIdx.x / gridDim.x, u1 = n_units * (blockIdx.x + 1) / gridDim.x;
    const int ntiles = (int)(u1 - u0);
    // The units of this CTA, walked in order by every role: (M tile, domain tile) of unit t, and the
    // M tile of unit t + 1.  The local search reads its list three units ahead (registers), so no
    // dependent global load sits on the TMA / MMA critical path.
    struct UnitStream {
        const uint2 *units;
        int n_dt;
        long long u0;
        int ntiles, t;
        uint2 a, b, c;  // units t, t + 1, t + 2
        __device__ uint2 load(int i) const {  // local search only
            return i < ntiles ? __ldg(units + u0 + i) : make_uint2(0xFFFFFFFFu, 0u);
        }
        __device__ uint2 step(uint2 u) const {  // dense: the next unit, M-major
            return u.y + 1 == (uint32_t)n_dt ? make_uint2(u.x + 1, 0u) : make_uint2(u.x, u.y + 1);
        }
        __device__ UnitStream(const uint2 *un, int ndt, long long uu0, int nt)
            : units(un), n_dt(ndt), u0(uu0), ntiles(nt), t(0) {
            if (LOCAL) {
                a = load(0);
                b = load(1);
                c = load(2);
            } else {
                a = make_uint2((uint32_t)(u0 / n_dt), (uint32_t)(u0 % n_dt));
                b = step(a);
            }
        }
        __device__ int m() const { return (int)a.x; }
        __device__ int dt() const { return (int)a.y; }
        __device__ int next_m() const { return (int)b.x; }
        __device__ void advance() {
            if (LOCAL) {
                a = b;
                b = c;
                c = load(++t + 2);
            } else {
                a = b;
                b = step(b);
            }
        }
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        for (int a = 0; a < 2; a++) {
            mbar_init(&a_full[a], 1);
            mbar_init(&a_empty[a], 1);
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], EPI_WARPS);
        }
        for (int a = 0; a < NCB; a++) {
            mbar_init(&cfull[a], 1);
            mbar_init(&cempty[a], EPI_WARPS);
        }
        *c_issued = 0;
        *q_head = 0;
        *q_tail = 0;
        *q_done = 0;
        fence_mbar_init();
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_base_sh)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < QSIZE; i += NTHREADS) reinterpret_cast<uint4 *>(queue)[i].w = 0;  // no slot ready
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_base_sh;

    if (warp == 0) {
        // ===== TMA producer: the A operand of every new M tile into the other A buffer, B tiles.
        // Its waits sleep briefly (a 4-deep ring): spinning would steal issue slots from the
        // epilogue warps on the same scheduler.
        if (lane == 0) {
            prefetch_tmap(&tmA);
            prefetch_tmap(&tmB);
            int seg = -1, cur_m = -1;
            UnitStream us(p.units, p.n_dt, u0, ntiles);
            for (int t = 0; t < ntiles; t++, us.advance()) {
                const int m = us.m(), dt = us.dt();
                if (m != cur_m) {
                    cur_m = m;
                    seg++;
                    const int ab = seg & 1;
                    if (seg >= 2) mbar_wait_ns(&a_empty[ab], ((seg >> 1) - 1) & 1);
                    mbar_arrive_expect_tx(&a_full[ab], A_BYTES);
                    for (int h = 0; h < MH; h++)
                        tma_load_2d(sA + ab * A_BYTES + h * BM * BK * 2, &tmA, 0, (m * MH + h) * BM, &a_full[ab]);
                }
                const int s = t % STAGES;
                if (t >= STAGES) mbar_wait_ns(&empty_bar[s], ((t / STAGES) - 1) & 1);
                mbar_arrive_expect_tx(&full_bar[s], B_BYTES);
                tma_load_2d(sB + s * B_BYTES, &tmB, 0, dt * BN, &full_bar[s]);
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (one thread)
        if (lane == 0) {
            // instruction descriptor: F32 accumulate, F16 A/B, K-major both, N = BN, M = 128
            const uint32_t idesc = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                   ((uint32_t)(BM >> 4) << 24);
            int seg = -1, cur_m = -1;
            uint64_t adesc0 = 0;
            UnitStream us(p.units, p.n_dt, u0, ntiles);
            for (int t = 0; t < ntiles; t++, us.advance()) {
                const int m = us.m();
                if (m != cur_m) {
                    cur_m = m;
                    seg++;
                    mbar_spin(&a_full[seg & 1], (seg >> 1) & 1);
                    tc_fence_after();
                    adesc0 = umma_desc_sw128(smem_u32(sA + (seg & 1) * A_BYTES));
                }
                const int s = t % STAGES, acc = t & 1;
#if !(defined(TC_EXP) && TC_EXP >= 4)
                if (t >= 2) mbar_spin(&tempty[acc], ((t / 2) - 1) & 1);
#endif
                mbar_spin(&full_bar[s], (t / STAGES) & 1);
                tc_fence_after();
                const uint64_t bdesc = umma_desc_sw128(smem_u32(sB + s * B_BYTES));
#pragma unroll
                for (int h = 0; h < MH; h++) {  // both M halves against the same B tile
                    const uint64_t adesc = adesc0 + (uint64_t)((h * BM * BK * 2) >> 4);
#pragma unroll
                    for (int k = 0; k < BK / 16; k++)  // +32 B per K=16 step inside the 128B swizzle atom
                        umma_f16(tmem + (acc * MH + h) * BN, adesc + 2 * k, bdesc + 2 * k, idesc, k > 0 ? 1u : 0u);
                }
                umma_commit(&empty_bar[s]);  // frees the B stage when these MMAs complete
                umma_commit(&tfull[acc]);    // accumulator ready for the epilogue
                const bool seg_end = t + 1 == ntiles || us.next_m() != m;
                if (seg_end) umma_commit(&a_empty[seg & 1]);  // A buffer reusable once these complete
            }
        }
    } else if (warp == 2) {
        // ===== column constants of tile t into ring slot t % NCB (read only on the rare level-2 path)
        if (lane == 0) {
            UnitStream us(p.units, p.n_dt, u0, ntiles);
#if defined(TC_EXP) && TC_EXP >= 4
            for (int t = 0; t < 0; t++) {
#else
            for (int t = 0; t < ntiles; t++, us.advance()) {
#endif
                const int dt = us.dt();
                const int cb = t % NCB;
                if (t >= NCB) {  // the slot's previous copy has landed and every epilogue warp is past it
                    mbar_wait_ns(&cfull[cb], ((t / NCB) - 1) & 1);
                    mbar_wait_ns(&cempty[cb], ((t / NCB) - 1) & 1);
                }
                mbar_arrive_expect_tx(&cfull[cb], CONST_BYTES);
                const long long b0 = (long long)dt * BN;
                bulk_g2s(sC + cb * CONST_BYTES, p.consts + b0, BN * 8, &cfull[cb]);
                bulk_g2s(sC + cb * CONST_BYTES + BN * 8, p.pD + b0, BN * 8, &cfull[cb]);
                *(volatile uint32_t *)c_issued = (uint32_t)(t + 1);  // copy t issued: cfull[cb]'s phase is t / NCB
            }
        }
    } else if (warp == 3) {
        // ===== exact warp: pops the candidates that passed levels 1 and 2 (one per lane) and
        // evaluates them exactly in int64 from the pooled q and the raw range row; improvements go
        // to the global keys (atomicMin), which every epilogue lane polls.  The epilogue never waits
        // on these global round trips.
        uint32_t tail = 0;
        for (;;) {
            const uint32_t head = *(volatile uint32_t *)q_head;
            if (head == tail) {
                if (*(volatile uint32_t *)q_done == EPI_WARPS && *(volatile uint32_t *)q_head == tail) break;
                __nanosleep(100);
                continue;
            }
            const uint32_t cnt = min(head - tail, 32u);
            uint32_t code = 0, m = 0, dt = 0;
            if (lane < cnt) {
                const uint32_t slot = tail + lane;
                volatile uint4 *e = reinterpret_cast<volatile uint4 *>(queue) + (slot % QSIZE);
                while (e->w != slot + 1) {
                }
                code = e->x;
                m = e->y;
                dt = e->z;
            }
            __syncwarp();
            tail += cnt;
            if (lane == 0) *(volatile uint32_t *)q_tail = tail;  // slots free once read
            if (lane < cnt) {
                const int col = (int)(code & 0xFF), rl = (int)(code >> 8);
                const int row = (int)m * (MH * BM) + rl;
                const int rr = row / p.n_iso, iso = row % p.n_iso;
                const long long dcol = (long long)dt * BN + col;
                const long long d = dcol * p.dstride;
                const float *lq = reinterpret_cast<const float *>(p.consts + (long long)dt * BN);  // -Sq | sqrt_rd(D)
                const long long C = exact_cross(p.pool, p.araw, p.n, d, row);
                const long long N = (long long)p.n * C - (long long)(int)(-__ldg(lq + col)) * p.row_sr[row];
                const unsigned long long key = make_key_cb(best_val_exact(N, __ldg(p.pD + dcol)), d * p.n_iso + iso,
                                                              key_cand_bits(p.n));
#ifdef MNS_TC_STATS
                atomicAdd(&g_tc_stats[3], 1ull);
#endif
                atomicMin(&p.best[rr], key);
            }
        }
    } else if (warp >= EPI_WARP0) {
        // ===== epilogue: one TMEM lane (= row) per thread, half of the columns per warp
        const int ew = warp - EPI_WARP0;       // 0..15
        const int quarter = warp & 3;          // TMEM lane quarter this warp may access
        const int mh = (ew >> 2) % MH;         // M half
        const int half = ew / (4 * MH);        // column block of EPI_COLS columns
        const int rl = mh * BM + quarter * 32 + lane;  // row within the M tile
        float *stash = reinterpret_cast<float *>(tsm + STASH_OFF) + ew * (GRP * 32);  // [GRP][32] per warp
        const float n64 = -64.f * (float)p.n;
        const float inv_n = 1.0f / (float)p.n;  // exact (power of two)
        int cur_m = -1, rr = 0;
        uint32_t wx = 0xFFFF0000u, wy = 0xFFFF0000u;  // local search: the row's window, lo | hi << 16
        bool live = false;
        float erow = 0.f, thr = -1.f;
        long long vstar = LLONG_MAX;  // an upper bound of this range's best value (a real candidate's)
        auto set_threshold = [&](long long v) {
            if (v < vstar) {
                vstar = v;
                // -1024 n^2 x^2 > V*  <=>  |x| < sqrt(-V*/1024)/n  (scl rounded down, thr = scl - e_row)
                thr = v < 0 ? __fsub_rd(__fmul_rd(__fsqrt_rd(__fmul_rd(__ll2float_rd(-v), 0.999f / 1024.f)), inv_n),
                                        erow)
                            : -1.f;
            }
        };
        unsigned long long g = ~0ull;
        // the epilogue walks its units with a one-ahead prefetch (local) or incrementally (dense)
        uint2 u_cur = ntiles > 0 ? (LOCAL ? __ldg(p.units + u0) : make_uint2((uint32_t)(u0 / p.n_dt), (uint32_t)(u0 % p.n_dt)))
                                 : make_uint2(0u, 0u);
#if defined(TC_EXP) && TC_EXP >= 4
        for (int t = 0; t < 0; t++) {
            int m = 0, dt = 0;
#else
        for (int t = 0; t < ntiles; t++) {
            const int m = (int)u_cur.x, dt = (int)u_cur.y;
            if (LOCAL)
                u_cur = t + 1 < ntiles ? __ldg(p.units + u0 + t + 1) : u_cur;
            else
                u_cur = u_cur.y + 1 == (uint32_t)p.n_dt ? make_uint2(u_cur.x + 1, 0u) : make_uint2(u_cur.x, u_cur.y + 1);
#endif
            if (m != cur_m) {  // new M tile: load the row
                cur_m = m;
                const int row = m * (MH * BM) + rl;
                const bool active = row < p.n_rows;
                const bool flat = active ? p.row_flat[row] != 0 : true;
                live = active && !flat;
                rr = row / p.n_iso;
                if (!LOCAL && active && flat && row % p.n_iso == 0 && half == 0)
                    atomicMin(&p.best[rr], *p.flat_key);  // (local search: local_flat_kernel)
                if (LOCAL && active) {  // the range's window of candidate origins
                    const int ri = p.r0 + rr, rpr = p.W / p.B;
                    const int bx = clampi((ri % rpr) * p.B - p.B / 2, 0, p.W - 2 * p.B);
                    const int by = clampi((ri / rpr) * p.B - p.B / 2, 0, p.H - 2 * p.B);
                    wx = (uint32_t)clampi(bx - p.local_R, 0, p.ndx - 1) |
                         ((uint32_t)clampi(bx + p.local_R, 0, p.ndx - 1) << 16);
                    wy = (uint32_t)clampi(by - p.local_R, 0, p.ndy - 1) |
                         ((uint32_t)clampi(by + p.local_R, 0, p.ndy - 1) << 16);
                }
                erow = live ? p.row_err[row] : 0.f;
                vstar = LLONG_MAX;
                thr = -1.f;
                g = live ? ld_relaxed_u64(&p.best[rr]) : ~0ull;
            }
            const int acc = t & 1, cbuf = t % NCB;
            // the range's running best from every CTA's exact warp and every isometry row of the range
            // (global key, loaded a tile ahead)
            if (g != ~0ull) set_threshold(key_val(g, key_cand_bits(p.n)));
            g = ~0ull;
            mbar_spin(&tfull[acc], (t >> 1) & 1);
            tc_fence_after();
            if ((t & TC_POLL) == TC_POLL) g = live ? ld_relaxed_u64(&p.best[rr]) : ~0ull;
            float c[EPI_COLS];
            const uint32_t tbase = tmem + ((uint32_t)(quarter * 32) << 16) + (acc * MH + mh) * BN + half * EPI_COLS;
#pragma unroll
            for (int i = 0; i < EPI_COLS; i += 32) tmem_ld32(tbase + i, c + i);
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);  // accumulator drained: the MMA may reuse it
#ifdef TC_EXP
            if (TC_EXP == 2) {
                if (lane == 0) mbar_arrive(&cempty[cbuf]);
                continue;  // timing experiment: MMA + accumulator drain only
            }
#endif
            // local search: the 16-bit mask of group gi's columns inside the row's window (packed
            // window bounds, so the mask costs no registers across the tile)
            int gy0 = 0, gx0 = 0;  // domain (x, y) of the thread's first column of this tile
            // the thread's EPI_COLS columns span at most two domain rows when ndx >= EPI_COLS: the
            // window's columns are then two intervals [i1a, i1b] and [i2a, i2b] (empty: a > b)
            int i1a = 1, i1b = 0, i2a = 1, i2b = 0;
            if (LOCAL && live) {
                const int base = dt * BN + half * EPI_COLS;  // < 2^31 (domain indices)
                gy0 = base / p.ndx;
                gx0 = base - gy0 * p.ndx;
                const int lx = (int)(wx & 0xFFFF), hx = (int)(wx >> 16), ly = (int)(wy & 0xFFFF), hy = (int)(wy >> 16);
                const int split = p.ndx - gx0;  // first column of the next domain row
                if (gy0 >= ly && gy0 <= hy) {
                    i1a = max(lx - gx0, 0);
                    i1b = min(min(hx - gx0, split - 1), EPI_COLS - 1);
                }
                if (split < EPI_COLS && gy0 + 1 >= ly && gy0 + 1 <= hy) {
                    i2a = max(split + lx, split);
                    i2b = min(split + hx, EPI_COLS - 1);
                }
            }
            // exact 16-bit window mask of group gi (small images, ndx < EPI_COLS: column by column)
            auto group_mask = [&](int gi) -> uint32_t {
                if (p.ndx >= EPI_COLS) {
                    const int g0 = gi * GRP;
                    uint32_t mk = 0;
                    int lo = max(i1a - g0, 0), hi = min(i1b - g0, GRP - 1);
                    if (lo <= hi) mk |= ((2u << hi) - 1u) & ~((1u << lo) - 1u);
                    lo = max(i2a - g0, 0);
                    hi = min(i2b - g0, GRP - 1);
                    if (lo <= hi) mk |= ((2u << hi) - 1u) & ~((1u << lo) - 1u);
                    return mk;
                }
                const int lx = (int)(wx & 0xFFFF), hx = (int)(wx >> 16), ly = (int)(wy & 0xFFFF), hy = (int)(wy >> 16);
                int x = gx0 + gi * GRP, y = gy0;
                while (x >= p.ndx) {
                    x -= p.ndx;
                    y++;
                }
                uint32_t mk = 0;
                for (int j = 0; j < GRP; j++) {
                    if (y >= ly && y <= hy && x >= lx && x <= hx) mk |= 1u << j;
                    if (++x == p.ndx) {
                        x = 0;
                        y++;
                    }
                }
                return mk;
            };
            // level 1: one |max| per 16-column group against the row threshold (FMNMX3 per 2 columns);
            // local search: groups outside the window are skipped, partial ones filtered whole (the
            // rare path applies the exact column mask)
            unsigned gpass = 0;
#pragma unroll
            for (int gi = 0; gi < EPI_COLS / GRP; gi++) {
                float ma = 0.f, mb = 0.f;
#pragma unroll
                for (int j = 0; j < GRP; j += 4) {
                    ma = absmax3(ma, c[gi * GRP + j], c[gi * GRP + j + 1]);
                    mb = absmax3(mb, c[gi * GRP + j + 2], c[gi * GRP + j + 3]);
                }
                bool in = true;
                if (LOCAL) {
                    const int g0 = gi * GRP, g1 = g0 + GRP - 1;
                    in = p.ndx >= EPI_COLS ? ((i1a <= i1b && i1a <= g1 && i1b >= g0) || (i2a <= i2b && i2a <= g1 && i2b >= g0))
                                           : group_mask(gi) != 0;
                }
                gpass |= (live && in && fmaxf(ma, mb) >= thr) ? 1u << gi : 0u;
            }
#ifdef MNS_TC_STATS
            if (lane == 0) atomicAdd(&g_tc_stats[0], (unsigned long long)(EPI_COLS / GRP));
#endif
            if (__any_sync(FULL, gpass != 0)) {
                // rare path, per lane (no warp votes): the lane's passing columns one by one.  Level 2:
                // rigorous lower and upper bounds of the quantised value over the odd k2 from
                // x ~ N/(n sqrt D).  The lower bound discards; a survivor is queued for the exact warp
                // and its upper bound (a real candidate's value is at most that) tightens the lane's
                // threshold at once.
                while (*(volatile uint32_t *)c_issued < (uint32_t)(t + 1)) {
                }
                mbar_spin(&cfull[cbuf], (t / NCB) & 1);  // exact: copy t is issued (see the producer)
                const float *lq = reinterpret_cast<const float *>(sC + cbuf * CONST_BYTES);  // -Sq
                const float *ls = lq + BN;                                                  // sqrt_rd(D)
                const long long *ld = reinterpret_cast<const long long *>(sC + cbuf * CONST_BYTES + BN * 8);
#pragma unroll
                for (int gi = 0; gi < EPI_COLS / GRP; gi++) {
                    if (!(gpass & (1u << gi))) continue;
                    uint32_t mask = 0;
#pragma unroll
                    for (int j = 0; j < GRP; j++) {
                        mask |= (fabsf(c[gi * GRP + j]) >= thr ? 1u : 0u) << j;
                        stash[j * 32 + lane] = c[gi * GRP + j];  // lane-private column, for dynamic access
                    }
                    if (LOCAL) mask &= group_mask(gi);
#ifdef MNS_TC_STATS
                    atomicAdd(&g_tc_stats[1], 1ull);
#endif
                    while (mask) {
                        const int jj = __ffs(mask) - 1;
                        mask &= mask - 1;
                        const float x = stash[jj * 32 + lane];
                        if (!(fabsf(x) >= thr)) continue;  // the threshold may have tightened meanwhile
#ifdef MNS_TC_STATS
                        atomicAdd(&g_tc_stats[2], 1ull);
#endif
                        const int col = half * EPI_COLS + gi * GRP + jj;
                        if ((dt * BN + col) * (long long)p.dstride >= p.ndom) continue;
                        const float sg = ls[col];
                        const float n1 = x * sg;  // ~ N/n
                        // |n1 - N/n| <= sqrt(D) e_row + |x| |sqrt(D) - sg| + rounding of the product
                        const float err = fmaf(fabsf(x), 0x1p-20f, erow) * sg * 1.0001f + 1e-6f;
                        const long long Dx = ld[col];
                        const float Df = (float)Dx;
                        const float a = n64 * n1, eb = -n64 * err;
                        float vlb = INFINITY, vub = INFINITY;
#pragma unroll
                        for (int k2i = -7; k2i <= 7; k2i += 2) {
                            const float k2 = (float)k2i;
                            const float mid = k2 * fmaf(k2, Df, a);
                            vlb = fminf(vlb, fmaf(-fabsf(k2), eb, mid));
                            vub = fminf(vub, fmaf(fabsf(k2), eb, mid));
                        }
                        const float margin = 1024.f + 1e-5f * (fabsf(vlb) + fabsf(vub) + 49.f * Df + fabsf(a) * 7.f);
                        if (vstar != LLONG_MAX && vlb - margin > (float)vstar) continue;
                        set_threshold((long long)ceilf(vub + margin));
                        // queue it (16-B entry, sequence number written last)
                        const uint32_t slot = atomicAdd(q_head, 1u);
                        while (slot - *(volatile uint32_t *)q_tail >= (uint32_t)QSIZE) {
                        }
                        uint4 *e = reinterpret_cast<uint4 *>(queue) + (slot % QSIZE);
                        *reinterpret_cast<uint2 *>(e) = make_uint2((uint32_t)col | ((uint32_t)rl << 8), (uint32_t)m);
                        reinterpret_cast<uint32_t *>(e)[2] = (uint32_t)dt;
                        __threadfence_block();
                        reinterpret_cast<volatile uint32_t *>(e)[3] = slot + 1;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&cempty[cbuf]);  // done with this tile's constants
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            atomicAdd(q_done, 1u);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

// ---- operand preparation
// Thread per domain (consecutive threads = consecutive domains of a row: the byte loads of a warp
// coalesce): the exact pooled q (2x2 sums, u16), Sq, D = n Sqq - Sq^2, and the GEMM operand
// (q_k - Sq/n) / sqrt(D) in fp16 (0 for a flat domain) with the planar column constants.
template <int B>
__global__ void __launch_bounds__(128) pool_tc_kernel(const uint8_t *img, int W, int step, int ndx, long long ndom,
                                                      long long ndom_pad, uint16_t *pool, int32_t *psq,
                                                      long long *pD, __half *Q, float2 *consts) {
    constexpr int n = B * B;
    constexpr int RS = BK / 8 + 1;  // staged row stride in 16-B chunks (one pad chunk: conflict-free)
    __shared__ uint4 sq_rows[128 * RS], sp_rows[n == 64 ? 128 * RS : 1];
    const int tid = threadIdx.x;
    const long long d0 = blockIdx.x * 128ll, d = d0 + tid;  // ndom_pad is a multiple of 128
    float *cf = reinterpret_cast<float *>(consts) + (d / BN) * 2 * BN + d % BN;
    int q[n];
    int sq = 0;
    long long sqq = 0;
    if (d < ndom) {
        const int x = (int)(d % ndx) * step, y = (int)(d / ndx) * step;
#pragma unroll
        for (int i = 0; i < B; i++) {
            const uint8_t *p0 = img + (size_t)(y + 2 * i) * W + x, *p1 = p0 + W;
#pragma unroll
            for (int j = 0; j < B; j++) {
                const int v = (int)__ldg(p0 + 2 * j) + __ldg(p0 + 2 * j + 1) + __ldg(p1 + 2 * j) + __ldg(p1 + 2 * j + 1);
                q[i * B + j] = v;
                sq += v;
                sqq += v * v;
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < n; k++) q[k] = 0;
    }
    const long long D = n * sqq - (long long)sq * sq;
    if (d < ndom) {
        psq[d] = sq;
        pD[d] = D;
        if (n == 64) {
#pragma unroll
            for (int k = 0; k < n; k += 8)
                sp_rows[tid * RS + k / 8] =
                    make_uint4((uint32_t)q[k] | ((uint32_t)q[k + 1] << 16), (uint32_t)q[k + 2] | ((uint32_t)q[k + 3] << 16),
                               (uint32_t)q[k + 4] | ((uint32_t)q[k + 5] << 16), (uint32_t)q[k + 6] | ((uint32_t)q[k + 7] << 16));
        } else {
#pragma unroll
            for (int k = 0; k < n; k++) pool[d * n + k] = (uint16_t)q[k];
        }
    }
    const bool ok = d < ndom && D > 0;
    const float mean = (float)sq / (float)n;  // exact: Sq < 2^18, n a power of two
    const float inv = ok ? 1.0f / sqrtf((float)D) : 0.f;
    uint32_t h[BK / 2];
#pragma unroll
    for (int k = 0; k < BK; k += 2) {
        const float a = k < n && ok ? ((float)q[k < n ? k : 0] - mean) * inv : 0.f;
        const float b = k + 1 < n && ok ? ((float)q[k + 1 < n ? k + 1 : 0] - mean) * inv : 0.f;
        const __half2 hv = __floats2half2_rn(a, b);
        h[k / 2] = *reinterpret_cast<const uint32_t *>(&hv);
    }
#pragma unroll
    for (int i = 0; i < BK / 8; i++) sq_rows[tid * RS + i] = make_uint4(h[4 * i], h[4 * i + 1], h[4 * i + 2], h[4 * i + 3]);
    cf[0] = d < ndom ? -(float)sq : 0.f;
    cf[BN] = d < ndom ? __fsqrt_rd(__ll2float_rd(D)) : 0.f;
    __syncthreads();
    // the CTA's 128 rows are contiguous in global memory: coalesced 16-B stores
    uint4 *Qo = reinterpret_cast<uint4 *>(Q + d0 * BK);
    for (int c = tid; c < 128 * (BK / 8); c += 128) Qo[c] = sq_rows[(c / (BK / 8)) * RS + c % (BK / 8)];
    if (n == 64) {
        const int rows = (int)min(128ll, ndom - d0);
        uint4 *Po = reinterpret_cast<uint4 *>(pool + d0 * n);
        for (int c = tid; c < rows * 8; c += 128) Po[c] = sp_rows[(c / 8) * RS + c % 8];
    }
}

// Range operand rows (range, isometry), one warp per row: raw r (exact recompute) and centred
// r - Sr/n (the GEMM), both fp16, plus Sr, the constant-range flag and e_row = 2^-9 max |r - Sr/n|.
// row[k] = r(e) with k = src_t(e), i.e. e = src_{t^-1}(k) (rotations 5 and 6 are each other's inverse).
__global__ void range_rows_kernel(const uint8_t *img, int W, int B, int n_iso, int r0, int n_rows, int n_rows_pad,
                                  __half *Araw, __half *Ac, int32_t *row_sr, int32_t *row_flat, float *row_err) {
    const int lane = threadIdx.x & 31;
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= n_rows_pad) return;
    const int n = B * B;
    int v[2] = {0, 0};
    const bool real = row < n_rows;
    if (real) {
        const int ri = r0 + row / n_iso, t = row % n_iso, rpr = W / B;
        const int ti = t == 5 ? 6 : (t == 6 ? 5 : t);
        const int rx = (ri % rpr) * B, ry = (ri / rpr) * B;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int k = lane + 32 * h;
            if (k < n) {
                const int e = iso_src(ti, k / B, k % B, B);
                v[h] = img[(size_t)(ry + e / B) * W + rx + e % B];
            }
        }
    }
    const int sr = __reduce_add_sync(FULL, v[0] + v[1]);
    const int srr = __reduce_add_sync(FULL, v[0] * v[0] + v[1] * v[1]);
    const float mean = (float)sr / (float)n;  // exact
    float emax = 0.f;
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int k = lane + 32 * h;
        const float rc = real && k < n ? (float)v[h] - mean : 0.f;  // exact (multiple of 1/64, |rc| < 256)
        Araw[(size_t)row * BK + k] = __float2half_rn((float)v[h]);
        Ac[(size_t)row * BK + k] = __float2half_rn(rc);
        emax = fmaxf(emax, fabsf(rc));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) emax = fmaxf(emax, __shfl_xor_sync(FULL, emax, o));
    if (lane == 0) {
        row_sr[row] = sr;
        row_flat[row] = !real || ((long long)n * srr - (long long)sr * sr) == 0;
        row_err[row] = emax * 0x1p-9f + 1e-6f;
    }
}

// prepass column constants: every `stride`-th domain, contiguous, zero-padded
__global__ void gather_sample_kernel(const float2 *consts, const long long *pD, long long ndom, int stride,
                                     long long nsample_pad, float2 *cs, long long *ds) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nsample_pad;
         i += (long long)gridDim.x * blockDim.x) {
        const long long d = i * stride;
        const float *src = reinterpret_cast<const float *>(consts) + (d / BN) * 2 * BN + d % BN;
        float *dst = reinterpret_cast<float *>(cs) + (i / BN) * 2 * BN + i % BN;
        dst[0] = d < ndom ? src[0] : 0.f;
        dst[BN] = d < ndom ? src[BN] : 0.f;
        ds[i] = d < ndom ? pD[d] : 0;
    }
}

// Seeds every range's best key before the prepass (which otherwise starts without a threshold):
// one warp per range.  The domains around the co-centred one (offsets in {-B, -B/2, 0, B/2, B}^2,
// clamped and snapped to the stride) are scored against every isometry row of the range by the
// continuous bound N^2/D -- lane = (isometry, quarter of the 64 pixels), 16 integer MACs and two
// shuffles per candidate -- and the best one is evaluated exactly (any real candidate is a valid
// seed; the final argmin is unchanged).
__global__ void seed_best_kernel(const __half *A, const int32_t *row_sr, const uint16_t *pool, const int32_t *psq,
                                 const long long *pD, int W, int B, int step, int ndx, int ndy, int n_iso, int r0,
                                 int n_ranges, unsigned long long *best, int soff) {
    const int lane = threadIdx.x & 31;
    const int rr = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (rr >= n_ranges) return;
    const int n = B * B, ri = r0 + rr, rpr = W / B;
    const int rx = (ri % rpr) * B, ry = (ri / rpr) * B, sr = row_sr[rr * n_iso];
    // lane = (slot, quarter): slot s = lane / 4 scores the (candidate, isometry) pairs s, s + 8, ... of
    // the 25 * n_iso pairs (n_iso in {1, 8}, so a lane's isometry t = s % n_iso is fixed)
    const int sl = lane >> 2, k0 = (lane & 3) * 16, t = sl % n_iso;
    int rk[16];
    {
        const __half *ar = A + (size_t)(rr * n_iso + t) * BK + k0;
#pragma unroll
        for (int k = 0; k < 16; k++) rk[k] = k0 + k < n ? __half2int_rn(ar[k]) : 0;
    }
    float best_est = -1.f;
    int bd = -1, bc = 0;
    for (int p0 = 0; p0 < 25 * n_iso; p0 += 8) {
        const int pi = p0 + sl;
        const bool valid = pi < 25 * n_iso;
        const int c = valid ? pi / n_iso : 0;
        const int ox = (c % 5 - 2) * soff, oy = (c / 5 - 2) * soff;  // soff = B/2 (local: <= R/2)
        const int dx = clampi((rx - B / 2 + ox) / step, 0, ndx - 1), dy = clampi((ry - B / 2 + oy) / step, 0, ndy - 1);
        const int d = dy * ndx + dx;
        const uint16_t *qd = pool + (long long)d * n + k0;
        int part = 0;
#pragma unroll
        for (int k = 0; k < 16; k++) part += (k0 + k < n ? (int)__ldg(qd + k) : 0) * rk[k];
        part += __shfl_xor_sync(0xffffffffu, part, 1);
        part += __shfl_xor_sync(0xffffffffu, part, 2);  // C of (candidate c, isometry t), exact (< 2^24)
        const long long D = __ldg(pD + d);
        const float N = fmaf((float)n, (float)part, -(float)__ldg(psq + d) * (float)sr);
        const float est = valid && D > 0 ? N * N / (float)D : -1.f;
        if (est > best_est) {
            best_est = est;
            bd = d;
            bc = part;
        }
    }
    // warp argmax of the estimate (ties: any -- every candidate is valid)
    int bt = t;
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        const float e2 = __shfl_xor_sync(0xffffffffu, best_est, o);
        const int d2 = __shfl_xor_sync(0xffffffffu, bd, o), c2 = __shfl_xor_sync(0xffffffffu, bc, o),
                  t2 = __shfl_xor_sync(0xffffffffu, bt, o);
        if (e2 > best_est) {
            best_est = e2;
            bd = d2;
            bc = c2;
            bt = t2;
        }
    }
    if (lane == 0) {
        if (bd < 0) {  // flat range or flat domains only: the co-centred domain, isometry 0
            bd = clampi((ry - B / 2) / step, 0, ndy - 1) * ndx + clampi((rx - B / 2) / step, 0, ndx - 1);
            bt = 0;
            const uint16_t *qd = pool + (long long)bd * n;
            const __half *ar = A + (size_t)(rr * n_iso) * BK;
            bc = 0;
            for (int k = 0; k < n; k++) bc += (int)qd[k] * __half2int_rn(ar[k]);
        }
        const long long N = (long long)n * bc - (long long)psq[bd] * sr;  // exact
        atomicMin(&best[rr], make_key_cb(best_val_exact(N, pD[bd]), (long long)bd * n_iso + bt, key_cand_bits(n)));
    }
}

__global__ void flat_key_kernel(const long long *pD, long long ndom, int n_iso, int n, unsigned long long *key) {
    unsigned long long best = ~0ull;
    for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < ndom;
         d += (long long)gridDim.x * blockDim.x) {
        const unsigned long long k = make_key_cb(pD[d], d * n_iso, key_cand_bits(n));  // constant range: val = D (k2 = +-1), iso 0
        best = k < best ? k : best;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(FULL, best, o);
        best = other < best ? other : best;
    }
    if ((threadIdx.x & 31) == 0) atomicMin(key, best);
}

// ---- local search (encoder.py:312-347) on the same tensor-core pipeline
// Constant ranges: every candidate's value is its D (k2 = +-1, s = 0.125 as the reference's
// fit gives s = 0); the window's minimum D (lowest index on ties, isometry 0). One warp per range.
__global__ void local_flat_kernel(const int32_t *row_flat, const long long *pD, int W, int H, int B, int R, int ndx,
                                  int ndy, int n_iso, int n_ranges, unsigned long long *best) {
    const int lane = threadIdx.x & 31;
    const int rr = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (rr >= n_ranges || !row_flat[rr * n_iso]) return;
    const int rpr = W / B;
    const int bx = clampi((rr % rpr) * B - B / 2, 0, W - 2 * B), by = clampi((rr / rpr) * B - B / 2, 0, H - 2 * B);
    const int lx = clampi(bx - R, 0, ndx - 1), hx = clampi(bx + R, 0, ndx - 1);
    const int ly = clampi(by - R, 0, ndy - 1), hy = clampi(by + R, 0, ndy - 1);
    const int wx = hx - lx + 1, nwin = wx * (hy - ly + 1);
    unsigned long long k = ~0ull;
    for (int i = lane; i < nwin; i += 32) {
        const long long d = (long long)(ly + i / wx) * ndx + lx + i % wx;
        const unsigned long long key = make_key_cb(pD[d], d * n_iso, key_cand_bits(B * B));
        k = key < k ? key : k;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(FULL, k, o);
        k = other < k ? other : k;
    }
    if (lane == 0) atomicMin(&best[rr], k);
}

// The (M tile, domain tile) units of the local search: per M tile (one block) the domain tiles that
// meet the union of its ranges' windows.  The ranges of an M tile are consecutive in raster order,
// so per range row the union is one rectangle of origins; its rows mark tile intervals in a shared
// bitmap over the tile's hull, read back in order into scratch[m * cap ..], count in counts[m].
constexpr int LT_BITS = 32768;  // hull bound (domain tiles) per M tile
__global__ void local_units_kernel(int W, int H, int B, int R, int ndx, int ndy, int n_iso, int n_rows, int cap,
                                   uint32_t *scratch, int *counts) {
    __shared__ uint32_t bm[LT_BITS / 32];
    __shared__ int hull[2];
    const int m = blockIdx.x, tid = threadIdx.x;
    const int rpr = W / B;
    const int row0 = m * (MH * BM), row1 = min(n_rows, row0 + MH * BM);
    const int ra = row0 / n_iso, rb = (row1 - 1) / n_iso;  // the tile's ranges [ra, rb]
    auto win_y = [&](int rowr, int &lo, int &hi) {
        const int by = clampi(rowr * B - B / 2, 0, H - 2 * B);
        lo = clampi(by - R, 0, ndy - 1);
        hi = clampi(by + R, 0, ndy - 1);
    };
    auto win_x = [&](int c0, int c1, int &lo, int &hi) {  // union over range columns c0..c1 of one row
        lo = clampi(clampi(c0 * B - B / 2, 0, W - 2 * B) - R, 0, ndx - 1);
        hi = clampi(clampi(c1 * B - B / 2, 0, W - 2 * B) + R, 0, ndx - 1);
    };
    if (tid == 0) {
        int ylo, yhi, tmp;
        win_y(ra / rpr, ylo, tmp);
        win_y(rb / rpr, tmp, yhi);
        hull[0] = (int)(((long long)ylo * ndx) / BN);
        hull[1] = (int)(((long long)yhi * ndx + ndx - 1) / BN);
    }
    for (int i = tid; i < LT_BITS / 32; i += blockDim.x) bm[i] = 0;
    __syncthreads();
    const int h0 = hull[0];
    const int nh = min(hull[1] - h0 + 1, LT_BITS);
    for (int rowr = ra / rpr; rowr <= rb / rpr; rowr++) {
        const int c0 = rowr == ra / rpr ? ra % rpr : 0, c1 = rowr == rb / rpr ? rb % rpr : rpr - 1;
        int ylo, yhi, xlo, xhi;
        win_y(rowr, ylo, yhi);
        win_x(c0, c1, xlo, xhi);
        for (int y = ylo + tid; y <= yhi; y += blockDim.x) {
            const long long a = (long long)y * ndx + xlo, b = (long long)y * ndx + xhi;
            for (long long t = a / BN; t <= b / BN; t++) {
                const int bit = (int)(t - h0);
                if (bit >= 0 && bit < nh) atomicOr(&bm[bit >> 5], 1u << (bit & 31));
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        // centre-out order (tiles alternately after and before the one holding the M tile's central
        // window origin): the best candidates are usually near the range, so the row thresholds
        // tighten early and fewer elements reach the exact evaluation
        const int rc = (ra + rb) / 2;
        int cy, tmp;
        win_y(rc / rpr, cy, tmp);
        cy = (cy + tmp) / 2;
        int cx0, cx1;
        win_x(rc % rpr, rc % rpr, cx0, cx1);
        const int c0 = min(max((int)(((long long)cy * ndx + (cx0 + cx1) / 2) / BN) - h0, 0), nh - 1);
        int k = 0;
        for (int dlt = 0; dlt < nh; dlt++) {
            for (int sgn = 0; sgn < (dlt ? 2 : 1); sgn++) {
                const int b = sgn ? c0 - dlt : c0 + dlt;
                if (b < 0 || b >= nh || !((bm[b >> 5] >> (b & 31)) & 1u)) continue;
                if (k < cap) scratch[(long long)m * cap + k] = (uint32_t)(h0 + b);
                k++;
            }
        }
        counts[m] = min(k, cap);
    }
}

// exclusive scan of the per-M-tile counts (one block of 1024 threads, each a contiguous chunk)
__global__ void local_units_scan_kernel(const int *counts, int n_mt, int *offsets, int *n_units) {
    __shared__ int part[1024];
    const int tid = threadIdx.x, per = (n_mt + 1023) / 1024, a = tid * per, b = min(n_mt, a + per);
    int s = 0;
    for (int m = a; m < b; m++) s += counts[m];
    part[tid] = s;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scan
        const int v = tid >= o ? part[tid - o] : 0;
        __syncthreads();
        part[tid] += v;
        __syncthreads();
    }
    int run = part[tid] - s;
    for (int m = a; m < b; m++) {
        offsets[m] = run;
        run += counts[m];
    }
    if (tid == 1023) *n_units = part[1023];
}

// the flattened (m, dt) unit list, M-major (one block per M tile)
__global__ void local_units_flatten_kernel(const uint32_t *scratch, const int *counts, const int *offsets, int cap,
                                           uint2 *units) {
    const int m = blockIdx.x, c = counts[m], o = offsets[m];
    for (int i = threadIdx.x; i < c; i += blockDim.x)
        units[o + i] = make_uint2((uint32_t)m, scratch[(long long)m * cap + i]);
}

int sm_count_tc() {
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

#ifdef MNS_TC_STATS
extern "C" void mns_tc_stats(unsigned long long *out) {
    cudaMemcpyFromSymbol(out, g_tc_stats, sizeof(g_tc_stats));
    unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(g_tc_stats, z, sizeof(z));
}
#endif

int64_t search_tc_workspace_bytes(int W, int H, int B, int step, int n_iso) {
    const long long ndx = (W - 2 * B) / step + 1, ndy = (H - 2 * B) / step + 1, ndom = ndx * ndy;
    const long long ndom_pad = (ndom + BN - 1) / BN * BN;
    const long long rows_pad = ((long long)(W / B) * (H / B) * n_iso + MH * BM - 1) / (MH * BM) * (MH * BM);
    const long long nsample_pad = (ndom / TC_SAMPLE + 1 + BN - 1) / BN * BN;
    return ndom_pad * BK * 2 + ndom_pad * 8 + 2 * rows_pad * BK * 2 + rows_pad * 12 + nsample_pad * 16 + 4096;
}

// The tensor-core path; it also builds the pooled domains (pool, psq, pD) the finalize step reads.
// *handled = false (nothing launched) when B or the workspace rule it out.
int full_search_tc(const uint8_t *img, int W, int H, int B, int step, int n_iso, int r0, int r1,
                   uint16_t *pool, int32_t *psq, long long *pD, long long ndom,
                   unsigned long long *best, void *tc_ws, cudaStream_t st, bool *handled) {
    *handled = false;
    if (!(B == 2 || B == 4 || B == 8) || !tc_ws) return 0;
    const int n = B * B;
    const long long ndom_pad = (ndom + BN - 1) / BN * BN;
    const int n_rows = (r1 - r0) * n_iso;
    const int n_rows_pad = (n_rows + MH * BM - 1) / (MH * BM) * (MH * BM);
    char *q = (char *)tc_ws;
    __half *Q = (__half *)q;
    q += ndom_pad * BK * 2;
    float2 *consts = (float2 *)q;
    q += ndom_pad * 8;
    __half *Araw = (__half *)q;
    q += (long long)n_rows_pad * BK * 2;
    __half *Ac = (__half *)q;
    q += (long long)n_rows_pad * BK * 2;
    int32_t *row_sr = (int32_t *)q;
    q += (long long)n_rows_pad * 4;
    int32_t *row_flat = (int32_t *)q;
    q += (long long)n_rows_pad * 4;
    float *row_err = (float *)q;
    q += (long long)n_rows_pad * 4;
    q = (char *)(((uintptr_t)q + 255) & ~(uintptr_t)255);
    const long long nsample_pad = (ndom / TC_SAMPLE + 1 + BN - 1) / BN * BN;
    float2 *cons_s = (float2 *)q;
    q += nsample_pad * 8;
    long long *pD_s = (long long *)q;
    q += nsample_pad * 8;
    unsigned long long *fkey = (unsigned long long *)(((uintptr_t)q + 255) & ~(uintptr_t)255);

    const int sms = sm_count_tc();
    {
        const int ndx = (W - 2 * B) / step + 1;
        const unsigned blocks = (unsigned)((ndom_pad + 127) / 128);
        switch (B) {
        case 2: pool_tc_kernel<2><<<blocks, 128, 0, st>>>(img, W, step, ndx, ndom, ndom_pad, pool, psq, pD, Q, consts); break;
        case 4: pool_tc_kernel<4><<<blocks, 128, 0, st>>>(img, W, step, ndx, ndom, ndom_pad, pool, psq, pD, Q, consts); break;
        default: pool_tc_kernel<8><<<blocks, 128, 0, st>>>(img, W, step, ndx, ndom, ndom_pad, pool, psq, pD, Q, consts); break;
        }
    }
    range_rows_kernel<<<(n_rows_pad + 7) / 8, 256, 0, st>>>(img, W, B, n_iso, r0, n_rows, n_rows_pad, Araw, Ac, row_sr,
                                                          row_flat, row_err);
    MNS_CUDA_TRY(cudaMemsetAsync(fkey, 0xFF, 8, st));
    flat_key_kernel<<<148, 256, 0, st>>>(pD, ndom, n_iso, B * B, fkey);
#ifndef TC_NO_SEED
    {
        const int ndx = (W - 2 * B) / step + 1, ndy = (int)(ndom / ndx);
        seed_best_kernel<<<(r1 - r0 + 7) / 8, 256, 0, st>>>(Araw, row_sr, pool, psq, pD, W, B, step, ndx, ndy, n_iso,
                                                            r0, r1 - r0, best, B / 2);
    }
#endif

    CUtensorMap tmA, tmB, tmS;
    constexpr int SAMPLE = TC_SAMPLE;  // prepass: every TC_SAMPLE-th domain seeds each row's best (strided TMA view)
    const long long nsample = (ndom + SAMPLE - 1) / SAMPLE;
    if (encode_tmap_2d_swizzled(&tmA, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, Ac, BK, n_rows_pad, BK * 2, BK, BM)) return -1;
    if (encode_tmap_2d_swizzled(&tmB, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, Q, BK, ndom_pad, BK * 2, BK, BN)) return -1;
    if (encode_tmap_2d_swizzled(&tmS, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, Q, BK, nsample, (uint64_t)BK * 2 * SAMPLE, BK,
                                BN))
        return -1;

    TcParams p{};
    p.n_rows = n_rows;
    p.n_iso = n_iso;
    p.r0 = r0;
    p.n = n;
    p.ndom = ndom;
    p.consts = consts;
    p.pD = pD;
    p.pool = pool;
    p.araw = Araw;
    p.row_sr = row_sr;
    p.row_flat = row_flat;
    p.row_err = row_err;
    p.flat_key = fkey;
    p.local_R = -1;
    p.best = best;
    {
        static std::atomic<unsigned long long> done{0};
        MNS_CUDA_TRY(ensure_dynamic_smem(full_search_tc_kernel<false>, SMEM_BYTES, done));
    }
    const long long n_mt = n_rows_pad / (MH * BM);
#ifdef TC_NO_PREPASS
    if (false) {
#else
    if (ndom >= 16 * SAMPLE) {  // prepass over the sample
#endif
        gather_sample_kernel<<<64, 256, 0, st>>>(consts, pD, ndom, SAMPLE, nsample_pad, cons_s, pD_s);
        TcParams q2 = p;
        q2.consts = cons_s;
        q2.pD = pD_s;
        q2.dstride = SAMPLE;
        q2.n_dt = (int)((nsample + BN - 1) / BN);
        q2.n_units = n_mt * q2.n_dt;
        const int grid = (int)(q2.n_units < sms ? q2.n_units : sms);
        full_search_tc_kernel<false><<<grid, NTHREADS, SMEM_BYTES, st>>>(tmA, tmS, q2);
    }
    p.dstride = 1;
    p.n_dt = (int)(ndom_pad / BN);
    p.n_units = n_mt * p.n_dt;
    const int grid = (int)(p.n_units < sms ? p.n_units : sms);
    full_search_tc_kernel<false><<<grid, NTHREADS, SMEM_BYTES, st>>>(tmA, tmB, p);
    MNS_CUDA_TRY(cudaGetLastError());
    *handled = true;
    return 0;
}


// Local search on the tensor-core pipeline (local_R >= 0): the full-search kernel walks only the
// units that meet some window and masks every element outside its row's window.  Workspace:
// local_search_tc_workspace_bytes; pool/psq/pD/best as for the full search.
int64_t local_units_cap(int W, int H, int B, int R, int n_iso) {
    const int rpr = W / B, ndx = W - 2 * B + 1;
    const int range_rows = (MH * BM / n_iso + rpr - 1) / rpr + 1;  // range rows an M tile spans
    const long long span = (long long)(range_rows * B + 2 * R + 2) * ndx;
    return span / BN + 3;
}

int64_t local_search_tc_workspace_bytes(int W, int H, int B, int R, int n_iso) {
    const long long n_rows = (long long)(W / B) * (H / B) * n_iso;
    const long long n_mt = (n_rows + MH * BM - 1) / (MH * BM);
    const long long cap = local_units_cap(W, H, B, R, n_iso);
    return search_tc_workspace_bytes(W, H, B, 1, n_iso) + 256 + n_mt * 4 + 256 + 256 + n_mt * 4 + 256 +
           n_mt * cap * 4 + 256 + n_mt * cap * 8 + 256;
}

int local_search_tc(const uint8_t *img, int W, int H, int R, int n_iso, uint16_t *pool, int32_t *psq, long long *pD,
                    long long ndom, unsigned long long *best, void *tc_ws, cudaStream_t st) {
    const int B = 8, n = 64;
    const int ndx = W - 2 * B + 1, ndy = H - 2 * B + 1;
    const long long ndom_pad = (ndom + BN - 1) / BN * BN;
    const int n_ranges = (W / B) * (H / B);
    const int n_rows = n_ranges * n_iso;
    const int n_rows_pad = (n_rows + MH * BM - 1) / (MH * BM) * (MH * BM);
    const int n_mt = n_rows_pad / (MH * BM);
    const long long cap = local_units_cap(W, H, B, R, n_iso);
    MNS_CHECK_ARG(cap <= LT_BITS, "local search window hull too large for the tensor-core path");
    char *q = (char *)tc_ws;
    __half *Q = (__half *)q;
    q += ndom_pad * BK * 2;
    float2 *consts = (float2 *)q;
    q += ndom_pad * 8;
    __half *Araw = (__half *)q;
    q += (long long)n_rows_pad * BK * 2;
    __half *Ac = (__half *)q;
    q += (long long)n_rows_pad * BK * 2;
    int32_t *row_sr = (int32_t *)q;
    q += (long long)n_rows_pad * 4;
    int32_t *row_flat = (int32_t *)q;
    q += (long long)n_rows_pad * 4;
    float *row_err = (float *)q;
    q = (char *)tc_ws + search_tc_workspace_bytes(W, H, B, 1, n_iso);
    q = (char *)(((uintptr_t)q + 255) & ~(uintptr_t)255);
    int *counts = (int *)q;
    q += n_mt * 4 + 256;
    q = (char *)(((uintptr_t)q + 255) & ~(uintptr_t)255);
    int *offsets = (int *)q;
    q += n_mt * 4 + 256;
    q = (char *)(((uintptr_t)q + 255) & ~(uintptr_t)255);
    uint32_t *scratch = (uint32_t *)q;
    q += n_mt * cap * 4 + 256;
    q = (char *)(((uintptr_t)q + 255) & ~(uintptr_t)255);
    uint2 *units = (uint2 *)q;
    q += n_mt * cap * 8 + 256;
    int *n_units = counts + n_mt;  // the slot after the counts (256 B of slack reserved there)

    const unsigned blocks = (unsigned)((ndom_pad + 127) / 128);
    pool_tc_kernel<8><<<blocks, 128, 0, st>>>(img, W, 1, ndx, ndom, ndom_pad, pool, psq, pD, Q, consts);
    range_rows_kernel<<<(n_rows_pad + 7) / 8, 256, 0, st>>>(img, W, B, n_iso, 0, n_rows, n_rows_pad, Araw, Ac, row_sr,
                                                          row_flat, row_err);
    const int soff = R / 2 < B / 2 ? R / 2 : B / 2;  // seeds stay inside the window
    seed_best_kernel<<<(n_ranges + 7) / 8, 256, 0, st>>>(Araw, row_sr, pool, psq, pD, W, B, 1, ndx, ndy, n_iso, 0,
                                                        n_ranges, best, soff);
    local_flat_kernel<<<(n_ranges + 7) / 8, 256, 0, st>>>(row_flat, pD, W, H, B, R, ndx, ndy, n_iso, n_ranges, best);
    local_units_kernel<<<n_mt, 256, 0, st>>>(W, H, B, R, ndx, ndy, n_iso, n_rows, (int)cap, scratch, counts);
    local_units_scan_kernel<<<1, 1024, 0, st>>>(counts, n_mt, offsets, n_units);
    local_units_flatten_kernel<<<n_mt, 128, 0, st>>>(scratch, counts, offsets, (int)cap, units);

    CUtensorMap tmA, tmB;
    if (encode_tmap_2d_swizzled(&tmA, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, Ac, BK, n_rows_pad, BK * 2, BK, BM)) return -1;
    if (encode_tmap_2d_swizzled(&tmB, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, Q, BK, ndom_pad, BK * 2, BK, BN)) return -1;
    TcParams p{};
    p.n_rows = n_rows;
    p.n_iso = n_iso;
    p.r0 = 0;
    p.n = n;
    p.ndom = ndom;
    p.consts = consts;
    p.pD = pD;
    p.pool = pool;
    p.araw = Araw;
    p.row_sr = row_sr;
    p.row_flat = row_flat;
    p.row_err = row_err;
    p.flat_key = nullptr;
    p.best = best;
    p.dstride = 1;
    p.n_dt = (int)(ndom_pad / BN);
    p.n_units = 0;
    p.units = units;
    p.n_units_dev = n_units;
    p.local_R = R;
    p.W = W;
    p.H = H;
    p.B = B;
    p.ndx = ndx;
    p.ndy = ndy;
    {
        static std::atomic<unsigned long long> done{0};
        MNS_CUDA_TRY(ensure_dynamic_smem(full_search_tc_kernel<true>, SMEM_BYTES, done));
    }
    const int sms = sm_count_tc();
    full_search_tc_kernel<true><<<sms, NTHREADS, SMEM_BYTES, st>>>(tmA, tmB, p);
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

}  // namespace mns
