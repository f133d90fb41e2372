// Shared device/host helpers for libmns_b200 (sm_100a).
#pragma once

#include <atomic>

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mns_b200.h"

namespace mns {

// Thread-local last error (mns_last_error) -- set by the ABI layer.
void set_error(const char *fmt, ...);

#define MNS_CUDA_TRY(expr)                                                               \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess) {                                                         \
            ::mns::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),     \
                             __FILE__, __LINE__);                                        \
            return -1;                                                                   \
        }                                                                                \
    } while (0)

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is a per-device setting: set it once per
// (kernel, device) -- `done` is the call site's bitmask of devices already configured.
template <class Kernel>
inline cudaError_t ensure_dynamic_smem(Kernel kernel, int bytes, std::atomic<unsigned long long> &done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

#define MNS_CHECK_ARG(cond, msg)                                                         \
    do {                                                                                 \
        if (!(cond)) {                                                                   \
            ::mns::set_error("invalid argument: %s", msg);                               \
            return -2;                                                                   \
        }                                                                                \
    } while (0)

// Largest double x with fl(sqrt(x)) <= E (IEEE sqrt is correctly rounded, so
// "rms <= E" <=> "mean square <= bound(E)" exactly).  +inf for E = +inf.
double sqrt_bound(double E);

__host__ __device__ inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Isometry t of a B x B block (full-search extension; the reference has none):
// d_t(i, j) = d(src_t(i, j)); t = 0 is the identity.
// Search argmin keys: (val + 2^(63-cb)) << cb | candidate, lexicographic = (value, first index).
// |val| = |min_k2 (k2^2 D - 64 k2 N)| < n^2 * 4.18e7 (|N| <= n^2 * 65025 by Cauchy-Schwarz,
// D <= n^2 * 260100), so the value needs 31/35/39/43 bits at n = 4/16/64/256 and the candidate
// index gets the rest: 33/29/25/21 bits (B = 8: 2^25 (domain, isometry) pairs).
__host__ __device__ inline int key_cand_bits(int n) { return n <= 4 ? 33 : n <= 16 ? 29 : n <= 64 ? 25 : 21; }
__host__ __device__ inline unsigned long long make_key_cb(long long val, long long cand, int cb) {
    return ((unsigned long long)(val + (1ll << (63 - cb))) << cb) | (unsigned long long)cand;
}
__host__ __device__ inline long long key_val(unsigned long long key, int cb) {
    return (long long)(key >> cb) - (1ll << (63 - cb));
}
__host__ __device__ inline long long key_cand(unsigned long long key, int cb) {
    return (long long)(key & ((1ull << cb) - 1));
}

__host__ __device__ inline int iso_src(int t, int i, int j, int B) {
    switch (t) {
    case 0: return i * B + j;                      // identity
    case 1: return i * B + (B - 1 - j);            // mirror columns
    case 2: return (B - 1 - i) * B + j;            // mirror rows
    case 3: return (B - 1 - i) * B + (B - 1 - j);  // rotate 180
    case 4: return j * B + i;                      // transpose
    case 5: return (B - 1 - j) * B + i;            // rotate 90 clockwise
    case 6: return j * B + (B - 1 - i);            // rotate 90 counter-clockwise
    default: return (B - 1 - j) * B + (B - 1 - i); // anti-transpose
    }
}

// numpy pairwise_sum for float64 (loops_utils.h.src), restated; a points to
// shared or local memory.  n <= 256.
__device__ inline double pw_sum_dev(const double *a, int n) {
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; i++) res = __dadd_rn(res, a[i]);
        return res;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] = a[j];
        int i;
        for (i = 8; i < n - (n % 8); i += 8)
#pragma unroll
            for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], a[i + j]);
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; i++) res = __dadd_rn(res, a[i]);
        return res;
    }
    // n in (128, 256]: split at n/2 rounded down to a multiple of 8 (one level suffices)
    int n2 = n / 2;
    n2 -= n2 % 8;
    double lo, hi;
    {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j];
        int i;
        for (i = 8; i < n2 - (n2 % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], a[i + j]);
        lo = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                       __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n2; i++) lo = __dadd_rn(lo, a[i]);
    }
    {
        const double *b = a + n2;
        int m = n - n2;
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = b[j];
        int i;
        for (i = 8; i < m - (m % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], b[i + j]);
        hi = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                       __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < m; i++) hi = __dadd_rn(hi, b[i]);
    }
    return __dadd_rn(lo, hi);
}

// Packed fp32 pair FMA (sm_100 FFMA2): per lane the same IEEE rounding as fmaf.
__device__ __forceinline__ float2 ffma2_rn(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}

__device__ inline unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ inline unsigned long long ld_acquire_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ inline void st_release_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ inline unsigned long long ld_relaxed_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Decoupled look-back (single-pass exclusive scan over tiles in launch order).
// status[] must be zeroed before the launch.  Called by ONE thread per tile;
// returns the exclusive prefix of `agg` over tiles [0, tile).
constexpr unsigned long long LB_AGG = 1ull << 62;
constexpr unsigned long long LB_PREFIX = 2ull << 62;
constexpr unsigned long long LB_MASK = (1ull << 62) - 1;

__device__ inline long long lookback_exclusive(unsigned long long *status, long long tile, long long agg) {
    if (tile == 0) {
        st_release_u64(&status[0], LB_PREFIX | (unsigned long long)agg);
        return 0;
    }
    st_release_u64(&status[tile], LB_AGG | (unsigned long long)agg);
    long long excl = 0;
    long long p = tile - 1;
    while (true) {
        unsigned long long v = ld_acquire_u64(&status[p]);
        unsigned long long flag = v & ~LB_MASK;
        if (flag == 0) {
            __nanosleep(32);
            continue;
        }
        excl += (long long)(v & LB_MASK);
        if (flag == LB_PREFIX) break;
        --p;
    }
    st_release_u64(&status[tile], LB_PREFIX | (unsigned long long)(excl + agg));
    return excl;
}

// Warp-cooperative decoupled look-back: called by ALL 32 lanes of one warp; the
// 32 lanes poll 32 predecessors at once (relaxed loads: each status word is a
// self-contained flag|value), wait only until every predecessor up to the nearest
// inclusive prefix has published (not the whole window), sum those aggregates, and
// slide the window back while none is inclusive.  Returns the exclusive prefix
// (same value in every lane).
__device__ inline long long lookback_exclusive_warp(unsigned long long *status, long long tile, long long agg) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) st_release_u64(&status[0], LB_PREFIX | (unsigned long long)agg);
        return 0;
    }
    if (lane == 0) st_release_u64(&status[tile], LB_AGG | (unsigned long long)agg);
    long long excl = 0;
    long long base = tile - 1;
    while (true) {
        const long long idx = base - lane;
        unsigned long long v = idx >= 0 ? ld_relaxed_u64(&status[idx]) : LB_PREFIX;
        unsigned pm;
        while (true) {  // wait only for the predecessors up to the nearest inclusive prefix
            const unsigned inv = __ballot_sync(0xffffffffu, (v & ~LB_MASK) == 0);
            pm = __ballot_sync(0xffffffffu, (v & ~LB_MASK) == LB_PREFIX);
            if (inv == 0 || (pm && __ffs(pm) < __ffs(inv))) break;
            __nanosleep(20);
            if ((v & ~LB_MASK) == 0) v = ld_relaxed_u64(&status[idx]);
        }
        const int first = pm ? __ffs(pm) - 1 : 32;  // nearest predecessor holding an inclusive prefix
        long long c = lane <= first ? (long long)(v & LB_MASK) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        excl += c;
        if (pm) break;
        base -= 32;
    }
    if (lane == 0) st_release_u64(&status[tile], LB_PREFIX | (unsigned long long)(excl + agg));
    return excl;
}

}  // namespace mns
