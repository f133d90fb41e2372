// Exact fp64 Jacobi decode with the reference's early stop (decoder.py:66-77).
//
// The reference iterates decode_step in float64 and stops after the first sweep whose
// max|nxt - current| is below stop_delta (decoder.py:70-75).  An fp32 raster cannot make that
// decision exactly (a sweep whose true delta lies within fp32 error of stop_delta could stop one
// sweep early or late), so codes decoded with stop_delta > 0 run here: every sweep is the
// bit-exact fp64 step of decode_step_f64 (numpy's downsample order, pairwise mean, unfused
// mul/add, clip), the sweep's max|delta| is an exact fp64 max (order-independent) folded into a
// state word, and a one-thread kernel applies the reference's test.  Sweeps after convergence are
// no-ops (every kernel reads the converged flag first), so the host enqueues max_iters sweeps
// with no synchronisation; the final uint8 image is clip(floor(x + 0.5)) of the raster that holds
// the last sweep -- bit-identical to the reference's decode.
//
// Strips (multi-GPU): the same kernels on a rank's strip with a 16-row halo ("virtual global"
// base pointers); between the sweep and the decision the caller all-reduces (max) the state's
// delta word over the ranks (sharding.StripDecoderF64), so every rank stops at the same sweep.
//
// State (int64[4]): [0] converged flag, [1] sweeps done, [2] this sweep's max|delta| (fp64 bits,
// non-negative, so the integer max is the fp64 max), [3] spare.

#include <cooperative_groups.h>
#include <math.h>

#include "mns_common.cuh"

namespace mns {

namespace {

constexpr unsigned FULL = 0xffffffffu;

// One unit of decode_step (decoder.py:32-63, transform.py:63-66) in the reference's fp64 order.
// Returns this unit's max |v - cur| over its pixels.
__device__ double paint_unit_f64(int x, int y, int size, int iso, int dx, int dy, double s, double o, int W,
                                 const double *cur, double *out) {
    const int m = size * size;
    double d[256];
    for (int i = 0; i < size; i++)
        for (int j = 0; j < size; j++) {  // isometry extension: d_t(i, j) = d(src_t(i, j)), in output order
            const int k = iso ? iso_src(iso, i, j, size) : i * size + j;
            const double *pp = cur + (size_t)(dy + 2 * (k / size)) * W + dx + 2 * (k % size);
            d[i * size + j] = __dmul_rn(__dadd_rn(__dadd_rn(__dadd_rn(pp[0], pp[1]), pp[W]), pp[W + 1]), 0.25);
        }
    const double dm = __ddiv_rn(pw_sum_dev(d, m), (double)m);
    double dmax = 0.0;
    for (int i = 0; i < size; i++)
        for (int j = 0; j < size; j++) {
            double v = __dadd_rn(__dmul_rn(s, __dsub_rn(d[i * size + j], dm)), o);
            v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
            const size_t idx = (size_t)(y + i) * W + x + j;
            dmax = fmax(dmax, fabs(__dsub_rn(v, cur[idx])));
            out[idx] = v;
        }
    return dmax;
}

// numpy's pairwise float64 sum (loops_utils.h.src) for a compile-time n <= 128, a in registers
template <int NN>
__device__ __forceinline__ double pw_sum_fixed(const double (&a)[NN]) {
    if constexpr (NN < 8) {
        double res = 0.0;
#pragma unroll
        for (int i = 0; i < NN; i++) res = __dadd_rn(res, a[i]);
        return res;
    } else {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] = a[j];
#pragma unroll
        for (int i = 8; i < NN - (NN % 8); i += 8)
#pragma unroll
            for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], a[i + j]);
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
#pragma unroll
        for (int i = NN - (NN % 8); i < NN; i++) res = __dadd_rn(res, a[i]);
        return res;
    }
}

// paint_unit_f64 for a compile-time side (2 or 4: the bulk of quadtree codes), everything in
// registers; the domain's 2x2 cells are read as double2 (even domain origins for side >= 4)
template <int S>
__device__ __forceinline__ double paint_unit_f64_fixed(int x, int y, int iso, int dx, int dy, double s, double o,
                                                       int W, const double *cur, double *out) {
    double d[S * S];
#pragma unroll
    for (int i = 0; i < S; i++)
#pragma unroll
        for (int j = 0; j < S; j++) {
            const int k = iso ? iso_src(iso, i, j, S) : i * S + j;
            const double *pp = cur + (size_t)(dy + 2 * (k / S)) * W + dx + 2 * (k % S);
            double a0, a1, b0, b1;
            if (S >= 4 && !((dx | W) & 1)) {  // 16-byte aligned pairs (quadtree domains; search domains may be odd)
                const double2 ra = *reinterpret_cast<const double2 *>(pp), rb = *reinterpret_cast<const double2 *>(pp + W);
                a0 = ra.x; a1 = ra.y; b0 = rb.x; b1 = rb.y;
            } else {
                a0 = pp[0]; a1 = pp[1]; b0 = pp[W]; b1 = pp[W + 1];
            }
            d[i * S + j] = __dmul_rn(__dadd_rn(__dadd_rn(__dadd_rn(a0, a1), b0), b1), 0.25);
        }
    const double dm = __ddiv_rn(pw_sum_fixed<S * S>(d), (double)(S * S));
    double dmax = 0.0;
    if ((x | W) & 1) {  // odd origin or pitch (unit lists of arbitrary images): scalar accesses
#pragma unroll
        for (int i = 0; i < S; i++)
#pragma unroll
            for (int j = 0; j < S; j++) {
                double v = __dadd_rn(__dmul_rn(s, __dsub_rn(d[i * S + j], dm)), o);
                v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
                const size_t idx = (size_t)(y + i) * W + x + j;
                dmax = fmax(dmax, fabs(__dsub_rn(v, cur[idx])));
                out[idx] = v;
            }
        return dmax;
    }
#pragma unroll
    for (int i = 0; i < S; i++)
#pragma unroll
        for (int j = 0; j < S; j += 2) {  // 16-byte pairs
            const size_t idx = (size_t)(y + i) * W + x + j;
            const double2 c = *reinterpret_cast<const double2 *>(cur + idx);
            double v0 = __dadd_rn(__dmul_rn(s, __dsub_rn(d[i * S + j], dm)), o);
            double v1 = __dadd_rn(__dmul_rn(s, __dsub_rn(d[i * S + j + 1], dm)), o);
            v0 = v0 < 0.0 ? 0.0 : (v0 > 255.0 ? 255.0 : v0);
            v1 = v1 < 0.0 ? 0.0 : (v1 > 255.0 ? 255.0 : v1);
            dmax = fmax(dmax, fmax(fabs(__dsub_rn(v0, c.x)), fabs(__dsub_rn(v1, c.y))));
            *reinterpret_cast<double2 *>(out + idx) = make_double2(v0, v1);
        }
    return dmax;
}

// A unit of side 8 or 16 painted by a half-warp, bit-identical to paint_unit_f64: numpy's pairwise
// mean keeps 8 accumulators over each block of <= 128 elements (accumulator k sums elements 8s + k
// in order), so lane (h, k) -- block h of a side-16 unit, accumulator k -- owns exactly the elements
// one accumulator sums: it forms their downsampled values, sums them in order, and the half-warp
// combines ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)) (then lo + hi for side 16) by xor
// shuffles (fp64 addition is commutative, so every lane gets the same bits).  The lane then paints
// its own elements.  All 16 lanes of the half-warp (mask) must call it.
__device__ double paint_big_f64(int x, int y, int side, int iso, int dx, int dy, double s, double o, int W,
                                const double *cur, double *out, int hl, unsigned mask) {
    const bool big = side == 16;
    const bool on = big || hl < 8;
    const int k = hl & 7, base = big ? 128 * (hl >> 3) : 0, nst = big ? 16 : 8, lg = big ? 4 : 3;
    double d[16];
    double r = 0.0;
    if (on) {
#pragma unroll
        for (int st = 0; st < 16; st++) {
            if (st < nst) {
                const int e = base + 8 * st + k, i = e >> lg, j = e & (side - 1);
                const int kk = iso ? iso_src(iso, i, j, side) : e;
                const double *pp = cur + (size_t)(dy + 2 * (kk >> lg)) * W + dx + 2 * (kk & (side - 1));
                d[st] = __dmul_rn(__dadd_rn(__dadd_rn(__dadd_rn(pp[0], pp[1]), pp[W]), pp[W + 1]), 0.25);
                r = st == 0 ? d[0] : __dadd_rn(r, d[st]);
            }
        }
    }
    const double t1 = __dadd_rn(r, __shfl_xor_sync(mask, r, 1));
    const double t2 = __dadd_rn(t1, __shfl_xor_sync(mask, t1, 2));
    double tot = __dadd_rn(t2, __shfl_xor_sync(mask, t2, 4));
    const double other = __shfl_xor_sync(mask, tot, 8);
    if (big) tot = __dadd_rn(tot, other);
    const double dm = __dmul_rn(tot, big ? 1.0 / 256.0 : 1.0 / 64.0);  // exact: division by a power of two
    double dmax = 0.0;
    if (on) {
#pragma unroll
        for (int st = 0; st < 16; st++) {
            if (st < nst) {
                const int e = base + 8 * st + k, i = e >> lg, j = e & (side - 1);
                double v = __dadd_rn(__dmul_rn(s, __dsub_rn(d[st], dm)), o);
                v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
                const size_t idx = (size_t)(y + i) * W + x + j;
                dmax = fmax(dmax, fabs(__dsub_rn(v, cur[idx])));
                out[idx] = v;
            }
        }
    }
    return dmax;
}

#ifndef F64_MINB
#define F64_MINB 4  // resident CTAs per SM the sweep is compiled for (5 and 6 spill or gain nothing: profiles/r2/README.md)
#endif
constexpr int F64_T = 256;  // threads (unit slots) per CTA of the sweep
constexpr long long F64_COOP_MAX_PX = 1ll << 21;  // decode_f64: images up to this many pixels decode in one launch

// Slot u of a sweep (thread per unit slot; every thread of the warp must call it): paints a unit of
// side 2 / 4 (or an odd side) itself, then the warp's units of side 8 / 16 a half-warp each (BIGSEP:
// those are left to sweep_big_slots).  Returns the thread's max |delta|.
template <bool BIGSEP>
__device__ __forceinline__ double sweep_slot(long long u, const int32_t *ux, const int32_t *uy, const int32_t *usize,
                                             const int32_t *udx, const int32_t *udy, const double *us,
                                             const double *uo, long long n, int W, const double *cur, double *nxt) {
    double dmax = 0.0;
    bool big = false;
    if (u < n && (usize[u] & 255) > 0) {  // usize = side | isometry << 8
        const int side = usize[u] & 255, iso = usize[u] >> 8;
        if (side == 4)
            dmax = paint_unit_f64_fixed<4>(ux[u], uy[u], iso, udx[u], udy[u], us[u], uo[u], W, cur, nxt);
        else if (side == 2)
            dmax = paint_unit_f64_fixed<2>(ux[u], uy[u], iso, udx[u], udy[u], us[u], uo[u], W, cur, nxt);
        else if (side == 8 || side == 16)
            big = !BIGSEP;  // painted below by a half-warp (BIGSEP: by sweep_big_slots)
        else
            dmax = paint_unit_f64(ux[u], uy[u], side, iso, udx[u], udy[u], us[u], uo[u], W, cur, nxt);
    }
    // this warp's units of side 8 / 16, a half-warp each (no CTA barrier: codes without such units
    // pay one ballot)
    unsigned bb = __ballot_sync(FULL, big);
    if (!BIGSEP && bb) {
        const int lane = threadIdx.x & 31, hl = lane & 15, hw = lane >> 4;
        const unsigned mask = 0xFFFFu << (16 * hw);
        const long long w0 = u - lane;
        for (int r = 0; bb; r++) {
            const int b0 = __ffs(bb) - 1;  // round r: half-warp 0 takes the lowest, half-warp 1 the next
            bb &= bb - 1;
            const int b1 = bb ? __ffs(bb) - 1 : -1;
            if (b1 >= 0) bb &= bb - 1;
            const int b = hw ? b1 : b0;
            if (b >= 0) {
                const long long v = w0 + b;
                const int side = usize[v] & 255, iso = usize[v] >> 8;
                dmax = fmax(dmax, paint_big_f64(ux[v], uy[v], side, iso, udx[v], udy[v], us[v], uo[v], W, cur, nxt,
                                                hl, mask));
            }
        }
    }
    return dmax;
}

// The units of side 8 / 16 of slot group g, by one half-warp (lanes hl of `mask`): one record's
// units in records_to_units' layout (slot g, then n/4 + 3g .. + 2) when n is a multiple of 4, else
// slots 4g .. 4g + 3; either way every slot is visited once.
__device__ __forceinline__ double sweep_big_slots(long long g, int hl, unsigned mask, const int32_t *ux,
                                                  const int32_t *uy, const int32_t *usize, const int32_t *udx,
                                                  const int32_t *udy, const double *us, const double *uo, long long n,
                                                  int W, const double *cur, double *nxt) {
    const long long nrec = (n & 3) ? 0 : n >> 2;
    double dmax = 0.0;
#pragma unroll 1
    for (int k = 0; k < 4; k++) {
        const long long v = nrec ? (g < nrec ? (k == 0 ? g : nrec + 3 * g + (k - 1)) : n) : 4 * g + k;
        const int sz = v < n ? usize[v] : 0, side = sz & 255;
        if (side == 8 || side == 16)  // uniform across the half-warp
            dmax = fmax(dmax, paint_big_f64(ux[v], uy[v], side, sz >> 8, udx[v], udy[v], us[v], uo[v], W, cur, nxt,
                                            hl, mask));
    }
    return dmax;
}

// max over the warp of a non-negative fp64 (its bits order as integers), folded into *slot
__device__ __forceinline__ void fold_delta(double dmax, long long *slot) {
    long long bits = __double_as_longlong(dmax);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bits = max(bits, __shfl_xor_sync(FULL, bits, o));
    if ((threadIdx.x & 31) == 0 && bits > 0)
        atomicMax(reinterpret_cast<unsigned long long *>(slot), (unsigned long long)bits);
}

template <bool BIGSEP>
__global__ void __launch_bounds__(F64_T, F64_MINB) sweep_f64_kernel(const int32_t *ux, const int32_t *uy, const int32_t *usize,
                                                          const int32_t *udx, const int32_t *udy, const double *us,
                                                          const double *uo, long long n, int W, const double *cur,
                                                          double *nxt, long long *state) {
    if (state[0]) return;  // converged in an earlier sweep
    const long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    fold_delta(sweep_slot<BIGSEP>(u, ux, uy, usize, udx, udy, us, uo, n, W, cur, nxt), &state[2]);
}

// Codes made mostly of units of side 8 / 16 (e.g. the 8-isometry encodes, whose roots mostly stay
// whole): a half-warp per group of four unit slots -- one record's units in records_to_units'
// layout (slot g, then n/4 + 3g .. + 2) when n is a multiple of 4, else slots 4g .. 4g + 3; either
// way every slot is visited once -- so every big unit gets its own half-warp instead of waiting
// its turn in a warp holding eight.
__global__ void __launch_bounds__(256) sweep_big_f64_kernel(const int32_t *ux, const int32_t *uy,
                                                            const int32_t *usize, const int32_t *udx,
                                                            const int32_t *udy, const double *us, const double *uo,
                                                            long long n, int W, const double *cur, double *nxt,
                                                            long long *state) {
    if (state[0]) return;
    const long long g = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 4;
    const unsigned mask = 0xFFFFu << (16 * ((threadIdx.x >> 4) & 1));
    fold_delta(sweep_big_slots(g, threadIdx.x & 15, mask, ux, uy, usize, udx, udy, us, uo, n, W, cur, nxt), &state[2]);
}

// decoder.py:71-75: current = nxt; stop if delta < stop_delta
__global__ void decide_kernel(long long *state, double stop_delta) {
    if (state[0]) return;
    state[1] += 1;
    if (__longlong_as_double(state[2]) < stop_delta) state[0] = 1;
    state[2] = 0;
}

// decoder.py:76: clip(floor(x + 0.5)) of the raster holding the last sweep (sweep i writes
// buffer (i + 1) % 2), rows [y0, y1) into out (pitch W)
__global__ void finalize_f64_kernel(const double *ping, const double *pong, const long long *state, int W, int y0,
                                    int y1, uint8_t *out, int32_t *iters_done) {
    const double *src = (state[1] & 1) ? pong : ping;
    const long long n = (long long)(y1 - y0) * W, base = (long long)y0 * W;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double v = floor(src[base + i] + 0.5);
        out[i] = (uint8_t)(v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v));
    }
    if (iters_done && blockIdx.x == 0 && threadIdx.x == 0) *iters_done = (int32_t)state[1];
}

__global__ void fill_f64_kernel(double *a, double v, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        a[i] = v;
}

// Small images (c1 / c2): the whole decode -- fill, every sweep with its stop decision, the uint8
// image -- in ONE cooperative launch, a grid barrier per sweep instead of two or three launches
// (a 512^2 sweep is a few microseconds of work; ten sweeps were launch-bound).  Same slot helpers,
// so the same bits.  Sweep `it` folds its max |delta| into state[2 + it % 3]; thread 0 clears the
// next sweep's word before the barrier (its last readers passed the previous barrier), and every
// thread applies decoder.py:71-75 to the word after it, so the whole grid leaves the loop together.
template <bool BIGSEP>
__global__ void __launch_bounds__(F64_T, 2) decode_f64_coop_kernel(
    const int32_t *ux, const int32_t *uy, const int32_t *usize, const int32_t *udx, const int32_t *udy,
    const double *us, const double *uo, long long n, int W, int H, int iters, double stop_delta, double init,
    double *ping, double *pong, long long *state, uint8_t *out, int32_t *iters_done) {
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    const long long gsz = (long long)gridDim.x * blockDim.x, gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long npx = (long long)W * H;
    for (long long i = gt; i < npx; i += gsz) ping[i] = init;
    grid.sync();
    int done = 0;
    for (int it = 0; it < iters; it++) {
        const double *cur = (it & 1) ? pong : ping;
        double *nxt = (it & 1) ? ping : pong;
        double dmax = 0.0;
        for (long long base = blockIdx.x * (long long)blockDim.x; base < n; base += gsz)  // CTA-uniform trip count
            dmax = fmax(dmax, sweep_slot<BIGSEP>(base + threadIdx.x, ux, uy, usize, udx, udy, us, uo, n, W, cur, nxt));
        if (BIGSEP) {
            const unsigned mask = 0xFFFFu << (16 * ((threadIdx.x >> 4) & 1));
            const long long groups = (n + 3) / 4;
            for (long long g = gt >> 4; g < groups; g += gsz >> 4)
                dmax = fmax(dmax, sweep_big_slots(g, threadIdx.x & 15, mask, ux, uy, usize, udx, udy, us, uo, n, W,
                                                  cur, nxt));
        }
        fold_delta(dmax, &state[2 + it % 3]);
        if (gt == 0) state[2 + (it + 1) % 3] = 0;
        grid.sync();
        done = it + 1;
        const long long bits = *reinterpret_cast<volatile long long *>(&state[2 + it % 3]);
        if (__longlong_as_double(bits) < stop_delta) break;
    }
    const double *src = (done & 1) ? pong : ping;  // sweep i writes buffer (i + 1) % 2
    for (long long i = gt; i < npx; i += gsz) {
        const double v = floor(src[i] + 0.5);
        out[i] = (uint8_t)(v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v));
    }
    if (gt == 0) {
        state[0] = 1;
        state[1] = done;
        if (iters_done) *iters_done = done;
    }
}

// Records (include/mns_record.h) -> painted units (decoder.py:48-59), 4 slots per record: slot i
// holds record i's first unit (a phase-1 leaf itself, or quadrant 0 of a phase-2 record), slots
// n + 3i + (k - 1) its quadrants k = 1..3 (size 0 for a phase-1 record: skipped by the sweep).  The
// first n slots are therefore dense -- a sweep warp over them paints 32 units, and the parameter
// arrays of a mostly phase-1 code are read once, not through three empty slots in four.
__global__ void records_to_units_kernel(const uint64_t *rec, long long n, int W, int H, int32_t *ux, int32_t *uy,
                                        int32_t *usize, int32_t *udx, int32_t *udy, double *us, double *uo) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= 4 * n) return;
    const long long i = t >> 2;
    const int k = (int)(t & 3);
    const uint64_t r = rec[i];
    const int x = 2 * (int)(r & 0x7FFF), y = 2 * (int)((r >> 15) & 0x7FFF);
    const int level = (int)((r >> MNS_REC_LEVEL_SHIFT) & 3) + 1;
    const int size = 32 >> level;
    const bool p2 = (r >> 32) & 1;
    const int ob = (int)((r >> 33) & 0xFF);
    int sz, px, py;
    double s, o;
    const long long slot = k == 0 ? i : n + 3 * i + (k - 1);
    if (!p2) {
        if (k) {
            usize[slot] = 0;
            return;
        }
        sz = size | (int)(((r >> MNS_REC_ISO_SHIFT) & 7) << 8);  // side | isometry << 8
        px = x;
        py = y;
        s = -0.875 + 0.25 * (double)((r >> 41) & 7);
        o = (double)ob;
    } else {
        const int h = size / 2;
        int d[3];
        for (int j = 0; j < 3; j++) {
            const int v = (int)((r >> (41 + 6 * j)) & 63);
            d[j] = v >= 32 ? v - 64 : v;
        }
        const int target = k < 3 ? ob + d[k] : ob - (d[0] + d[1] + d[2]);
        const int bit = (int)((r >> (59 + k)) & 1);
        // CONTRAST_SETS (encoder.py:36)
        const double lo[3] = {0.2, 0.4, 0.5}, hi[3] = {0.5, 0.65, 0.9};
        sz = h;
        px = x + (k & 1) * h;
        py = y + (k >> 1) * h;
        s = bit ? hi[level - 1] : lo[level - 1];
        o = (double)target;
    }
    ux[slot] = px;
    uy[slot] = py;
    usize[slot] = sz;
    const int side = sz & 255;
    udx[slot] = clampi(px - side / 2, 0, W - 2 * side);  // co_domain_rect (image.py:174-187)
    udy[slot] = clampi(py - side / 2, 0, H - 2 * side);
    us[slot] = s;
    uo[slot] = o;
}

int sm_count_f64() {
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

int records_to_units(const uint64_t *records, int64_t n, int W, int H, int32_t *ux, int32_t *uy, int32_t *usize,
                     int32_t *udx, int32_t *udy, double *us, double *uo, cudaStream_t st) {
    MNS_CHECK_ARG(n >= 0 && W >= 2 && H >= 2, "bad record count or raster size");
    if (n == 0) return 0;
    records_to_units_kernel<<<(unsigned)((4 * n + 255) / 256), 256, 0, st>>>(records, n, W, H, ux, uy, usize, udx,
                                                                             udy, us, uo);
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

static int f64_sweep(const int32_t *ux, const int32_t *uy, const int32_t *usize, const int32_t *udx,
                     const int32_t *udy, const double *us, const double *uo, int64_t n, int W, const double *cur,
                     double *nxt, int64_t *state, bool bigsep, cudaStream_t st) {
    if (n == 0) return 0;
    const unsigned grid = (unsigned)((n + F64_T - 1) / F64_T);
    long long *stt = reinterpret_cast<long long *>(state);
    if (bigsep) {
        sweep_f64_kernel<true><<<grid, F64_T, 0, st>>>(ux, uy, usize, udx, udy, us, uo, n, W, cur, nxt, stt);
        const long long groups = (n + 3) / 4;
        sweep_big_f64_kernel<<<(unsigned)((groups * 16 + 255) / 256), 256, 0, st>>>(ux, uy, usize, udx, udy, us, uo,
                                                                                    n, W, cur, nxt, stt);
    } else {
        sweep_f64_kernel<false><<<grid, F64_T, 0, st>>>(ux, uy, usize, udx, udy, us, uo, n, W, cur, nxt, stt);
    }
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

int decode_f64_sweep(const int32_t *ux, const int32_t *uy, const int32_t *usize, const int32_t *udx,
                     const int32_t *udy, const double *us, const double *uo, int64_t n, int W, const double *cur,
                     double *nxt, int64_t *state, cudaStream_t st) {
    MNS_CHECK_ARG(n >= 0 && W > 0, "bad unit count or width");
    if (n == 0) return 0;
    return f64_sweep(ux, uy, usize, udx, udy, us, uo, n, W, cur, nxt, state, false, st);
}

int decode_f64_decide(int64_t *state, double stop_delta, cudaStream_t st) {
    decide_kernel<<<1, 1, 0, st>>>(reinterpret_cast<long long *>(state), stop_delta);
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

int decode_f64_finalize(const double *ping, const double *pong, const int64_t *state, int W, int y0, int y1,
                        uint8_t *out, int32_t *iters_done, cudaStream_t st) {
    MNS_CHECK_ARG(W > 0 && 0 <= y0 && y0 <= y1, "bad raster rows");
    finalize_f64_kernel<<<sm_count_f64() * 4, 256, 0, st>>>(ping, pong, reinterpret_cast<const long long *>(state), W,
                                                            y0, y1, out, iters_done);
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

int decode_f64(const int32_t *ux, const int32_t *uy, const int32_t *usize, const int32_t *udx, const int32_t *udy,
               const double *us, const double *uo, int64_t n, int W, int H, int iters, double stop_delta,
               double init, double *ping, double *pong, uint8_t *out, int32_t *d_iters_done, void *workspace,
               int64_t workspace_bytes, cudaStream_t st) {
    MNS_CHECK_ARG(W > 0 && H > 0, "bad raster size");
    MNS_CHECK_ARG(iters >= 1, "max_iters must be >= 1");
    MNS_CHECK_ARG(workspace_bytes >= 32, "workspace too small");
    int64_t *state = reinterpret_cast<int64_t *>(workspace);
    // leaves of 64+ pixels on average (n = 4 unit slots per leaf): units of side 8 / 16 dominate, give each
    // its own half-warp
    const bool bigsep = (long long)W * H >= 16 * (long long)n;
    if (n > 0 && (long long)W * H <= F64_COOP_MAX_PX && workspace_bytes >= 64) {  // one cooperative launch
        static int per_sm[2] = {0, 0}, coop = -1;
        if (coop < 0) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[0], decode_f64_coop_kernel<false>, F64_T, 0);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[1], decode_f64_coop_kernel<true>, F64_T, 0);
        }
        if (coop > 0 && per_sm[bigsep] > 0) {
            const long long slots = (n + F64_T - 1) / F64_T, groups = bigsep ? ((n + 3) / 4 * 16 + F64_T - 1) / F64_T : 0;
            long long grid = slots > groups ? slots : groups;
            const long long cap = (long long)per_sm[bigsep] * sm_count_f64();
            if (grid > cap) grid = cap;
            MNS_CUDA_TRY(cudaMemsetAsync(state, 0, 64, st));
            long long nn = n;
            long long *stt = reinterpret_cast<long long *>(state);
            void *args[] = {&ux, &uy, &usize, &udx, &udy, &us, &uo, &nn, &W, &H, &iters, &stop_delta, &init,
                            &ping, &pong, &stt, &out, &d_iters_done};
            const void *fn = bigsep ? (const void *)decode_f64_coop_kernel<true> : (const void *)decode_f64_coop_kernel<false>;
            MNS_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3((unsigned)grid), dim3(F64_T), args, 0, st));
            return 0;
        }
    }
    MNS_CUDA_TRY(cudaMemsetAsync(state, 0, 32, st));
    fill_f64_kernel<<<sm_count_f64() * 4, 256, 0, st>>>(ping, init, (long long)W * H);
    for (int it = 0; it < iters; it++) {
        const double *cur = (it & 1) ? pong : ping;
        double *nxt = (it & 1) ? ping : pong;
        if (int rc = f64_sweep(ux, uy, usize, udx, udy, us, uo, n, W, cur, nxt, state, bigsep, st)) return rc;
        if (int rc = decode_f64_decide(state, stop_delta, st)) return rc;
    }
    return decode_f64_finalize(ping, pong, state, W, 0, H, out, d_iters_done, st);
}

}  // namespace mns
