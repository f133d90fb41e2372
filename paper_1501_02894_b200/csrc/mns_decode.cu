// Iterative (Jacobi) decoder for sm_100a (K4).
//
// Replaces decoder.py:37-77 (decode_step / decode / _paint) and
// transform.py:63-66 (apply_map).  One launch = one sweep: every painted unit
// reads the previous raster only and writes its own disjoint square of the next
// one, so leaf order is immaterial (decoder.py:8-10, test_decoder.py:27-34).
//
// Quadtree path (mns_decode_quadtree): a CTA owns a TRY x TRX tile of 16x16
// roots.  It stages the fp32 window [tile - 16, tile + 16) of the previous
// raster in shared memory with 16-byte loads (every co-centred domain of every
// unit of its roots lies inside it), decodes each root's packed records into a
// 64-entry Morton-cell table of (s, o, domain, size), and then each lane paints
// the 2x4 pixels it owns: q = 2x2 sum of the domain group, per-unit domain sum by
// segmented warp reductions (pair / 8-lane / 32-lane / in-lane), and
// clip(s*(q/4 - mean) + o, 0, 255) stored with coalesced 16-byte stores.  The
// final sweep writes the rounded uint8 image directly (floor(x+0.5), clip).
//
// Generic path (mns_decode_units): one warp per unit, explicit domains
// (search-baseline BaselinePayload codes, encoder.py:101-107).
//
// Exact path (mns_decode_step_f64): one thread per unit replaying numpy's fp64
// order (pairwise mean), bit-identical to decode_step, for parity evidence.

#include <math.h>

#include <type_traits>

#include "mns_common.cuh"
#include "mns_tma.cuh"

namespace mns {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int BR = 8;                 // roots per column band (128 px)
constexpr int NW = BR / 2;            // warps; each paints two side-by-side roots per root row
constexpr int DT = NW * 32;
constexpr int WINW = BR * 16 + 32;    // 160-px window: band +- 16 px (every clamped domain lies inside)
constexpr int QW = WINW / 2;          // 80 columns of the even 2x2-sum lattice
constexpr int QS = QW + 4;            // padded row stride (rows 2 apart land 8 banks apart)
constexpr int QH = QW / 2;            // lattice rows are stored de-interleaved: even columns, then odd
constexpr int WINWP = WINW + 4;       // t+1 raw-ring row stride (rows 4 apart land 16 banks apart)
constexpr int QR = 32;                // lattice ring rows (24 live + 8 being built)
constexpr int QRP = QR + 3;           // + copies of ring rows 0..2, so a 4-row read never wraps
constexpr int BLK = 16;               // raster rows per TMA block
constexpr int NBUF = 5;               // raw ring: 3 blocks readable by compute + 2 in flight
constexpr int CR = 32;                // root rows walked by one CTA
constexpr int RAW_BYTES = BLK * WINW * 4;

// contrast of a unit-map index (mns_record.h): 0..7 phase-1 codes, 8..13 phase-2 sets
__constant__ float kUnitS[16] = {-0.875f, -0.625f, -0.375f, -0.125f, 0.125f, 0.375f, 0.625f, 0.875f,
                                 0.2f,    0.5f,    0.4f,    0.65f,   0.5f,   0.9f,   0.f,    0.f};

struct SweepParams {
    const uint32_t *unit_map;  // 32 words (64 cells) per root of the rows [rr0, rr1)
    const uint16_t *block_map; // lattice passes: 16 block descriptors per root (mns_record.h)
    int W, H, rw, rr0, rr1, y_lo;
    const float *cur;    // null on the first sweep: the flat start raster (init) is implied
    float init;
    float *nxt;          // virtual-global base; null on a fused final sweep
    uint8_t *out_u8;     // virtual-global base; non-null on the final sweep
    int *state;          // [0] done, [1] sweeps done, [2] finished-CTA counter, [3] max |delta| bits
    int track_delta;
    float stop_delta;
    int n_ctas;
    int umap_r0;         // first root row held by unit_map (pair kernel: may be rr0 - 1)
    int cr;              // root rows walked by one CTA (rows_per_cta)
};

// Root rows per CTA: the kernel's nominal chunk, shortened on small images so the grid still
// covers the SMs (c1/c2 are latency-bound: fewer serial rows per CTA beat the extra halo rows).
static int rows_per_cta(int rows, int bands, int nominal) {
    const int target = 2 * 148;  // two CTAs per SM
    int cr = nominal;
    while (cr > 4 && (long long)bands * ((rows + cr - 1) / cr) < target) cr /= 2;
    return cr;
}

__device__ __forceinline__ int morton_of(int cx, int cy) {  // 3-bit coordinates -> 6-bit Morton (y major)
    int m = 0;
#pragma unroll
    for (int i = 0; i < 3; i++) m |= (((cx >> i) & 1) << (2 * i)) | (((cy >> i) & 1) << (2 * i + 1));
    return m;
}

// Domain offset of a lane's 4x4 block inside a unit of side 2^(k+1) (k = 1..3): the block's
// first domain pixel is (rxg + X - 16, ryg + Y - 16) with X = 2px - ux - side/2 + 16 (ux = px
// rounded down to the unit), i.e. the co-centred domain (encoder.py:139-157) plus twice the
// block's offset inside the unit.  Interior roots never clamp, so the three sizes fit one
// register per coordinate (3 x 6 bits), built once per lane.
__device__ __forceinline__ uint32_t offset_table(int pc) {
    uint32_t t = 0;
#pragma unroll
    for (int k = 1; k <= 3; k++) {
        const int side = 2 << k;
        t |= (uint32_t)(2 * pc - (pc & ~(side - 1)) - side / 2 + 16) << (6 * k);
    }
    return t;
}

// Same offset for roots on the image border: the domain is clamped into the image.
__device__ __forceinline__ int clamped_offset(int pc, int side, int rg, int extent) {
    const int uc = pc & ~(side - 1);
    return clampi(rg + uc - side / 2, 0, extent - 2 * side) - rg + 2 * (pc - uc) + 16;
}

__device__ __forceinline__ float unit_o(uint32_t d) { return (float)((int)((d >> 4) & 1023) - 32); }

// Where a lane paints: the Morton-aligned 4x4 block l = lane & 15 of a root; any unit of side
// >= 4 covers the whole block (units are aligned to their side), so one 64-bit unit-map load
// (cells 4l..4l+3), one unit decode and 16 lattice loads serve 16 pixels; only 2x2 units
// (odd domains) sum raster pixels directly.
struct Lane {
    int lx, ly;        // block offset in the root
    uint32_t tx, ty;   // offset_table(lx), offset_table(ly)
};

__device__ __forceinline__ Lane lane_of(int lane) {
    Lane L;
    const int l = lane & 15;
    L.lx = 4 * (l & 1) + 8 * ((l >> 2) & 1);
    L.ly = 4 * ((l >> 1) & 1) + 8 * ((l >> 3) & 1);
    L.tx = offset_table(L.lx);
    L.ty = offset_table(L.ly);
    return L;
}

// Lattice rows are de-interleaved (column c at (c & 1) * HALF + c / 2): the 4 columns a lane
// reads come from two base pointers with immediate offsets, and the lanes of a warp, whose
// columns all share one parity, spread over all 32 banks.  Store the pair of columns (c, c+1),
// c even, at ring row r (mod QR) and, for ring rows 0..2, at their padded copies.
template <int QSTR, int HALF>
__device__ __forceinline__ void lat_store(float *lat, int r, int c, float2 val) {
    const int rr = r & (QR - 1);
    float *row = lat + rr * QSTR + (c >> 1);
    row[0] = val.x;
    row[HALF] = val.y;
    if (rr < QRP - QR) {
        row[QR * QSTR] = val.x;
        row[QR * QSTR + HALF] = val.y;
    }
}

// Packed fp32 pairs (sm_100 FFMA2 / FADD2): same per-lane IEEE rounding as fmaf / fadd.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}

__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}

// v[16] = clip(s * (q - mean) + o) of the lane's 4x4 block of root (rxg, ryg) (decoder.py:32-34,
// transform.py:63-66).  Domain sums q come from the even 2x2-sum lattice ring `lat` (row =
// absolute raster row / 2 mod QR, column = window column / 2, window origin wx0) or, for 2x2
// units, from raw_sum(R, C) = the 2x2 raster sum at absolute row R, window column C.  Every
// lane of the warp must call it (segmented shuffles); `live` lanes get v.
// Lattice addressing of an interior lane, per unit size k = 1..3, fixed for a kernel: the column
// offsets of its two de-interleaved base pointers (8 bits each) and the lattice-row offset of its
// domain from 8 * (root row) + 8 (5 bits) -- so a paint needs no per-block coordinate arithmetic.
struct LaneTab {
    uint32_t t[3];
};

template <int QSTR, int HALF>
__device__ __forceinline__ LaneTab lane_tab(const Lane &L, int rc, int col_base) {
    LaneTab T;
#pragma unroll
    for (int k = 1; k <= 3; k++) {
        const int dx = (int)((L.tx >> (6 * k)) & 63) / 2 - 8, dy = (int)((L.ty >> (6 * k)) & 63) / 2 - 8;
        const int qc = 8 * rc + col_base + dx;  // window lattice column of the domain's first column
        const uint32_t c0 = (qc & 1) * HALF + (qc >> 1), c1 = ((qc + 1) & 1) * HALF + ((qc + 1) >> 1);
        T.t[k - 1] = c0 | (c1 << 8) | ((uint32_t)(dy + 8) << 16);
    }
    return T;
}

template <int QSTR, int HALF, int RING = QR, bool RAW = true, bool FAST = false, class RawSum>
__device__ __forceinline__ void paint_block(uint2 word, bool live, const Lane &L, const float *st, const float *lat,
                                            const RawSum &raw_sum, bool flat, float init, int rxg, int ryg, int wx0,
                                            bool interior, int W, int H, float (&v)[16],
                                            const LaneTab *tab = nullptr) {
    if (flat) {
        // Flat start raster (kernel-uniform): every domain mean is init exactly (sums of equal
        // power-of-two multiples of init are exact), so each unit paints the constant
        // clip(fl(s/4 * 4 init + fl(o - s init))) -- the generic path's value, without its loads,
        // sums and shuffles.
        if (live) {
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const uint32_t d = c == 0 ? word.x & 0xFFFFu
                                          : (c == 1 ? word.x >> 16 : (c == 2 ? word.y & 0xFFFFu : word.y >> 16));
                const float sc = st[d & 15];
                const float x = fminf(255.f, fmaxf(0.f, fmaf(0.25f * sc, 4.f * init, fmaf(-sc, init, unit_o(d)))));
#pragma unroll
                for (int i = 0; i < 2; i++)
#pragma unroll
                    for (int jj = 0; jj < 2; jj++) v[4 * (2 * (c >> 1) + i) + 2 * (c & 1) + jj] = x;
            }
        }
        return;
    }
    const uint32_t d0 = word.x & 0xFFFFu;
    // Lattice passes (FAST): every lane paints -- dead lanes and the flagged 2x2 units through the
    // in-ring table addresses, results discarded (liveness is per root, so no dead sum reaches a
    // live unit) -- which keeps the paint free of divergent branches.
    const int k = FAST ? max(1, (int)(d0 >> 14)) : (int)(d0 >> 14);  // log2(side) - 1 of cell 0's unit
    const bool go = FAST || (live && k > 0);
    const bool use_tab = FAST && (interior || !live);
    float own = 0.f, sa = 0.f, sb = 0.f;
    if (go) {  // one unit of side >= 4 covers the 4x4 block
        sa = st[d0 & 15];
        sb = unit_o(d0);
        {
            const float *p0, *p1;  // columns qc, qc + 2 and qc + 1, qc + 3 of the domain's first lattice row
            if (use_tab) {
                const uint32_t t = k == 1 ? tab->t[0] : (k == 2 ? tab->t[1] : tab->t[2]);
                const float *row = lat + ((ryg >> 1) + (int)(t >> 16) - 8 & (RING - 1)) * QSTR;
                p0 = row + (t & 255);
                p1 = row + ((t >> 8) & 255);
            } else {
                int X, Y;
                if (interior) {
                    X = (int)((L.tx >> (6 * k)) & 63);
                    Y = (int)((L.ty >> (6 * k)) & 63);
                } else {
                    X = clamped_offset(L.lx, 2 << k, rxg, W);
                    Y = clamped_offset(L.ly, 2 << k, ryg, H);
                }
                const int qr = (ryg - 16 + Y) >> 1, qc = (rxg - 16 + X - wx0) >> 1;
                const float *row = lat + (qr & (RING - 1)) * QSTR;  // rows +0..+3 stay inside the padded ring
                p0 = row + (qc & 1) * HALF + (qc >> 1);
                p1 = row + ((qc + 1) & 1) * HALF + ((qc + 1) >> 1);
            }
#pragma unroll
            for (int i = 0; i < 4; i++) {
                v[4 * i + 0] = p0[i * QSTR];
                v[4 * i + 1] = p1[i * QSTR];
                v[4 * i + 2] = p0[i * QSTR + 1];
                v[4 * i + 3] = p1[i * QSTR + 1];
            }
        }
        const float2 p0 = fadd2(make_float2(v[0], v[1]), make_float2(v[2], v[3]));
        const float2 p1 = fadd2(make_float2(v[4], v[5]), make_float2(v[6], v[7]));
        const float2 p2 = fadd2(make_float2(v[8], v[9]), make_float2(v[10], v[11]));
        const float2 p3 = fadd2(make_float2(v[12], v[13]), make_float2(v[14], v[15]));
        const float2 pp = fadd2(fadd2(p0, p1), fadd2(p2, p3));
        own = pp.x + pp.y;
    } else if (RAW && live) {  // four 2x2 units with odd (or clamped) 4x4 domains
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const uint32_t d = c == 0 ? d0 : (c == 1 ? word.x >> 16 : (c == 2 ? word.y & 0xFFFFu : word.y >> 16));
            const int px = L.lx + 2 * (c & 1), py = L.ly + 2 * (c >> 1);
            float q[4];
            {
                const int dx = clampi(rxg + px - 1, 0, W - 4), dy = clampi(ryg + py - 1, 0, H - 4);
#pragma unroll
                for (int i = 0; i < 2; i++)
#pragma unroll
                    for (int jj = 0; jj < 2; jj++) q[2 * i + jj] = raw_sum(dy + 2 * i, dx - wx0 + 2 * jj);
            }
            const float s = st[d & 15];
            const float b = fmaf(-s, ((q[0] + q[1]) + (q[2] + q[3])) * 0.0625f, unit_o(d));
#pragma unroll
            for (int i = 0; i < 2; i++)
#pragma unroll
                for (int jj = 0; jj < 2; jj++)
                    v[4 * (2 * (c >> 1) + i) + 2 * (c & 1) + jj] =
                        fminf(255.f, fmaxf(0.f, fmaf(0.25f * s, q[2 * i + jj], b)));
        }
    }
    // unit sums: 4x4 = own block, 8x8 = 4 lanes (lane bits 0,1), 16x16 = the root's 16 lanes; two
    // shuffle rounds of three independent butterflies (every lane of a group adds the same pair
    // sums, so the group's sum is bit-identical on all its lanes)
    // (skipped when no lane of the warp holds a unit larger than its own 4x4 block)
    float s8 = own, s16 = own;
    if (__any_sync(FULL, go && k > 1)) {
        const float t1 = __shfl_xor_sync(FULL, own, 1), t2 = __shfl_xor_sync(FULL, own, 2),
                    t3 = __shfl_xor_sync(FULL, own, 3);
        s8 = (own + t1) + (t2 + t3);
        const float u1 = __shfl_xor_sync(FULL, s8, 4), u2 = __shfl_xor_sync(FULL, s8, 8),
                    u3 = __shfl_xor_sync(FULL, s8, 12);
        s16 = (s8 + u1) + (u2 + u3);
    }
    if (go) {
        const float sum = k == 1 ? own : (k == 2 ? s8 : s16);
        const float mean = sum * __int_as_float((127 - 4 - 2 * k) << 23);  // sum * 0.25 / side^2
        const float b = fmaf(-sa, mean, sb), a = 0.25f * sa;
        const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
#pragma unroll
        for (int m = 0; m < 8; m++) {
            const float2 r = ffma2(make_float2(v[2 * m], v[2 * m + 1]), a2, b2);
            v[2 * m] = r.x;
            v[2 * m + 1] = r.y;
        }
        // clip(v) = max(min(bits, bits(255)), 0) on the fp32 bit patterns: one VIMNMX.RELU per pixel
        // (non-negative floats order as their bits, negative ones are negative ints), identical to
        // fminf(255, fmaxf(0, v)) up to the sign of a zero.  Unconditional: cheaper than testing
        // whether the unit's map can leave [0, 255] and branching on it.
#pragma unroll
        for (int e = 0; e < 16; e++) v[e] = __int_as_float(__vimin_s32_relu(__float_as_int(v[e]), 0x437F0000));
    }
}

// fp32 -> rounded uint8 rows of a 4x4 block (floor(x + 0.5); x is already clipped to [0, 255])
__device__ __forceinline__ void store_block(const float (&v)[16], float *nxt, uint8_t *out, int W, int gx, int gy) {
    if (nxt) {
        float *d = nxt + (ptrdiff_t)gy * W + gx;
#pragma unroll
        for (int i = 0; i < 4; i++, d += W)
            *reinterpret_cast<float4 *>(d) = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    }
    if (out) {
        uint8_t *d = out + (ptrdiff_t)gy * W + gx;
#pragma unroll
        for (int i = 0; i < 4; i++, d += W) {
            uint32_t w = 0;
#pragma unroll
            for (int jj = 0; jj < 4; jj++) w |= (uint32_t)floorf(v[4 * i + jj] + 0.5f) << (8 * jj);
            *reinterpret_cast<uint32_t *>(d) = w;
        }
    }
}

// One Jacobi sweep (decoder.py:37-63) for a 128-px column band over p.cr root rows.
// TMA streams 16-row raster blocks (OOB zero fill) into a 5-deep smem ring, two blocks
// ahead of the root row being painted; each block is reduced once into the even 2x2-sum
// lattice ring (numpy's downsample_mean2 order, image.py), so no raster row is reloaded
// vertically.  Warp w paints roots 2w, 2w+1 of the band (paint_block).  The unit-map
// words of the next root row are prefetched into registers one step ahead.
__global__ void __launch_bounds__(DT) decode_sweep_kernel(const __grid_constant__ CUtensorMap tmap,
                                                          const SweepParams p) {
    extern __shared__ __align__(128) unsigned char dsm[];
    float(*raw)[BLK][WINW] = reinterpret_cast<float(*)[BLK][WINW]>(dsm);
    float(*qe)[QS] = reinterpret_cast<float(*)[QS]>(dsm + NBUF * RAW_BYTES);
    __shared__ __align__(8) uint64_t bars[NBUF];
    __shared__ float cta_max;
    __shared__ float st[16];

    if (p.state[0]) return;  // converged in an earlier sweep (stop_delta > 0)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int x0 = blockIdx.x * BR * 16, wx0 = x0 - 16;
    const int r_s = p.rr0 + blockIdx.y * p.cr, r_e = min(r_s + p.cr, p.rr1);
    const bool flat = p.cur == nullptr;
    const int nblocks = (r_e - r_s) + 2;  // block k = raster rows [16(r_s-1+k), 16(r_s+k))
    if (tid < 16) st[tid] = kUnitS[tid];
    if (tid == 0) {
        for (int b = 0; b < NBUF; b++) mbar_init(&bars[b], 1);
        fence_mbar_init();
        cta_max = 0.f;
    }
    __syncthreads();
    auto issue = [&](int k) {
        if (k < nblocks) {
            const int b = k % NBUF;
            mbar_arrive_expect_tx(&bars[b], RAW_BYTES);
            tma_load_2d(raw[b], &tmap, wx0, 16 * (r_s - 1 + k) - p.y_lo, &bars[b]);
        }
    };
    // this thread's lattice-build elements (the same for every block): e = tid + i * DT
    constexpr int NE = 8 * (WINW / 4), NPT = (NE + DT - 1) / DT;
    int b_raw[NPT], b_row[NPT], b_col[NPT];
#pragma unroll
    for (int i = 0; i < NPT; i++) {
        const int e = tid + i * DT, r = e / (WINW / 4), c4 = e % (WINW / 4);
        b_raw[i] = 2 * r * WINW + 4 * c4;
        b_row[i] = r;
        b_col[i] = 2 * c4;
    }
    const uint32_t bar0 = smem_u32(&bars[0]);
    auto build = [&](int k) {  // lattice rows [8(r_s-1+k), 8(r_s+k)) from block k
        const int b = k % NBUF;
        mbar_wait_addr(bar0 + 8 * b, (k / NBUF) & 1);
        const int g0 = 8 * (r_s - 1 + k);
        const float *rb = &raw[b][0][0];
#pragma unroll
        for (int i = 0; i < NPT; i++) {
            if (i + 1 < NPT || tid + i * DT < NE) {
                const float4 u = *reinterpret_cast<const float4 *>(rb + b_raw[i]);
                const float4 w = *reinterpret_cast<const float4 *>(rb + b_raw[i] + WINW);
                // numpy order of downsample_mean2 up to the 0.25 scale: ((a + b) + c) + d
                lat_store<QS, QH>(&qe[0][0], g0 + b_row[i], b_col[i],
                              make_float2(((u.x + u.y) + w.x) + w.y, ((u.z + u.w) + w.z) + w.w));
            }
        }
    };
    if (!flat) {
        if (tid == 0) {
            prefetch_tmap(&tmap);
            for (int k = 0; k < 4; k++) issue(k);
        }
        build(0);
        build(1);
    }
    auto raw_sum = [&](int R, int C) {  // 2x2 raster sum at absolute row R, window column C
        const int k0 = R / BLK - (r_s - 1), k1 = (R + 1) / BLK - (r_s - 1);
        const float *r0 = raw[k0 % NBUF][R % BLK];
        const float *r1 = raw[k1 % NBUF][(R + 1) % BLK];
        return ((r0[C] + r0[C + 1]) + r1[C]) + r1[C + 1];
    };

    const Lane L = lane_of(lane);
    const int rc = 2 * warp + (lane >> 4);  // root column in the band
    const int rxi = blockIdx.x * BR + rc;
    const bool live_col = rxi < p.rw;
    const uint2 *umap = reinterpret_cast<const uint2 *>(p.unit_map + (size_t)((r_s - p.rr0) * p.rw + rxi) * 32) +
                        (lane & 15);
    const size_t ustride = (size_t)p.rw * 16;
    uint2 word = live_col ? __ldg(umap) : make_uint2(0u, 0u);
    const bool interior_col = rxi >= 1 && rxi + 1 < p.rw;
    const int rh = p.H / 16;
    float lmax = 0.f;
    for (int j = 0; j < r_e - r_s; j++) {
        umap += ustride;
        const uint2 wnext = (live_col && j + 1 < r_e - r_s) ? __ldg(umap) : make_uint2(0u, 0u);
        if (!flat) build(j + 2);
        __syncthreads();
        if (!flat && tid == 0) {
            fence_proxy_async();  // generic reads of block j-1 complete before the async refill
            issue(j + 4);
        }
        const int ry = r_s + j;
        const int rxg = rxi * 16, ryg = ry * 16;
        float v[16];
        paint_block<QS, QH>(word, live_col, L, st, &qe[0][0], raw_sum, flat, p.init, rxg, ryg, wx0,
                        interior_col && ry >= 1 && ry + 1 < rh, p.W, p.H, v);
        word = wnext;
        if (!live_col) continue;
        if (p.track_delta) {
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const float *old = flat ? nullptr : raw[(j + 1) % NBUF][L.ly + i];
#pragma unroll
                for (int jj = 0; jj < 4; jj++)
                    lmax = fmaxf(lmax, fabsf(v[4 * i + jj] - (flat ? p.init : old[16 + 16 * rc + L.lx + jj])));
            }
        }
        store_block(v, p.nxt, p.out_u8, p.W, rxg + L.lx, ryg + L.ly);
    }
    if (p.track_delta) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(FULL, lmax, o));
        if (lane == 0) atomicMax(reinterpret_cast<int *>(&cta_max), __float_as_int(lmax));
        __syncthreads();
        if (tid == 0) {
            atomicMax(&p.state[3], __float_as_int(cta_max));
            __threadfence();
            const int done = atomicAdd(&p.state[2], 1);
            if (done == p.n_ctas - 1) {  // last CTA of this sweep decides the early stop
                __threadfence();
                const float delta = __int_as_float(atomicAdd(&p.state[3], 0));
                p.state[1] += 1;
                if (delta < p.stop_delta) p.state[0] = 1;
                p.state[2] = 0;
                p.state[3] = 0;
            }
        }
    }
}

// ------------------------------------------------------------- two sweeps per pass
// Sweeps t -> t+1 -> t+2 in one pass over HBM (no early stop): raster t is read once and
// t+2 written once; t+1 never leaves shared memory.  Stage A (NWA warps) paints t+1 for the
// band plus one root on each side (its domains reach 16 px out) into a 4-deep raw ring and
// straight into the t+1 lattice ring (the 2x2 sums of a lane's own 4x4 block, numpy order);
// stage B (NW warps) paints t+2 of the band two root rows behind, from those rings.  Raster t
// streams through a 3-deep TMA ring (one block being reduced into the t lattice, two in
// flight); stage A's rare 2x2 units read raster t through L2.  Rows: A recomputes one root
// row above and below the CTA's CR2 rows; resident halo 32 rows (mns_decode_sweep2).
constexpr int WA = BR * 16 + 64;      // 192-px window of raster t: band +- 32 px
constexpr int QSA = WA / 2 + 4;       // t-lattice row stride (100: rows 2 apart 8 banks apart)
#ifndef PAIR_NT
#define PAIR_NT 3
#endif
#ifndef PAIR_CR2
#define PAIR_CR2 64
#endif
constexpr int NT = PAIR_NT;           // raster-t ring
constexpr int NM = 4;                 // t+1 raw ring (B reads rows i-3..i-1 while A writes i)
constexpr int CR2 = PAIR_CR2;         // root rows per CTA
constexpr int NWA = (BR + 2) / 2;     // stage-A warps (two roots each)
constexpr int DT2 = (NWA + NW) * 32;
constexpr int TRAW_BYTES = BLK * WA * 4;
constexpr int MRAW_BYTES = BLK * WINWP * 4;
constexpr int PAIR_SMEM = NT * TRAW_BYTES + NM * MRAW_BYTES + QRP * QSA * 4 + QRP * QS * 4;

__global__ void __launch_bounds__(DT2, 2) decode_pair_kernel(const __grid_constant__ CUtensorMap tmap,
                                                             const SweepParams p) {
    extern __shared__ __align__(128) unsigned char dsm[];
    float(*traw)[BLK][WA] = reinterpret_cast<float(*)[BLK][WA]>(dsm);
    float(*mraw)[BLK][WINWP] = reinterpret_cast<float(*)[BLK][WINWP]>(dsm + NT * TRAW_BYTES);
    float(*qa)[QSA] = reinterpret_cast<float(*)[QSA]>(dsm + NT * TRAW_BYTES + NM * MRAW_BYTES);
    float(*qb)[QS] = reinterpret_cast<float(*)[QS]>(dsm + NT * TRAW_BYTES + NM * MRAW_BYTES + QRP * QSA * 4);
    __shared__ __align__(8) uint64_t bars[NT];
    __shared__ float st[16];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int x0 = blockIdx.x * BR * 16, xa0 = x0 - 32, xb0 = x0 - 16;
    const int r_s = p.rr0 + blockIdx.y * p.cr, r_e = min(r_s + p.cr, p.rr1);
    const int rh = p.H / 16;
    const bool flat = p.cur == nullptr;
    const int nblocks = (r_e - r_s) + 4;  // block k = raster-t root row r_s - 2 + k
    if (tid < 16) st[tid] = kUnitS[tid];
    if (tid == 0) {
        for (int b = 0; b < NT; b++) mbar_init(&bars[b], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int k) {
        if (k < nblocks) {
            const int b = k % NT;
            mbar_arrive_expect_tx(&bars[b], TRAW_BYTES);
            tma_load_2d(traw[b], &tmap, xa0, 16 * (r_s - 2 + k) - p.y_lo, &bars[b]);
        }
    };
    constexpr int NE = 8 * (WA / 4), NPT = (NE + DT2 - 1) / DT2;
    int b_raw[NPT], b_row[NPT], b_col[NPT];
#pragma unroll
    for (int i = 0; i < NPT; i++) {
        const int e = tid + i * DT2, r = e / (WA / 4), c4 = e % (WA / 4);
        b_raw[i] = 2 * r * WA + 4 * c4;
        b_row[i] = r;
        b_col[i] = 2 * c4;
    }
    const uint32_t bar0 = smem_u32(&bars[0]);
    auto build = [&](int k) {  // t-lattice rows of root row r_s - 2 + k
        const int b = k % NT;
        mbar_wait_addr(bar0 + 8 * b, (k / NT) & 1);
        const int g0 = 8 * (r_s - 2 + k);
        const float *rb = &traw[b][0][0];
#pragma unroll
        for (int i = 0; i < NPT; i++) {
            if (i + 1 < NPT || tid + i * DT2 < NE) {
                const float4 u = *reinterpret_cast<const float4 *>(rb + b_raw[i]);
                const float4 w = *reinterpret_cast<const float4 *>(rb + b_raw[i] + WA);
                lat_store<QSA, WA / 4>(&qa[0][0], g0 + b_row[i], b_col[i],
                               make_float2(((u.x + u.y) + w.x) + w.y, ((u.z + u.w) + w.z) + w.w));
            }
        }
    };
    if (!flat) {
        if (tid == 0) {
            prefetch_tmap(&tmap);
            for (int k = 0; k < NT; k++) issue(k);
        }
        build(0);
        build(1);
        __syncthreads();
        if (tid == 0) {
            fence_proxy_async();
            issue(NT);
            issue(NT + 1);
        }
    }

    const Lane L = lane_of(lane);
    const bool stage_a = warp < NWA;
    // stage A: root columns -1 .. BR of the band; stage B: 0 .. BR-1
    const int rc = stage_a ? 2 * warp + (lane >> 4) - 1 : 2 * (warp - NWA) + (lane >> 4);
    const int rxi = blockIdx.x * BR + rc;
    const bool col_ok = rxi >= 0 && rxi < p.rw;
    const bool interior_col = rxi >= 1 && rxi + 1 < p.rw;
    const int lag = stage_a ? 0 : 2;  // iteration i: A paints root row i, B paints i - 2
    const int row_lo = stage_a ? max(r_s - 1, 0) : r_s, row_hi = stage_a ? min(r_e + 1, rh) : r_e;
    const uint2 *ubase = reinterpret_cast<const uint2 *>(p.unit_map) + ((ptrdiff_t)rxi - (ptrdiff_t)p.umap_r0 * p.rw) * 16 +
                         (lane & 15);
    const ptrdiff_t ustride = (ptrdiff_t)p.rw * 16;
    auto word_of = [&](int row, const uint2 *ptr) {
        return col_ok && row >= row_lo && row < row_hi ? __ldg(ptr) : make_uint2(0u, 0u);
    };
    auto raw_t = [&](int R, int C) {  // raster t through L2 (window origin xa0)
        const float *r0 = p.cur + (ptrdiff_t)R * p.W + xa0 + C;
        const float *r1 = r0 + p.W;
        return ((__ldg(r0) + __ldg(r0 + 1)) + __ldg(r1)) + __ldg(r1 + 1);
    };
    auto raw_m = [&](int R, int C) {  // raster t+1 from the smem ring (window origin xb0)
        const float *r0 = mraw[(R >> 4) & (NM - 1)][R & 15];
        const float *r1 = mraw[((R + 1) >> 4) & (NM - 1)][(R + 1) & 15];
        return ((r0[C] + r0[C + 1]) + r1[C]) + r1[C + 1];
    };
    const uint2 *uptr = ubase + (ptrdiff_t)(r_s - 1 - lag) * ustride;
    uint2 word = word_of(r_s - 1 - lag, uptr);
    for (int i = r_s - 1; i <= r_e + 1; i++) {
        const int row = i - lag;
        uptr += ustride;
        const uint2 wnext = word_of(row + 1, uptr);
        const int k = i - r_s + 3;
        if (!flat && k < nblocks) build(k);
        __syncthreads();
        if (!flat && tid == 0) {
            fence_proxy_async();  // generic reads of the block just reduced complete before its refill
            issue(k + NT);
        }
        const int rxg = rxi * 16, ryg = row * 16;
        const bool interior = interior_col && row >= 1 && row + 1 < rh;
        float v[16];
        if (stage_a) {
            const bool live = col_ok && row >= 0 && row < rh && row <= r_e;
            paint_block<QSA, WA / 4>(word, live, L, st, &qa[0][0], raw_t, flat, p.init, rxg, ryg, xa0, interior, p.W, p.H,
                             v);
            if (live) {
                const int wc = 16 * (rc + 1) + L.lx;  // window column in t+1 (origin xb0)
                float *m = &mraw[row & (NM - 1)][L.ly][wc];
#pragma unroll
                for (int r = 0; r < 4; r++)
                    *reinterpret_cast<float4 *>(m + r * WINWP) =
                        make_float4(v[4 * r], v[4 * r + 1], v[4 * r + 2], v[4 * r + 3]);
                const int g = (ryg + L.ly) >> 1;
#pragma unroll
                for (int r = 0; r < 2; r++)
                    lat_store<QS, QH>(&qb[0][0], g + r, wc >> 1,
                                  make_float2(((v[8 * r] + v[8 * r + 1]) + v[8 * r + 4]) + v[8 * r + 5],
                                              ((v[8 * r + 2] + v[8 * r + 3]) + v[8 * r + 6]) + v[8 * r + 7]));
            }
        } else {
            const bool live = col_ok && row >= r_s;
            paint_block<QS, QH>(word, live, L, st, &qb[0][0], raw_m, false, p.init, rxg, ryg, xb0, interior, p.W, p.H,
                            v);
            if (live) store_block(v, p.nxt, p.out_u8, p.W, rxg + L.lx, ryg + L.ly);
        }
        word = wnext;
    }
}

// ---------------------------------------------------------------- lattice-state passes
// A code without 2x2 units (every unit side >= 4, e.g. the 16->8->4 quadtree with e3 = inf) reads
// the previous raster only through its even 2x2-sum lattice (downsample_mean2's order), so the
// state carried between passes can be that lattice: a quarter of the raster's bytes, bit-identical
// values.  Global layout: (H/2) rows of W/2 floats, each row de-interleaved (the W/4 even lattice
// columns, then the W/4 odd ones) -- the layout paint_block reads, so TMA lands 8-row blocks of it
// straight in the stage-A ring (a 3D box: 52 columns x {even, odd} x 8 rows; the 4 extra columns
// keep the box row a 16-byte multiple and pad the ring row to 104 floats).  Stage A paints t+1
// into the on-chip lattice qb, stage B paints t+2 and stores its lattice (or, on the last pass, the
// uint8 image).  No raster reduction, no t+1 raw ring: ~35 KB of shared memory instead of 105 KB.
#ifndef LAT_BR
#define LAT_BR 8
#endif
constexpr int LBR = LAT_BR;               // roots per column band
constexpr int LNWA = (LBR + 2) / 2;       // stage-A warps (the band +- 1 root, two roots each)
constexpr int LNWB = LBR / 2;             // stage-B warps
constexpr int LDT = (LNWA + LNWB) * 32;
constexpr int LWA = LBR * 16 + 64;        // raster-t window: band +- 32 px
constexpr int LHB = LWA / 4 + 4;          // staged lattice columns per parity (+4: 16-byte box rows)
constexpr int LQS = 2 * LHB;              // ring row: even half | odd half
constexpr int LQR = 64;                   // t-lattice ring rows: 8 root-row slots (up to 5 in flight)
constexpr int LNS = LQR / 8;
constexpr int LQRP = LQR + 8;             // + a second copy of slot 0, so a 4-row read never wraps
constexpr int LBOX = 8 * LQS * 4;         // bytes of one slot
constexpr int LQBW = (LBR * 16 + 32) / 2; // t+1 lattice columns (band +- 16 px)
constexpr int LQBS = LQBW + 4;            // padded row stride
constexpr int LQBH = LQBW / 2;            // de-interleave half
constexpr int LAT_SMEM = LQRP * LQS * 4 + QRP * LQBS * 4;
#ifndef LAT_MINB
#define LAT_MINB (LBR == 8 ? 4 : 2)
#endif
// lane_tab packs column offsets into 8 bits (A: rc <= LBR, B: rc <= LBR - 1, |dx| <= 8)
static_assert(LHB + (8 * LBR + 16 + 8 + 1) / 2 < 256 && LQBH + (8 * LBR + 8 + 1) / 2 < 256,
              "lane_tab column offsets exceed 8 bits");

template <bool FLAT, bool OUT>
__global__ void __launch_bounds__(LDT, LAT_MINB) decode_pair_lat_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                        const SweepParams p) {
    extern __shared__ __align__(128) unsigned char dsm[];
    float(*qa)[LQS] = reinterpret_cast<float(*)[LQS]>(dsm);
    float(*qb)[LQBS] = reinterpret_cast<float(*)[LQBS]>(dsm + LQRP * LQS * 4);
    __shared__ __align__(8) uint64_t bars[LNS];
    __shared__ float st[16];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int x0 = blockIdx.x * LBR * 16, xa0 = x0 - 32, xb0 = x0 - 16;
    const int r_s = p.rr0 + blockIdx.y * p.cr, r_e = min(r_s + p.cr, p.rr1);
    const int rh = p.H / 16, lw = p.W / 2;
    const int nblocks = (r_e - r_s) + 4;  // block k = the 8 lattice rows of root row r_s - 2 + k
    if (tid < 16) st[tid] = kUnitS[tid];
    if (tid == 0) {
        for (int b = 0; b < LNS; b++) mbar_init(&bars[b], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int k) {
        if (k < nblocks) {
            const int row = r_s - 2 + k, slot = row & (LNS - 1), z = 8 * row - p.y_lo / 2;
            mbar_arrive_expect_tx(&bars[slot], slot == 0 ? 2 * LBOX : LBOX);
            tma_load_3d(&qa[8 * slot][0], &tmap, x0 / 4 - 8, 0, z, &bars[slot]);
            if (slot == 0) tma_load_3d(&qa[LQR][0], &tmap, x0 / 4 - 8, 0, z, &bars[0]);
        }
    };
    const uint32_t bar0 = smem_u32(&bars[0]);
    // block k is its slot's (k / LNS)-th fill: blocks are issued in order, one slot per block
    auto wait_block = [&](int k) {
        if (k < nblocks) mbar_wait_addr(bar0 + 8 * ((r_s - 2 + k) & (LNS - 1)), (k / LNS) & 1);
    };
    const Lane L = lane_of(lane);
    const bool stage_a = warp < LNWA;
    if (!FLAT) {
        if (tid == 0) {
            prefetch_tmap(&tmap);
            for (int k = 0; k < LNS; k++) issue(k);
        }
        if (stage_a) {
            wait_block(0);
            wait_block(1);
        }
    }
    auto no_raw = [](int, int) { return 0.f; };
    // One loop per stage (warp-uniform roles; the same iteration count, one barrier per iteration).
    // Iteration i: A paints root row i of t+1 (root columns -1 .. LBR of the band), B paints root
    // row i - 2 of t+2 (columns 0 .. LBR-1).
    auto run = [&](auto role) {
        constexpr bool A = decltype(role)::value;
        const int rc = A ? 2 * warp + (lane >> 4) - 1 : 2 * (warp - LNWA) + (lane >> 4);
        const int rxi = blockIdx.x * LBR + rc;
        const bool col_ok = rxi >= 0 && rxi < p.rw;
        const bool interior_col = rxi >= 1 && rxi + 1 < p.rw;
        constexpr int lag = A ? 0 : 2;
        const int row_lo = A ? max(r_s - 1, 0) : r_s, row_hi = A ? min(r_e + 1, rh) : r_e;
        // the block map: one descriptor per lane (its 4x4 block), replicated into the four cell
        // slots paint_block reads
        const uint16_t *uptr = p.block_map + ((ptrdiff_t)rxi - (ptrdiff_t)p.umap_r0 * p.rw) * 16 + (lane & 15) +
                               (ptrdiff_t)(r_s - 1 - lag) * p.rw * 16;
        const ptrdiff_t ustride = (ptrdiff_t)p.rw * 16;
        auto word_of = [&](int row, const uint16_t *ptr) {
            const uint32_t d = col_ok && row >= row_lo && row < row_hi ? (uint32_t)__ldg(ptr) : 0u;
            return make_uint2(d | (d << 16), d | (d << 16));
        };
        const int rxg = rxi * 16;
        const LaneTab tab = A ? lane_tab<LQS, LHB>(L, rc, 16) : lane_tab<LQBS, LQBH>(L, rc, 8);
        uint2 word = word_of(r_s - 1 - lag, uptr);
        for (int i = r_s - 1; i <= r_e + 1; i++) {
            const int row = i - lag;
            uptr += ustride;
            const uint2 wnext = word_of(row + 1, uptr);
            __syncthreads();
            const int ryg = row * 16;
            const bool interior = interior_col && row >= 1 && row + 1 < rh;
            float v[16];
            if (A) {
                if (!FLAT) {
                    if (tid == 0 && i >= r_s) {
                        fence_proxy_async();  // generic reads of the slot just released complete before its refill
                        issue(i - r_s + LNS);
                    }
                    wait_block(i - r_s + 3);
                }
                const bool live = col_ok && row >= 0 && row < rh && row <= r_e;
                paint_block<LQS, LHB, LQR, false, true>(word, live, L, st, &qa[0][0], no_raw, FLAT, p.init, rxg, ryg,
                                                        xa0, interior, p.W, p.H, v, &tab);
                {  // dead lanes too (no branch): into ring rows / columns no live lane reads
                    const int wc = 16 * (rc + 1) + L.lx;  // window column in t+1 (origin xb0)
                    const int g = (ryg + L.ly) >> 1;
#pragma unroll
                    for (int r = 0; r < 2; r++)
                        lat_store<LQBS, LQBH>(&qb[0][0], g + r, wc >> 1,
                                          make_float2(((v[8 * r] + v[8 * r + 1]) + v[8 * r + 4]) + v[8 * r + 5],
                                                      ((v[8 * r + 2] + v[8 * r + 3]) + v[8 * r + 6]) + v[8 * r + 7]));
                }
            } else {
                const bool live = col_ok && row >= r_s;
                paint_block<LQBS, LQBH, QR, false, true>(word, live, L, st, &qb[0][0], no_raw, false, p.init, rxg, ryg,
                                                     xb0, interior, p.W, p.H, v, &tab);
                if (live) {
                    if ((word.x & 0xFFFFu) >> 14 == 0) atomicOr(p.state, 1);  // a 2x2 unit: needs the raster path
                    if (!OUT) {  // the lattice of t+2, de-interleaved rows
                        const int gy = (ryg + L.ly) >> 1, gc = (rxg + L.lx) >> 2;
                        float *d = p.nxt + (ptrdiff_t)gy * lw + gc;
#pragma unroll
                        for (int r = 0; r < 2; r++, d += lw) {
                            d[0] = ((v[8 * r] + v[8 * r + 1]) + v[8 * r + 4]) + v[8 * r + 5];
                            d[lw / 2] = ((v[8 * r + 2] + v[8 * r + 3]) + v[8 * r + 6]) + v[8 * r + 7];
                        }
                    } else {
                        store_block(v, nullptr, p.out_u8, p.W, rxg + L.lx, ryg + L.ly);
                    }
                }
            }
            word = wnext;
        }
    };
    if (stage_a)
        run(std::true_type{});
    else
        run(std::false_type{});
}

// The first sweep from the flat raster (an odd sweep count) straight into lattice form, or, for a
// one-sweep decode, into the uint8 image: every unit paints the constant x = clip(s/4 * 4 init +
// (o - s init)) (paint_block's flat path), so a 4x4 block is one value, its four lattice entries
// ((x + x) + x) + x and its pixels floor(x + 0.5).  One thread per block-map entry.
__global__ void flat_lattice_kernel(const uint16_t *block_map, int umap_r0, int rw, int rr0, int rr1, float init,
                                    float *nxt, uint8_t *out, int W) {
    const long long n = (long long)(rr1 - rr0) * rw * 16;
    const int lw = rw * 8;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long root = i >> 4;
        const int l = (int)(i & 15), ry = rr0 + (int)(root / rw), rx = (int)(root % rw);
        const uint32_t d = block_map[((long long)(ry - umap_r0) * rw + rx) * 16 + l];
        const int bx = (l & 1) | ((l >> 1) & 2), by = ((l >> 1) & 1) | ((l >> 2) & 2);  // Morton -> block (x, y)
        const float sc = kUnitS[d & 15];
        const float x = fminf(255.f, fmaxf(0.f, fmaf(0.25f * sc, 4.f * init, fmaf(-sc, init, unit_o(d)))));
        if (out) {
            const uint32_t b = (uint32_t)floorf(x + 0.5f) * 0x01010101u;
            uint8_t *o = out + (ptrdiff_t)(16 * ry + 4 * by) * W + 16 * rx + 4 * bx;
#pragma unroll
            for (int r = 0; r < 4; r++) *reinterpret_cast<uint32_t *>(o + (ptrdiff_t)r * W) = b;
        } else {
            const float v = ((x + x) + x) + x;
            const int gy = 8 * ry + 2 * by, gc = 4 * rx + bx;  // lattice row; column pair (2gc, 2gc + 1)
#pragma unroll
            for (int r = 0; r < 2; r++) {
                float *row = nxt + (ptrdiff_t)(gy + r) * lw;
                row[gc] = v;
                row[lw / 2 + gc] = v;
            }
        }
    }
}

// Unit map from records grouped by root (one warp per root): cells in smem, then one
// coalesced 32-bit word (two cells) per lane.
// BLOCKS: the block map instead (the descriptor of each 4x4 block's first cell, 16 per root).
template <bool BLOCKS>
__global__ void build_unit_map_kernel(const uint64_t *records, const int32_t *root_offsets, int rw, int rr0,
                                      long long n_roots, void *map) {
    __shared__ uint16_t cells[8][64];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long root = (long long)blockIdx.x * 8 + warp;
    if (root >= n_roots) return;
    const int rxg = (int)(root % rw) * 16, ryg = (int)(rr0 + root / rw) * 16;
    for (int i = root_offsets[root] + lane; i < root_offsets[root + 1]; i += 32) {
        const uint64_t r = records[i];
        const int x = (int)((r >> MNS_REC_X_SHIFT) & 0x7FFF) * 2 - rxg, y = (int)((r >> MNS_REC_Y_SHIFT) & 0x7FFF) * 2 - ryg;
        const int size = 32 >> ((int)((r >> MNS_REC_LEVEL_SHIFT) & 3) + 1);
        for (int cy = y; cy < y + size; cy += 2)
            for (int cx = x; cx < x + size; cx += 2)
                cells[warp][morton_of(cx >> 1, cy >> 1)] = mns_unit_of_record(r, rxg, ryg, cx, cy);
    }
    __syncwarp();
    if (BLOCKS) {
        if (lane < 16) static_cast<uint16_t *>(map)[root * 16 + lane] = cells[warp][4 * lane];
    } else {
        static_cast<uint32_t *>(map)[root * 32 + lane] =
            (uint32_t)cells[warp][2 * lane] | ((uint32_t)cells[warp][2 * lane + 1] << 16);
    }
}

// Per-sweep iteration counter when stop_delta == 0 (no early stop possible).
__global__ void set_iters_kernel(int *state, int iters) {
    state[0] = 0;
    state[1] = iters;
}

// clip(floor(x + 0.5)) -> uint8 from the raster that holds the final sweep
__global__ void finalize_kernel(const float *ping, const float *pong, const int *state, uint8_t *out, long long n) {
    const float *src = (state[1] & 1) ? pong : ping;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float v = floorf(src[i] + 0.5f);
        out[i] = (uint8_t)fminf(255.f, fmaxf(0.f, v));
    }
}

__global__ void fill_kernel(float *a, float v, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        a[i] = v;
}

// ---------------------------------------------------------------- generic units
struct UnitParams {
    const int32_t *ux, *uy, *usize, *udx, *udy;
    const float *us, *uo;
    long long n;
    int W;
    const float *cur;
    float *nxt;
    int *state;
    int track_delta;
    float stop_delta;
    int n_ctas;
};

__global__ void __launch_bounds__(256) decode_units_kernel(const UnitParams p) {
    __shared__ float cta_max;
    if (p.state[0]) return;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) cta_max = 0.f;
    __syncthreads();
    float lmax = 0.f;
    const long long warps = (long long)gridDim.x * (blockDim.x / 32);
    for (long long u = blockIdx.x * (long long)(blockDim.x / 32) + (threadIdx.x >> 5); u < p.n; u += warps) {
        // usize = side | isometry << 8 (extension: d_t(i, j) = d(src_t(i, j)); the mean is order-free here)
        const int size = p.usize[u] & 255, iso = p.usize[u] >> 8, x = p.ux[u], y = p.uy[u], dx = p.udx[u],
                  dy = p.udy[u];
        const float s = p.us[u], o = p.uo[u];
        const int n = size * size;
        float acc = 0.f;
        for (int k = lane; k < n; k += 32) {
            const int i = k / size, j = k % size;
            const float *pp = p.cur + (size_t)(dy + 2 * i) * p.W + dx + 2 * j;
            acc += ((pp[0] + pp[1]) + pp[p.W]) + pp[p.W + 1];
        }
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) acc += __shfl_xor_sync(FULL, acc, o2);
        const float mean = acc * 0.25f / (float)n;
        for (int k = lane; k < n; k += 32) {
            const int i = k / size, j = k % size, m = iso ? iso_src(iso, i, j, size) : k;
            const float *pp = p.cur + (size_t)(dy + 2 * (m / size)) * p.W + dx + 2 * (m % size);
            const float q = ((pp[0] + pp[1]) + pp[p.W]) + pp[p.W + 1];
            const float v = fminf(255.f, fmaxf(0.f, fmaf(s, q * 0.25f - mean, o)));
            const size_t idx = (size_t)(y + i) * p.W + x + j;
            if (p.track_delta) lmax = fmaxf(lmax, fabsf(v - p.cur[idx]));
            p.nxt[idx] = v;
        }
    }
    if (p.track_delta) {
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(FULL, lmax, o2));
        if (lane == 0) atomicMax(reinterpret_cast<int *>(&cta_max), __float_as_int(lmax));
        __syncthreads();
        if (threadIdx.x == 0) {
            atomicMax(&p.state[3], __float_as_int(cta_max));
            __threadfence();
            const int done = atomicAdd(&p.state[2], 1);
            if (done == p.n_ctas - 1) {
                __threadfence();
                const float delta = __int_as_float(atomicAdd(&p.state[3], 0));
                p.state[1] += 1;
                if (delta < p.stop_delta) p.state[0] = 1;
                p.state[2] = 0;
                p.state[3] = 0;
            }
        }
    }
}

// ---------------------------------------------------------------- exact fp64 step
__global__ void decode_step_f64_kernel(const int32_t *ux, const int32_t *uy, const int32_t *usize,
                                       const int32_t *udx, const int32_t *udy, const double *us, const double *uo,
                                       long long n, int W, const double *cur, double *out) {
    const long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (u >= n) return;
    const int size = usize[u] & 255, iso = usize[u] >> 8, m = size * size;  // side | isometry << 8
    double d[256];
    for (int i = 0; i < size; i++)
        for (int j = 0; j < size; j++) {  // d_t(i, j) = d(src_t(i, j)), stored in output order
            const int k = iso ? iso_src(iso, i, j, size) : i * size + j;
            const double *pp = cur + (size_t)(udy[u] + 2 * (k / size)) * W + udx[u] + 2 * (k % size);
            d[i * size + j] = __dmul_rn(__dadd_rn(__dadd_rn(__dadd_rn(pp[0], pp[1]), pp[W]), pp[W + 1]), 0.25);
        }
    const double dm = __ddiv_rn(pw_sum_dev(d, m), (double)m);
    for (int i = 0; i < size; i++)
        for (int j = 0; j < size; j++) {
            double v = __dadd_rn(__dmul_rn(us[u], __dsub_rn(d[i * size + j], dm)), uo[u]);
            v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
            out[(size_t)(uy[u] + i) * W + ux[u] + j] = v;
        }
}

int sm_count() {
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

int decode_workspace_bytes(int W, int H, int64_t *bytes) {
    *bytes = 256 + 128ll * (W / 16) * (H / 16);  // state + unit map
    return 0;
}

static int sweep_smem() { return NBUF * RAW_BYTES + QRP * QS * 4; }

static int ensure_sweep_attr() {
    static std::atomic<unsigned long long> done{0};
    MNS_CUDA_TRY(ensure_dynamic_smem(decode_sweep_kernel, sweep_smem(), done));
    return 0;
}

int build_unit_map(const uint64_t *records, const int32_t *root_offsets, int W, int rr0, int rr1, uint32_t *unit_map,
                   cudaStream_t stream) {
    MNS_CHECK_ARG(W > 0 && W % 16 == 0 && 0 <= rr0 && rr0 < rr1, "bad unit-map geometry");
    const long long n_roots = (long long)(W / 16) * (rr1 - rr0);
    build_unit_map_kernel<false><<<(unsigned)((n_roots + 7) / 8), 256, 0, stream>>>(records, root_offsets, W / 16,
                                                                                    rr0, n_roots, unit_map);
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

int build_block_map(const uint64_t *records, const int32_t *root_offsets, int W, int rr0, int rr1,
                    uint16_t *block_map, cudaStream_t stream) {
    MNS_CHECK_ARG(W > 0 && W % 16 == 0 && 0 <= rr0 && rr0 < rr1, "bad block-map geometry");
    const long long n_roots = (long long)(W / 16) * (rr1 - rr0);
    build_unit_map_kernel<true><<<(unsigned)((n_roots + 7) / 8), 256, 0, stream>>>(records, root_offsets, W / 16,
                                                                                   rr0, n_roots, block_map);
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

// One Jacobi sweep over root rows [rr0, rr1).  cur/nxt/out are "virtual global" bases
// (row 0 of the full image); only rows [y_lo, y_hi) of cur are resident and read.
int decode_sweep(const uint32_t *unit_map, int W, int H, int rr0, int rr1, const float *cur, float init,
                 float *nxt, uint8_t *out, int *state, double stop_delta, cudaStream_t stream) {
    MNS_CHECK_ARG(W > 0 && H > 0 && W % 16 == 0 && H % 16 == 0, "width/height must be positive multiples of 16");
    MNS_CHECK_ARG(0 <= rr0 && rr0 < rr1 && rr1 <= H / 16, "bad root row range");
    MNS_CHECK_ARG(H <= 65534, "height exceeds the record coordinate range");
    if (ensure_sweep_attr()) return -1;
    SweepParams p{};
    p.unit_map = unit_map;
    p.W = W;
    p.H = H;
    p.rw = W / 16;
    p.rr0 = rr0;
    p.rr1 = rr1;
    p.y_lo = rr0 * 16 - 16 > 0 ? rr0 * 16 - 16 : 0;
    const int y_hi = rr1 * 16 + 16 < H ? rr1 * 16 + 16 : H;
    p.cur = cur;
    p.init = init;
    p.nxt = nxt;
    p.out_u8 = out;
    p.state = state;
    p.track_delta = stop_delta > 0.0;
    p.stop_delta = (float)stop_delta;
    CUtensorMap tmap{};
    if (cur) {
        if (encode_tmap_2d(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, cur + (ptrdiff_t)p.y_lo * W, (uint64_t)W,
                           (uint64_t)(y_hi - p.y_lo), (uint64_t)W * 4, WINW, BLK))
            return -1;
    }
    p.cr = rows_per_cta(rr1 - rr0, (p.rw + BR - 1) / BR, CR);
    dim3 grid((p.rw + BR - 1) / BR, (rr1 - rr0 + p.cr - 1) / p.cr);
    p.n_ctas = grid.x * grid.y;
    decode_sweep_kernel<<<grid, DT, sweep_smem(), stream>>>(tmap, p);
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

static int ensure_pair_attr() {
    {
        static std::atomic<unsigned long long> done{0};
        MNS_CUDA_TRY(ensure_dynamic_smem(decode_pair_kernel, PAIR_SMEM, done));
    }
    return 0;
}

// Two sweeps over root rows [rr0, rr1) in one pass.  cur/nxt/out are virtual-global bases;
// rows [16 rr0 - 32, 16 rr1 + 32) of cur are resident (32-row halo), and unit_map holds the
// root rows [umap_r0, ...) covering [rr0 - 1, rr1 + 1) clipped to the image.
int decode_sweep2(const uint32_t *unit_map, int umap_r0, int W, int H, int rr0, int rr1, const float *cur, float init,
                  float *nxt, uint8_t *out, cudaStream_t stream) {
    MNS_CHECK_ARG(W > 0 && H > 0 && W % 16 == 0 && H % 16 == 0, "width/height must be positive multiples of 16");
    MNS_CHECK_ARG(0 <= rr0 && rr0 < rr1 && rr1 <= H / 16, "bad root row range");
    MNS_CHECK_ARG(umap_r0 <= (rr0 > 0 ? rr0 - 1 : 0) && umap_r0 >= 0, "unit map must start at root row rr0 - 1");
    MNS_CHECK_ARG(H <= 65534, "height exceeds the record coordinate range");
    MNS_CHECK_ARG((nxt != nullptr) != (out != nullptr), "exactly one of nxt / out");
    if (ensure_pair_attr()) return -1;
    SweepParams p{};
    p.unit_map = unit_map;
    p.umap_r0 = umap_r0;
    p.W = W;
    p.H = H;
    p.rw = W / 16;
    p.rr0 = rr0;
    p.rr1 = rr1;
    p.y_lo = rr0 * 16 - 32 > 0 ? rr0 * 16 - 32 : 0;
    const int y_hi = rr1 * 16 + 32 < H ? rr1 * 16 + 32 : H;
    p.cur = cur;
    p.init = init;
    p.nxt = nxt;
    p.out_u8 = out;
    CUtensorMap tmap{};
    if (cur) {
        if (encode_tmap_2d(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, cur + (ptrdiff_t)p.y_lo * W, (uint64_t)W,
                           (uint64_t)(y_hi - p.y_lo), (uint64_t)W * 4, WA, BLK))
            return -1;
    }
    p.cr = rows_per_cta(rr1 - rr0, (p.rw + BR - 1) / BR, CR2);
    dim3 grid((p.rw + BR - 1) / BR, (rr1 - rr0 + p.cr - 1) / p.cr);
    p.n_ctas = grid.x * grid.y;
    decode_pair_kernel<<<grid, DT2, PAIR_SMEM, stream>>>(tmap, p);
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

static int ensure_lat_attr() {
    static std::atomic<unsigned long long> d0{0}, d1{0}, d2{0}, d3{0};
    MNS_CUDA_TRY(ensure_dynamic_smem(decode_pair_lat_kernel<false, false>, LAT_SMEM, d0));
    MNS_CUDA_TRY(ensure_dynamic_smem(decode_pair_lat_kernel<false, true>, LAT_SMEM, d1));
    MNS_CUDA_TRY(ensure_dynamic_smem(decode_pair_lat_kernel<true, false>, LAT_SMEM, d2));
    MNS_CUDA_TRY(ensure_dynamic_smem(decode_pair_lat_kernel<true, true>, LAT_SMEM, d3));
    return 0;
}

// Two sweeps over root rows [rr0, rr1) on lattice state (see decode_pair_lat_kernel).  cur/nxt are
// virtual-global lattice bases (lattice row 0); lattice rows [8 rr0 - 16, 8 rr1 + 16) of cur are
// resident.  err (device int) is set to 1 if a 2x2 unit is met.
int decode_pass_lattice(const uint16_t *block_map, int umap_r0, int W, int H, int rr0, int rr1, const float *cur,
                        float init, float *nxt, uint8_t *out, int *err, cudaStream_t stream) {
    MNS_CHECK_ARG(W > 0 && H > 0 && W % 16 == 0 && H % 16 == 0, "width/height must be positive multiples of 16");
    MNS_CHECK_ARG(0 <= rr0 && rr0 < rr1 && rr1 <= H / 16, "bad root row range");
    MNS_CHECK_ARG(umap_r0 <= (rr0 > 0 ? rr0 - 1 : 0) && umap_r0 >= 0, "block map must start at root row rr0 - 1");
    MNS_CHECK_ARG(H <= 65534, "height exceeds the record coordinate range");
    MNS_CHECK_ARG((nxt != nullptr) != (out != nullptr), "exactly one of nxt / out");
    MNS_CHECK_ARG(err != nullptr, "error flag required");
    if (ensure_lat_attr()) return -1;
    SweepParams p{};
    p.block_map = block_map;
    p.umap_r0 = umap_r0;
    p.W = W;
    p.H = H;
    p.rw = W / 16;
    p.rr0 = rr0;
    p.rr1 = rr1;
    p.y_lo = rr0 * 16 - 32 > 0 ? rr0 * 16 - 32 : 0;
    const int y_hi = rr1 * 16 + 32 < H ? rr1 * 16 + 32 : H;
    p.cur = cur;
    p.init = init;
    p.nxt = nxt;
    p.out_u8 = out;
    p.state = err;
    CUtensorMap tmap{};
    if (cur) {
        MNS_CHECK_ARG(((uintptr_t)cur & 15) == 0, "lattice must be 16-byte aligned");
        if (encode_tmap_3d(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, cur + (ptrdiff_t)(p.y_lo / 2) * (W / 2),
                           (uint64_t)(W / 4), 2, (uint64_t)((y_hi - p.y_lo) / 2), (uint64_t)W, (uint64_t)W * 2, LHB,
                           2, 8))
            return -1;
    }
    p.cr = rows_per_cta(rr1 - rr0, (p.rw + LBR - 1) / LBR, CR2);
    dim3 grid((p.rw + LBR - 1) / LBR, (rr1 - rr0 + p.cr - 1) / p.cr);
    p.n_ctas = grid.x * grid.y;
    if (cur)
        (out ? decode_pair_lat_kernel<false, true> : decode_pair_lat_kernel<false, false>)<<<grid, LDT, LAT_SMEM,
                                                                                               stream>>>(tmap, p);
    else
        (out ? decode_pair_lat_kernel<true, true> : decode_pair_lat_kernel<true, false>)<<<grid, LDT, LAT_SMEM,
                                                                                             stream>>>(tmap, p);
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

int decode_flat_lattice(const uint16_t *block_map, int umap_r0, int W, int H, int rr0, int rr1, float init, float *nxt,
                        uint8_t *out, cudaStream_t stream) {
    MNS_CHECK_ARG(W > 0 && H > 0 && W % 16 == 0 && H % 16 == 0, "width/height must be positive multiples of 16");
    MNS_CHECK_ARG(0 <= rr0 && rr0 < rr1 && rr1 <= H / 16 && 0 <= umap_r0 && umap_r0 <= rr0, "bad root row range");
    MNS_CHECK_ARG((nxt != nullptr) != (out != nullptr), "exactly one of nxt / out");
    const long long n = (long long)(rr1 - rr0) * (W / 16) * 16;
    const int blocks = (int)std::min<long long>((n + 255) / 256, (long long)sm_count() * 8);
    flat_lattice_kernel<<<blocks, 256, 0, stream>>>(block_map, umap_r0, W / 16, rr0, rr1, init, nxt, out, W);
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

// The whole lattice-state decode (codes without 2x2 units; stop_delta = 0, uint8 output) from a block
// map of all root rows (lat_ping / lat_pong: (H/2) x (W/2) floats each).  *err (device) = 1 if the code
// had a 2x2 unit (a one-sweep decode paints blocks whole and does not look).
int decode_umap_lattice(const uint16_t *umap, int W, int H, int iters, float init, float *lat_ping, float *lat_pong,
                        uint8_t *out, int32_t *err, cudaStream_t stream) {
    MNS_CHECK_ARG(W > 0 && H > 0 && W % 16 == 0 && H % 16 == 0, "width/height must be positive multiples of 16");
    MNS_CHECK_ARG(iters >= 1, "max_iters must be >= 1");
    MNS_CHECK_ARG(out != nullptr && err != nullptr, "out and err required");
    MNS_CUDA_TRY(cudaMemsetAsync(err, 0, 4, stream));
    if (iters == 1) return decode_flat_lattice(umap, 0, W, H, 0, H / 16, init, nullptr, out, stream);
    const float *cur = nullptr;
    int it = 0;
    int rc = 0;
    if (iters & 1) {
        rc = decode_flat_lattice(umap, 0, W, H, 0, H / 16, init, lat_pong, nullptr, stream);
        if (rc) return rc;
        cur = lat_pong;
        it = 1;
    }
    for (; it < iters; it += 2) {
        const bool last = it + 2 == iters;
        float *nxt = last ? nullptr : (cur == lat_ping ? lat_pong : lat_ping);
        rc = decode_pass_lattice(umap, 0, W, H, 0, H / 16, cur, init, nxt, last ? out : nullptr, err, stream);
        if (rc) return rc;
        cur = nxt;
    }
    return 0;
}

// decode_quadtree for codes without 2x2 units, on lattice state: the block map is built from the
// records into the workspace, then decode_umap_lattice.
int decode_quadtree_lattice(const uint64_t *records, const int32_t *root_offsets, int W, int H, int iters, float init,
                            float *lat_ping, float *lat_pong, uint8_t *out, int32_t *err, void *workspace,
                            int64_t workspace_bytes, cudaStream_t stream) {
    MNS_CHECK_ARG(W > 0 && H > 0 && W % 16 == 0 && H % 16 == 0, "width/height must be positive multiples of 16");
    int64_t need;
    decode_workspace_bytes(W, H, &need);
    MNS_CHECK_ARG(workspace_bytes >= need, "workspace too small");
    uint16_t *bmap = reinterpret_cast<uint16_t *>(reinterpret_cast<char *>(workspace) + 256);
    const int rc = build_block_map(records, root_offsets, W, 0, H / 16, bmap, stream);
    if (rc) return rc;
    return decode_umap_lattice(bmap, W, H, iters, init, lat_ping, lat_pong, out, err, stream);
}

// The raster sweeps of a whole-image decode from a unit map (map_form 0) of every root row.
static int decode_from_umap(const uint32_t *umap, int W, int H, int iters, double stop_delta, float init, float *ping,
                            float *pong, uint8_t *out, int32_t *d_iters_done, int *state, cudaStream_t stream) {
    const long long npx = (long long)W * H;
    int rc = 0;
    MNS_CUDA_TRY(cudaMemsetAsync(state, 0, 64, stream));
    const bool track = stop_delta > 0.0;
    if (out && !track && iters >= 2) {
        // no early stop and only the uint8 image wanted: an odd first sweep alone, then two
        // sweeps per pass (the fp32 raster is not materialised after the last sweep)
        const float *cur = nullptr;
        int it = 0;
        if (iters & 1) {
            rc = decode_sweep(umap, W, H, 0, H / 16, nullptr, init, pong, nullptr, state, 0.0, stream);
            if (rc) return rc;
            cur = pong;
            it = 1;
        }
        for (; it < iters; it += 2) {
            const bool last = it + 2 == iters;
            float *nxt = last ? nullptr : (cur == ping ? pong : ping);
            rc = decode_sweep2(umap, 0, W, H, 0, H / 16, cur, init, nxt, last ? out : nullptr, stream);
            if (rc) return rc;
            cur = nxt;
        }
        set_iters_kernel<<<1, 1, 0, stream>>>(state, iters);
        MNS_CUDA_TRY(cudaGetLastError());
        if (d_iters_done)
            MNS_CUDA_TRY(cudaMemcpyAsync(d_iters_done, state + 1, 4, cudaMemcpyDeviceToDevice, stream));
        return 0;
    }
    for (int it = 0; it < iters; it++) {
        // sweep 0 reads the implied flat raster (no fill pass, no read traffic)
        const float *cur = it == 0 ? nullptr : ((it & 1) ? pong : ping);
        // out != NULL and no early stop: the final sweep writes the rounded uint8 image directly
        const bool last_fused = out && !track && it == iters - 1;
        float *nxt = last_fused ? nullptr : ((it & 1) ? ping : pong);
        rc = decode_sweep(umap, W, H, 0, H / 16, cur, init, nxt, last_fused ? out : nullptr, state, stop_delta,
                          stream);
        if (rc) return rc;
    }
    if (!track) set_iters_kernel<<<1, 1, 0, stream>>>(state, iters);
    if (out && track) finalize_kernel<<<sm_count() * 4, 256, 0, stream>>>(ping, pong, state, out, npx);
    if (d_iters_done) MNS_CUDA_TRY(cudaMemcpyAsync(d_iters_done, state + 1, 4, cudaMemcpyDeviceToDevice, stream));
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

int decode_quadtree(const uint64_t *records, const int32_t *root_offsets, int W, int H, int iters,
                    double stop_delta, float init, float *ping, float *pong, uint8_t *out, int32_t *d_iters_done,
                    void *workspace, int64_t workspace_bytes, cudaStream_t stream) {
    MNS_CHECK_ARG(W > 0 && H > 0 && W % 16 == 0 && H % 16 == 0, "width/height must be positive multiples of 16");
    MNS_CHECK_ARG(iters >= 1, "max_iters must be >= 1");
    int64_t need;
    decode_workspace_bytes(W, H, &need);
    MNS_CHECK_ARG(workspace_bytes >= need, "workspace too small");
    MNS_CHECK_ARG(((uintptr_t)ping & 15) == 0 && ((uintptr_t)pong & 15) == 0, "rasters must be 16-byte aligned");
    int *state = reinterpret_cast<int *>(workspace);
    uint32_t *umap = reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(workspace) + 256);
    if (int rc = build_unit_map(records, root_offsets, W, 0, H / 16, umap, stream)) return rc;
    return decode_from_umap(umap, W, H, iters, stop_delta, init, ping, pong, out, d_iters_done, state, stream);
}

// mns_decode_quadtree from the unit map of every root row (as mns_encode_quadtree emits it with
// map_form = 0), skipping the map build; workspace >= 64 bytes.
int decode_unit_map(const uint32_t *unit_map, int W, int H, int iters, double stop_delta, float init, float *ping,
                    float *pong, uint8_t *out, int32_t *d_iters_done, void *workspace, int64_t workspace_bytes,
                    cudaStream_t stream) {
    MNS_CHECK_ARG(W > 0 && H > 0 && W % 16 == 0 && H % 16 == 0, "width/height must be positive multiples of 16");
    MNS_CHECK_ARG(iters >= 1, "max_iters must be >= 1");
    MNS_CHECK_ARG(workspace_bytes >= 64, "workspace too small");
    MNS_CHECK_ARG(((uintptr_t)ping & 15) == 0 && ((uintptr_t)pong & 15) == 0, "rasters must be 16-byte aligned");
    return decode_from_umap(unit_map, W, H, iters, stop_delta, init, ping, pong, out, d_iters_done,
                            reinterpret_cast<int *>(workspace), stream);
}

int decode_units(const int32_t *ux, const int32_t *uy, const int32_t *usize, const int32_t *udx,
                 const int32_t *udy, const float *us, const float *uo, int64_t n, int W, int H, int iters,
                 double stop_delta, float init, float *ping, float *pong, uint8_t *out, int32_t *d_iters_done,
                 void *workspace, int64_t workspace_bytes, cudaStream_t stream) {
    MNS_CHECK_ARG(W > 0 && H > 0, "bad raster size");
    MNS_CHECK_ARG(iters >= 1, "max_iters must be >= 1");
    MNS_CHECK_ARG(workspace_bytes >= 64, "workspace too small");
    int *state = reinterpret_cast<int *>(workspace);
    const long long npx = (long long)W * H;
    MNS_CUDA_TRY(cudaMemsetAsync(state, 0, 64, stream));
    fill_kernel<<<sm_count() * 4, 256, 0, stream>>>(ping, init, npx);
    UnitParams p{ux, uy, usize, udx, udy, us, uo, n, W, nullptr, nullptr, state, stop_delta > 0.0,
                 (float)stop_delta, 0};
    const long long want = (n + 7) / 8;
    const int blocks = (int)(want < sm_count() * 16 ? (want > 0 ? want : 1) : sm_count() * 16);
    p.n_ctas = blocks;
    for (int it = 0; it < iters; it++) {
        p.cur = (it & 1) ? pong : ping;
        p.nxt = (it & 1) ? ping : pong;
        decode_units_kernel<<<blocks, 256, 0, stream>>>(p);
    }
    if (!p.track_delta) set_iters_kernel<<<1, 1, 0, stream>>>(state, iters);
    if (out) finalize_kernel<<<sm_count() * 4, 256, 0, stream>>>(ping, pong, state, out, npx);
    if (d_iters_done) MNS_CUDA_TRY(cudaMemcpyAsync(d_iters_done, state + 1, 4, cudaMemcpyDeviceToDevice, stream));
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

int decode_step_f64(const int32_t *ux, const int32_t *uy, const int32_t *usize, const int32_t *udx,
                    const int32_t *udy, const double *us, const double *uo, int64_t n, int W, int H,
                    const double *cur, double *out, cudaStream_t stream) {
    MNS_CHECK_ARG(W > 0 && H > 0, "bad raster size");
    if (n == 0) return 0;
    decode_step_f64_kernel<<<(unsigned)((n + 63) / 64), 64, 0, stream>>>(ux, uy, usize, udx, udy, us, uo, n, W, cur,
                                                                          out);
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

}  // namespace mns
