// .mns bitstream reader for sm_100a.
//
// Replaces bitstream.py:208-279 (read_stream) for the leaf body of a container whose
// 13-byte header the host has validated.  The stream is a DFS of variable-width leaves with
// no synchronisation markers, so the parse is speculative:
//
//  * tokens: every leaf starts with a 2-bit level id except the 2nd..4th members of a level-4
//    quartet under Technique 2, and an id of 3 always opens a whole quartet (a level-4 leaf
//    only occurs as a split level-3 node's first child, bitstream.py:249-256).  So a token --
//    one level-1..3 leaf, or a level-4 quartet -- has a width that is a function of the bits
//    at its start: 2 + [phase bit] + payload, or 46 (Technique 2) / 52 bits for a quartet.
//  * chunks of CHUNK bits: the walk through a chunk maps its entry offset (< 52, the widest
//    token) to the next chunk's; every chunk tabulates that map for all 52 offsets (walks that
//    meet past a probe point share the rest), the maps
//    compose over groups and supergroups of 64, the true entries resolve top-down from the
//    stream start, and one walk per chunk marks the token starts in a bitmap (exit_table_kernel
//    .. mark_kernel).
//  * one pass over the token-start bitmap (tokens_kernel) sums each tile's token areas (in 2x2
//    cells: 64, 16, 4, 4 for a quartet) and leaf counts, scans them across tiles (decoupled
//    look-back), and walks the tokens again to emit every leaf at its root, Morton cell and record
//    slot -- no token list, no host round trip.
//  * every check the sequential parser makes (level id below the node's level, interrupted
//    quartet, negative-zero delta, truncation) is recorded as a key ordered by bit position;
//    the minimum is the parser's first error (the host maps it to StreamFormatError).

#include <algorithm>

#include "mns_common.cuh"

namespace mns {
namespace {

constexpr long long HDR = 13 * 8;
#ifndef RD_CHUNK
#define RD_CHUNK 8192
#endif
constexpr int CHUNK = RD_CHUNK;  // bits per chunk (CHUNK / 64 bitmap words)

enum { E_LEVEL = 1, E_SIBLING = 2, E_NEGZERO = 3, E_TRUNC = 4 };

__device__ __forceinline__ unsigned long long err_key(long long pos, int code, int a, int b) {
    return ((unsigned long long)pos << 16) | ((unsigned long long)code << 8) | ((unsigned long long)a << 4) |
           (unsigned long long)b;
}

__device__ __forceinline__ uint64_t bswap64(uint64_t v) {
    const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
    return ((uint64_t)__byte_perm(lo, 0, 0x0123) << 32) | (uint64_t)__byte_perm(hi, 0, 0x0123);
}

// 64 stream bits from bit position pos, MSB first; bytes past the end read as 0.  Two aligned
// 8-byte loads + a funnel shift (the buffer is 8-byte aligned; the tail takes the byte path).
__device__ __forceinline__ uint64_t peek64(const uint8_t *d, long long nbytes, long long pos) {
    const long long b = pos >> 3, a = b & ~7ll;
    const int off = (int)((b - a) * 8 + (pos & 7));
    uint64_t w0, w1;
    if (a + 16 <= nbytes) {
        w0 = bswap64(__ldg(reinterpret_cast<const unsigned long long *>(d + a)));
        w1 = bswap64(__ldg(reinterpret_cast<const unsigned long long *>(d + a + 8)));
    } else {
        w0 = w1 = 0;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            w0 = (w0 << 8) | (uint64_t)(a + i < nbytes ? __ldg(d + a + i) : 0);
            w1 = (w1 << 8) | (uint64_t)(a + 8 + i < nbytes ? __ldg(d + a + 8 + i) : 0);
        }
    }
    return off ? (w0 << off) | (w1 >> (64 - off)) : w0;
}

__device__ __forceinline__ int tok_width(uint64_t w, int mns, int t2) {
    const int lid = (int)(w >> 62);
    if (lid == 3) return t2 ? 46 : 52;
    const int ph = mns ? (int)((w >> 61) & 1) : 0;
    return 2 + mns + (ph ? (lid == 0 ? 27 : 30) : 11);
}

struct RP {
    const uint8_t *data;
    long long nbytes, nbits, nchunks;
    int mns, t2;
    unsigned long long *bitmap;  // token starts, bit (p - HDR)
    uint64_t wtab;               // tok_width by the token's top three bits, 6 bits per entry
};

// the same widths as one table lookup: width = (wtab >> 6 * top3) & 63
static uint64_t width_table(int mns, int t2) {
    uint64_t t = 0;
    for (int i = 0; i < 8; i++) {
        const uint64_t w = (uint64_t)i << 61;
        const int lid = (int)(w >> 62), ph = mns ? (int)((w >> 61) & 1) : 0;
        const int width = lid == 3 ? (t2 ? 46 : 52) : 2 + mns + (ph ? (lid == 0 ? 27 : 30) : 11);
        t |= (uint64_t)width << (6 * i);
    }
    return t;
}
__device__ __forceinline__ int tok_w(uint64_t w, uint64_t wtab) { return (int)((wtab >> (6 * (int)(w >> 61))) & 63); }

// Token synchronisation by exit tables.  A token is at most 52 bits wide, so the first token start
// at or after a chunk's first bit lies within 52 bits of it: the walk through chunk t is a function
// f_t of its entry offset (0..51) onto the next chunk's entry offset.  Every chunk tabulates f_t
// (one lane per entry offset, 52 walks in lockstep over the same bytes), the tables compose in a
// three-level hierarchy (64 chunks per group, 64 groups per supergroup; each level a chain of
// table lookups per possible entry), the true entries resolve top-down from offset 0 at the
// stream start, and a last walk per chunk marks the true token starts.  No host round trips, and
// the work does not depend on how slowly a misaligned walk re-synchronises.
constexpr int NE = 64;      // table row (entries 0..51 used)
constexpr int MAXW = 52;    // widest token (bits)
constexpr int TG = 64;      // chunks per group, groups per supergroup

// Sequential MSB-first reader for one walk: three big-endian stream words in registers (the one
// holding the cursor, the next, and one prefetched), so a token costs no load until the walk
// crosses a word, and that load was issued two words earlier.
struct Cursor {
    const uint8_t *d;
    long long nbytes, k;  // k: word index (8-byte units) of w0
    uint64_t w0, w1, w2;
    __device__ __forceinline__ uint64_t word(long long i) const {
        const long long a = 8 * i;
        if (a + 8 <= nbytes) return bswap64(__ldg(reinterpret_cast<const unsigned long long *>(d + a)));
        uint64_t v = 0;
        for (int b = 0; b < 8; b++) v = (v << 8) | (uint64_t)(a + b < nbytes ? __ldg(d + a + b) : 0);
        return v;
    }
    __device__ __forceinline__ Cursor(const uint8_t *data, long long nb, long long p) : d(data), nbytes(nb) {
        k = p >> 6;
        w0 = word(k);
        w1 = word(k + 1);
        w2 = word(k + 2);
    }
    // 64 bits from p (p >= 64 k, moving forward by less than 64 bits per call)
    __device__ __forceinline__ uint64_t peek(long long p) {
        if ((p >> 6) != k) {
            k++;
            w0 = w1;
            w1 = w2;
            w2 = word(k + 2);
        }
        const int off = (int)(p & 63);
        return off ? (w0 << off) | (w1 >> (64 - off)) : w0;
    }
};

// f_t: tab[t * NE + j] = (first token start at or after c1) - c1 for the walk from c0 + j.  Walks from
// nearby offsets land on common token starts after a few tokens, so the 52 walks of a chunk run in
// lockstep only to the probe point c0 + PROBE; walks whose first start past it coincide share the
// rest, and only one walk per distinct start goes on (exit_finish_kernel, one thread per distinct
// start), the others copy its exit (exit_copy_kernel).
#ifndef RD_PROBE
#define RD_PROBE 256
#endif
constexpr int PROBE = RD_PROBE;  // bits walked by all 52 offsets

__global__ void __launch_bounds__(256) exit_probe_kernel(const RP r, uint8_t *tab, uint8_t *lead,
                                                         unsigned long long *work, unsigned *nwork) {
    __shared__ long long qs[4][NE];
    const int c = threadIdx.x >> 6, j = threadIdx.x & 63;
    const long long t = blockIdx.x * 4ll + c;
    const bool on = t < r.nchunks && j < MAXW;
    const long long c0 = HDR + t * CHUNK, c1 = on ? min(c0 + CHUNK, r.nbits) : 0;
    long long p = c0 + j;
    if (on) {
        const long long stop = min(c0 + PROBE, c1);
        Cursor cur(r.data, r.nbytes, p);
        while (p < stop) p += tok_w(cur.peek(p), r.wtab);
        qs[c][j] = p;
    }
    __syncthreads();
    if (!on) return;
    int leader = j;
    for (int i = 0; i < j; i++)
        if (qs[c][i] == p) {
            leader = i;
            break;
        }
    lead[t * NE + j] = (uint8_t)leader;
    if (leader != j) return;
    if (p >= c1) {
        tab[t * NE + j] = (uint8_t)(p - c1);
    } else {  // (chunk, offset, walk position - c0)
        const unsigned k = atomicAdd(nwork, 1u);
        work[k] = ((unsigned long long)t << 20) | ((unsigned long long)j << 14) | (unsigned long long)(p - c0);
    }
}

__global__ void exit_finish_kernel(const RP r, uint8_t *tab, const unsigned long long *work, const unsigned *nwork) {
    const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k >= *nwork) return;
    const unsigned long long it = work[k];
    const long long t = (long long)(it >> 20), j = (long long)((it >> 14) & 63);
    const long long c0 = HDR + t * CHUNK, c1 = min(c0 + CHUNK, r.nbits);
    long long p = c0 + (long long)(it & 16383);
    Cursor cur(r.data, r.nbytes, p);
    while (p < c1) p += tok_w(cur.peek(p), r.wtab);
    tab[t * NE + j] = (uint8_t)(p - c1);
}

__global__ void exit_copy_kernel(const RP r, uint8_t *tab, const uint8_t *lead) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= r.nchunks * NE || (i & (NE - 1)) >= MAXW) return;
    const int l = lead[i];
    if (l != (int)(i & (NE - 1))) tab[i] = tab[(i & ~(long long)(NE - 1)) + l];
}

// one level up: out[g * NE + j] = the composition of in's rows [g * TG, g * TG + TG) from entry j
__global__ void __launch_bounds__(256) compose_kernel(const uint8_t *in, long long nrows, uint8_t *out,
                                                      long long ngroups) {
    const long long g = blockIdx.x * 4ll + (threadIdx.x >> 6);
    const int j = threadIdx.x & 63;
    if (g >= ngroups || j >= MAXW) return;
    int e = j;
    const long long t1 = min((g + 1) * TG, nrows);
    for (long long t = g * TG; t < t1; t++) e = in[t * NE + e];
    out[g * NE + j] = (uint8_t)e;
}

// entries top-down: ent[g] for every row of a level from the level above (one thread per parent
// row, a chain of TG lookups); the root level starts from offset 0 (the stream's first leaf)
__global__ void resolve_kernel(const uint8_t *tab, long long nrows, const int *parent_ent, long long nparents,
                               int *ent) {
    const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (q >= nparents) return;
    int e = parent_ent ? parent_ent[q] : 0;
    const long long t1 = min((q + 1) * TG, nrows);
    for (long long t = q * TG; t < t1; t++) {
        ent[t] = e;
        e = tab[t * NE + e];
    }
}

// the true token starts of chunk t: the walk from its resolved entry, marks accumulated per bitmap
// word in a register and each word stored once (a chunk's words are its own: chunks are word
// aligned; words without a start stay zero from the memset)
__global__ void mark_kernel(const RP r, const int *ent) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= r.nchunks) return;
    const long long c0 = HDR + t * CHUNK, c1 = min(c0 + CHUNK, r.nbits);
    long long p = c0 + ent[t], cw = (c0 - HDR) >> 6;
    unsigned long long acc = 0;
    Cursor cur(r.data, r.nbytes, p);
    while (p < c1) {
        const long long i = p - HDR;
        if ((i >> 6) != cw) {
            r.bitmap[cw] = acc;
            cw = i >> 6;
            acc = 0;
        }
        acc |= 1ull << (i & 63);
        p += tok_w(cur.peek(p), r.wtab);
    }
    if (acc) r.bitmap[cw] = acc;
}

// exclusive scan of n int64 (decoupled look-back over STILE-element tiles); total -> *total
struct EmitParams {
    long long total_cells;
    int rw;
    uint64_t *records;
    long long capacity;
    int32_t *root_offsets;
    int64_t *count;
    long long *status;  // [0] first error key (as unsigned), [1] end bit position of the final leaf
};

__device__ __forceinline__ void cell_xy(long long c, int rw, int &x, int &y) {
    const long long root = c >> 6;
    const int m = (int)(c & 63);
    int cx = 0, cy = 0;
#pragma unroll
    for (int i = 0; i < 3; i++) {
        cx |= ((m >> (2 * i)) & 1) << i;
        cy |= ((m >> (2 * i + 1)) & 1) << i;
    }
    x = (int)(root % rw) * 16 + 2 * cx;
    y = (int)(root / rw) * 16 + 2 * cy;
}

// The token at bit p, whose first 2x2 cell (in the DFS / Morton order of the roots) is c and whose
// first leaf is record L0: its records, and the checks the sequential parser makes at this token.
__device__ __forceinline__ void emit_token(const RP &r, const EmitParams &e, long long p, uint64_t w, long long c,
                                           long long L0) {
    unsigned long long *ekey = reinterpret_cast<unsigned long long *>(&e.status[0]);
    do {
        if (c >= e.total_cells) continue;
        const int lid = (int)(w >> 62);
        const int width = tok_width(w, r.mns, r.t2);
        if (p + 2 > r.nbits) {
            atomicMin(ekey, err_key(r.nbits, E_TRUNC, 0, 0));
            continue;
        }
        if (c % 64 == 0) e.root_offsets[c >> 6] = (int32_t)L0;
        if (lid == 3) {  // level-4 quartet: TL leaf with its id, then TR, BL, BR
            for (int k = 0; k < 4; k++) {
                const long long q = p + 13 * k;  // member k's id (no Technique 2)
                if (k > 0 && !r.t2) {
                    if (q + 2 > r.nbits) break;
                    const int sib = (int)(peek64(r.data, r.nbytes, q) >> 62);
                    if (sib != 3) {
                        atomicMin(ekey, err_key(q, E_SIBLING, sib + 1, 0));
                        break;
                    }
                }
                const long long pl = r.t2 ? p + 2 + 11 * k : q + 2;  // member k's payload
                const uint64_t v = peek64(r.data, r.nbytes, pl);
                int x, y;
                cell_xy(c + k, e.rw, x, y);
                if (L0 + k < e.capacity) e.records[L0 + k] = mns_rec_phase1(x, y, 4, (int)(v >> 56), (int)((v >> 53) & 7));
            }
        } else {
            const int depth = lid + 1, area = 64 >> (2 * lid);
            if (c % area) {
                const int lvl = c % 64 == 0 ? 1 : (c % 16 == 0 ? 2 : 3);
                atomicMin(ekey, err_key(p, E_LEVEL, depth, lvl));
                continue;
            }
            const int ph = r.mns ? (int)((w >> 61) & 1) : 0;
            const long long pl = p + 2 + r.mns;
            const uint64_t v = peek64(r.data, r.nbytes, pl);
            int x, y;
            cell_xy(c, e.rw, x, y);
            uint64_t rec;
            if (!ph) {
                rec = mns_rec_phase1(x, y, depth, (int)(v >> 56), (int)((v >> 53) & 7));
            } else {
                const int nb = depth == 1 ? 4 : 5;
                int d[3], off = 8;
                bool bad = false;
                for (int j = 0; j < 3; j++) {
                    const int sign = (int)((v >> (63 - off)) & 1);
                    const int mag = (int)((v >> (64 - (off + 1 + nb))) & ((1u << nb) - 1));
                    if (sign && mag == 0 && pl + off + 1 + nb <= r.nbits) {
                        atomicMin(ekey, err_key(pl + off, E_NEGZERO, 0, 0));
                        bad = true;
                        break;
                    }
                    d[j] = sign ? -mag : mag;
                    off += 1 + nb;
                }
                if (bad) continue;
                const int sb = (int)((v >> (64 - (off + 4))) & 15);
                rec = mns_rec_phase2(x, y, depth, (int)(v >> 56), d[0], d[1], d[2],
                                     ((sb >> 3) & 1) | (((sb >> 2) & 1) << 1) | (((sb >> 1) & 1) << 2) | ((sb & 1) << 3));
            }
            if (L0 < e.capacity) e.records[L0] = rec;
        }
        if (p + width > r.nbits) atomicMin(ekey, err_key(r.nbits, E_TRUNC, 0, 0));
        const int area = lid == 3 ? 4 : (64 >> (2 * lid));
        if (c + area == e.total_cells) {  // the final leaf
            e.status[1] = p + width;
            *e.count = L0 + (lid == 3 ? 4 : 1);
            e.root_offsets[e.total_cells >> 6] = (int32_t)(L0 + (lid == 3 ? 4 : 1));
        }
    } while (false);
}

// Token pass (one kernel from the token-start bitmap to the records): a tile of TT threads x TW
// bitmap words; each thread walks the token starts of its words twice -- first summing their
// (cells, leaves) packed as cells << 28 | leaves (< 2^34 and 2^28 for any stream the exit tables
// accept: <= 2^31 bits, tokens >= 13 bits, >= 11.5 bits per leaf), then, after a block scan and a
// decoupled look-back over the tiles, emitting each token at its running (cell, leaf) origin.
constexpr int TT = 256, TW = 4, TTILE = TT * TW;
constexpr int PK_SHIFT = 28;
constexpr unsigned long long PK_LEAF = (1ull << PK_SHIFT) - 1;

__device__ __forceinline__ unsigned long long tok_pack(uint64_t w) {
    const int lid = (int)(w >> 62);
    return lid == 3 ? (4ull << PK_SHIFT) | 4ull : ((64ull >> (2 * lid)) << PK_SHIFT) | 1ull;
}

__global__ void __launch_bounds__(TT) tokens_kernel(const RP r, const EmitParams e, long long nwords,
                                                    unsigned long long *status) {
    __shared__ unsigned long long warp_tot[TT / 32];
    __shared__ unsigned long long base_sh;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long long tile = blockIdx.x, w0 = tile * TTILE + (long long)tid * TW;
    unsigned long long m[TW];
    {
        const ulonglong2 *b2 = reinterpret_cast<const ulonglong2 *>(r.bitmap + w0);
#pragma unroll
        for (int k = 0; k < TW; k += 2) {
            if (w0 + k + 1 < nwords) {
                const ulonglong2 v = b2[k / 2];
                m[k] = v.x;
                m[k + 1] = v.y;
            } else {
                m[k] = w0 + k < nwords ? r.bitmap[w0 + k] : 0ull;
                m[k + 1] = 0ull;
            }
        }
    }
    unsigned long long run = 0;
#pragma unroll
    for (int k = 0; k < TW; k++) {
        for (unsigned long long b = m[k]; b; b &= b - 1)
            run += tok_pack(peek64(r.data, r.nbytes, HDR + (w0 + k) * 64 + (__ffsll((long long)b) - 1)));
    }
    unsigned long long incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    unsigned long long wbase = 0, tt = 0;
#pragma unroll
    for (int k = 0; k < TT / 32; k++) {
        wbase += k < warp ? warp_tot[k] : 0ull;
        tt += warp_tot[k];
    }
    if (warp == 0) {
        const long long b = lookback_exclusive_warp(status, tile, (long long)tt);
        if (lane == 0) base_sh = (unsigned long long)b;
    }
    __syncthreads();
    unsigned long long ex = base_sh + wbase + incl - run;
#pragma unroll
    for (int k = 0; k < TW; k++) {
        for (unsigned long long b = m[k]; b; b &= b - 1) {
            const long long p = HDR + (w0 + k) * 64 + (__ffsll((long long)b) - 1);
            const uint64_t w = peek64(r.data, r.nbytes, p);
            emit_token(r, e, p, w, (long long)(ex >> PK_SHIFT), (long long)(ex & PK_LEAF));
            ex += tok_pack(w);
        }
    }
}

// one thread per item, no cap (the token-synchronisation kernels do not grid-stride)
unsigned blocks_for(long long n, int threads) {
    const long long b = (n + threads - 1) / threads;
    return (unsigned)(b < 1 ? 1 : b);
}


struct ReadWs {
    unsigned long long *bitmap, *status;
    uint8_t *tab, *gtab, *sgtab;  // exit tables: chunks, groups, supergroups (NE bytes per row)
    uint8_t *lead;                // per chunk entry: the offset whose walk it shares past the probe
    unsigned long long *work;     // distinct walks past the probe (chunk, offset, position)
    unsigned *nwork;
    int *ent_c, *ent_g, *ent_s;   // resolved entry offsets per level
    long long nwords, nchunks, tok_tiles;
};

long long read_ws_layout(long long nbytes, ReadWs *w, char *base) {
    const long long nbits = nbytes * 8, body = nbits > HDR ? nbits - HDR : 0;
    const long long nwords = (body + 63) / 64 + 1, nchunks = (body + CHUNK - 1) / CHUNK + 1;
    const long long tok_tiles = (nwords + TTILE - 1) / TTILE + 1;
    long long off = 0;
    auto take = [&](long long bytes) {
        const long long o = off;
        off += (bytes + 255) / 256 * 256;
        return base ? base + o : nullptr;
    };
    ReadWs t{};
    t.bitmap = (unsigned long long *)take(nwords * 8);
    t.status = (unsigned long long *)take(tok_tiles * 8);
    const long long ngroups = (nchunks + TG - 1) / TG, nsg = (ngroups + TG - 1) / TG;
    t.tab = (uint8_t *)take(nchunks * NE);
    t.lead = (uint8_t *)take(nchunks * NE);
    t.work = (unsigned long long *)take(nchunks * MAXW * 8);
    t.nwork = (unsigned *)take(8);
    t.gtab = (uint8_t *)take(ngroups * NE);
    t.sgtab = (uint8_t *)take(nsg * NE);
    t.ent_c = (int *)take(nchunks * 4);
    t.ent_g = (int *)take(ngroups * 4);
    t.ent_s = (int *)take(nsg * 4);
    t.nwords = nwords;
    t.nchunks = nchunks;
    t.tok_tiles = tok_tiles;
    if (w) *w = t;
    return off;
}

}  // namespace

int read_stream_workspace_bytes(int64_t nbytes, int64_t *bytes) {
    *bytes = read_ws_layout(nbytes, nullptr, nullptr);
    return 0;
}

int read_stream(const uint8_t *data, int64_t nbytes, int mns, int t2, int pw, int ph, uint64_t *records,
                int64_t capacity, int32_t *root_offsets, int64_t *d_count, int64_t *d_status, void *workspace,
                int64_t workspace_bytes, cudaStream_t s) {
    MNS_CHECK_ARG(pw > 0 && ph > 0 && pw % 16 == 0 && ph % 16 == 0, "padded dimensions must be positive multiples of 16");
    MNS_CHECK_ARG(nbytes >= 13, "stream shorter than its header");
    MNS_CHECK_ARG(((uintptr_t)data & 7) == 0, "stream buffer must be 8-byte aligned");
    int64_t need;
    read_stream_workspace_bytes(nbytes, &need);
    MNS_CHECK_ARG(workspace_bytes >= need, "workspace too small");
    ReadWs w;
    read_ws_layout(nbytes, &w, reinterpret_cast<char *>(workspace));
    RP r{data, nbytes, nbytes * 8, 0, mns ? 1 : 0, t2 ? 1 : 0, w.bitmap, width_table(mns ? 1 : 0, t2 ? 1 : 0)};
    const long long body = r.nbits - HDR;
    r.nchunks = (body + CHUNK - 1) / CHUNK;
    const long long n_roots = (long long)(pw / 16) * (ph / 16);
    // status: no error, no final leaf yet
    const long long init[2] = {-1, -1};
    MNS_CUDA_TRY(cudaMemcpyAsync(d_status, init, 16, cudaMemcpyHostToDevice, s));
    MNS_CUDA_TRY(cudaMemsetAsync(d_count, 0, 8, s));
    MNS_CUDA_TRY(cudaMemsetAsync(w.bitmap, 0, w.nwords * 8, s));
    if (r.nchunks > 0) {
        const long long ngroups = (r.nchunks + TG - 1) / TG, nsg = (ngroups + TG - 1) / TG;
        MNS_CHECK_ARG(nsg <= TG, "stream longer than the reader's three table levels (268 MB)");
        MNS_CUDA_TRY(cudaMemsetAsync(w.nwork, 0, 4, s));
        exit_probe_kernel<<<(unsigned)((r.nchunks + 3) / 4), 256, 0, s>>>(r, w.tab, w.lead, w.work, w.nwork);
        exit_finish_kernel<<<blocks_for(r.nchunks * MAXW, 128), 128, 0, s>>>(r, w.tab, w.work, w.nwork);
        exit_copy_kernel<<<blocks_for(r.nchunks * NE, 256), 256, 0, s>>>(r, w.tab, w.lead);
        compose_kernel<<<(unsigned)((ngroups + 3) / 4), 256, 0, s>>>(w.tab, r.nchunks, w.gtab, ngroups);
        compose_kernel<<<(unsigned)((nsg + 3) / 4), 256, 0, s>>>(w.gtab, ngroups, w.sgtab, nsg);
        resolve_kernel<<<1, 32, 0, s>>>(w.sgtab, nsg, nullptr, 1, w.ent_s);  // from offset 0 (needs nsg <= 64)
        resolve_kernel<<<blocks_for(nsg, 64), 64, 0, s>>>(w.gtab, ngroups, w.ent_s, nsg, w.ent_g);
        resolve_kernel<<<blocks_for(ngroups, 64), 64, 0, s>>>(w.tab, r.nchunks, w.ent_g, ngroups, w.ent_c);
        mark_kernel<<<blocks_for(r.nchunks, 64), 64, 0, s>>>(r, w.ent_c);
        MNS_CUDA_TRY(cudaGetLastError());
        // token pass: cells and leaves of every token, their scan, the records
        const long long nwords = (body + 63) / 64;
        const long long tiles = (nwords + TTILE - 1) / TTILE;
        MNS_CUDA_TRY(cudaMemsetAsync(w.status, 0, tiles * 8, s));
        EmitParams e{n_roots * 64, pw / 16, records, capacity, root_offsets, d_count,
                     reinterpret_cast<long long *>(d_status)};
        tokens_kernel<<<(unsigned)tiles, TT, 0, s>>>(r, e, nwords, w.status);
        MNS_CUDA_TRY(cudaGetLastError());
    }
    return 0;
}

}  // namespace mns
