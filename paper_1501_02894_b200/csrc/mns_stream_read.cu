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
//  * chunks of CHUNK bits are walked token by token from their own start in parallel,
//    marking token starts in a bitmap; then, round after round, a chunk whose true entry (the
//    previous chunk's exit) differs from the start it walked from re-walks from the entry
//    until it lands on a start its old walk marked (the walks merge; the rest is shared) or
//    leaves the chunk with a new exit.  Rounds stop when no exit changes.
//  * the token starts are compacted; exclusive scans of token areas (in 2x2 cells: 64, 16, 4,
//    4 for a quartet) and leaf counts give every leaf its root, Morton cell and record slot.
//  * every check the sequential parser makes (level id below the node's level, interrupted
//    quartet, negative-zero delta, truncation) is recorded as a key ordered by bit position;
//    the minimum is the parser's first error (the host maps it to StreamFormatError).

#include <algorithm>

#include "mns_common.cuh"

namespace mns {
namespace {

constexpr long long HDR = 13 * 8;
constexpr int CHUNK = 8192;  // bits per speculative chunk (128 bitmap words)
constexpr int ST = 256, SIPT = 8, STILE = ST * SIPT;

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
};

__device__ __forceinline__ bool marked(const RP &r, long long p) {
    const long long i = p - HDR;
    return (r.bitmap[i >> 6] >> (i & 63)) & 1;
}
__device__ __forceinline__ void set_mark(const RP &r, long long p) {
    const long long i = p - HDR;
    r.bitmap[i >> 6] |= 1ull << (i & 63);
}

__global__ void spec_walk_kernel(const RP r, long long *exits, long long *starts) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= r.nchunks) return;
    const long long c0 = HDR + t * CHUNK, c1 = min(c0 + CHUNK, r.nbits);
    long long p = c0;
    while (p < c1) {
        set_mark(r, p);
        p += tok_width(peek64(r.data, r.nbytes, p), r.mns, r.t2);
    }
    exits[t] = p;
    starts[t] = c0;
}

__global__ void resync_kernel(const RP r, const long long *exit_in, long long *exit_out, long long *starts,
                              int *changed) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= r.nchunks) return;
    if (t == 0) {
        exit_out[0] = exit_in[0];
        return;
    }
    const long long e = exit_in[t - 1];
    if (e == starts[t]) {
        exit_out[t] = exit_in[t];
        return;
    }
    const long long c0 = HDR + t * CHUNK, c1 = min(c0 + CHUNK, r.nbits);
    long long p = e;
    bool merged = false;
    while (p < c1) {
        if (marked(r, p)) {
            merged = true;
            break;
        }
        p += tok_width(peek64(r.data, r.nbytes, p), r.mns, r.t2);
    }
    // rewrite this chunk's marks before the merge point: clear, then mark the walk from e
    const long long stop = min(p, c1);
    for (long long q = c0; q < stop;) {
        const long long i = q - HDR, wi = i >> 6;
        const int b = (int)(i & 63), n = (int)min(64ll - b, stop - q);
        const unsigned long long m = n == 64 ? ~0ull : (((1ull << n) - 1) << b);
        r.bitmap[wi] &= ~m;
        q += n;
    }
    for (long long q = e; q < stop;) {
        set_mark(r, q);
        q += tok_width(peek64(r.data, r.nbytes, q), r.mns, r.t2);
    }
    starts[t] = e;
    exit_out[t] = merged ? exit_in[t] : p;
    if (!merged && p != exit_in[t]) atomicAdd(changed, 1);
}

// exclusive scan of n int64 (decoupled look-back over STILE-element tiles); total -> *total
__global__ void __launch_bounds__(ST) scan_kernel(const long long *in, long long *out, long long n,
                                                  unsigned long long *status, long long *total) {
    __shared__ long long warp_tot[ST / 32];
    __shared__ long long base_sh;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long long tile = blockIdx.x, i0 = tile * STILE + (long long)tid * SIPT;
    long long v[SIPT], run = 0;
#pragma unroll
    for (int k = 0; k < SIPT; k++) {
        v[k] = i0 + k < n ? in[i0 + k] : 0;
        run += v[k];
    }
    long long incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    long long wbase = 0, tt = 0;
#pragma unroll
    for (int k = 0; k < ST / 32; k++) {
        wbase += k < warp ? warp_tot[k] : 0;
        tt += warp_tot[k];
    }
    if (warp == 0) {
        const long long b = lookback_exclusive_warp(status, tile, tt);
        if (lane == 0) base_sh = b;
    }
    __syncthreads();
    long long e = base_sh + wbase + incl - run;
#pragma unroll
    for (int k = 0; k < SIPT; k++) {
        if (i0 + k < n) out[i0 + k] = e;
        e += v[k];
    }
    if (tile == gridDim.x - 1 && tid == ST - 1) *total = e;
}

__global__ void popc_kernel(const unsigned long long *bitmap, long long nwords, long long *cnt) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nwords; i += (long long)gridDim.x * blockDim.x)
        cnt[i] = __popcll(bitmap[i]);
}

__global__ void token_list_kernel(const unsigned long long *bitmap, long long nwords, const long long *wbase,
                                  long long *tokpos) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nwords; i += (long long)gridDim.x * blockDim.x) {
        unsigned long long m = bitmap[i];
        long long k = wbase[i];
        while (m) {
            const int b = __ffsll((long long)m) - 1;
            tokpos[k++] = HDR + i * 64 + b;
            m &= m - 1;
        }
    }
}

__global__ void token_info_kernel(const RP r, const long long *tokpos, long long ntok, long long *area,
                                  long long *nleaf) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ntok; i += (long long)gridDim.x * blockDim.x) {
        const int lid = (int)(peek64(r.data, r.nbytes, tokpos[i]) >> 62);
        area[i] = lid == 3 ? 4 : (64 >> (2 * lid));
        nleaf[i] = lid == 3 ? 4 : 1;
    }
}

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

__global__ void emit_kernel(const RP r, const EmitParams e, const long long *tokpos, const long long *cell0,
                            const long long *leaf0, long long ntok) {
    unsigned long long *ekey = reinterpret_cast<unsigned long long *>(&e.status[0]);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ntok; i += (long long)gridDim.x * blockDim.x) {
        const long long c = cell0[i];
        if (c >= e.total_cells) continue;
        const long long p = tokpos[i];
        const uint64_t w = peek64(r.data, r.nbytes, p);
        const int lid = (int)(w >> 62);
        const int width = tok_width(w, r.mns, r.t2);
        if (p + 2 > r.nbits) {
            atomicMin(ekey, err_key(r.nbits, E_TRUNC, 0, 0));
            continue;
        }
        const long long L0 = leaf0[i];
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
    }
}

unsigned grid_for(long long n, int threads) {
    const long long b = (n + threads - 1) / threads;
    return (unsigned)(b < 1 ? 1 : (b > 4096 ? 4096 : b));
}

struct ReadWs {
    unsigned long long *bitmap, *status;
    long long *exit_a, *exit_b, *starts, *wcnt, *wbase, *tokpos, *area, *nleaf, *cell0, *leaf0, *totals;
    int *changed;
    long long nwords, nchunks, maxtok, scan_tiles;
};

long long read_ws_layout(long long nbytes, ReadWs *w, char *base) {
    const long long nbits = nbytes * 8, body = nbits > HDR ? nbits - HDR : 0;
    const long long nwords = (body + 63) / 64 + 1, nchunks = (body + CHUNK - 1) / CHUNK + 1;
    const long long maxtok = body / 13 + 2;
    const long long scan_tiles = (std::max(nwords, maxtok) + STILE - 1) / STILE + 1;
    long long off = 0;
    auto take = [&](long long bytes) {
        const long long o = off;
        off += (bytes + 255) / 256 * 256;
        return base ? base + o : nullptr;
    };
    ReadWs t{};
    t.bitmap = (unsigned long long *)take(nwords * 8);
    t.status = (unsigned long long *)take(scan_tiles * 8);
    t.exit_a = (long long *)take(nchunks * 8);
    t.exit_b = (long long *)take(nchunks * 8);
    t.starts = (long long *)take(nchunks * 8);
    t.wcnt = (long long *)take(nwords * 8);
    t.wbase = (long long *)take(nwords * 8);
    t.tokpos = (long long *)take(maxtok * 8);
    t.area = (long long *)take(maxtok * 8);
    t.nleaf = (long long *)take(maxtok * 8);
    t.cell0 = (long long *)take(maxtok * 8);
    t.leaf0 = (long long *)take(maxtok * 8);
    t.totals = (long long *)take(4 * 8);
    t.changed = (int *)take(8);
    t.nwords = nwords;
    t.nchunks = nchunks;
    t.maxtok = maxtok;
    t.scan_tiles = scan_tiles;
    if (w) *w = t;
    return off;
}

int scan(const long long *in, long long *out, long long n, ReadWs &w, long long *total, cudaStream_t s) {
    const long long tiles = (n + STILE - 1) / STILE;
    MNS_CUDA_TRY(cudaMemsetAsync(w.status, 0, (tiles > 0 ? tiles : 1) * 8, s));
    if (n == 0) {
        MNS_CUDA_TRY(cudaMemsetAsync(total, 0, 8, s));
        return 0;
    }
    scan_kernel<<<(unsigned)tiles, ST, 0, s>>>(in, out, n, w.status, total);
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
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
    RP r{data, nbytes, nbytes * 8, 0, mns ? 1 : 0, t2 ? 1 : 0, w.bitmap};
    const long long body = r.nbits - HDR;
    r.nchunks = (body + CHUNK - 1) / CHUNK;
    const long long n_roots = (long long)(pw / 16) * (ph / 16);
    // status: no error, no final leaf yet
    const long long init[2] = {-1, -1};
    MNS_CUDA_TRY(cudaMemcpyAsync(d_status, init, 16, cudaMemcpyHostToDevice, s));
    MNS_CUDA_TRY(cudaMemsetAsync(d_count, 0, 8, s));
    MNS_CUDA_TRY(cudaMemsetAsync(w.bitmap, 0, w.nwords * 8, s));
    long long ntok = 0;
    if (r.nchunks > 0) {
        spec_walk_kernel<<<grid_for(r.nchunks, 128), 128, 0, s>>>(r, w.exit_a, w.starts);
        MNS_CUDA_TRY(cudaGetLastError());
        long long *ein = w.exit_a, *eout = w.exit_b;
        for (int round = 0; round < 100000; round++) {  // bounded: each round fixes at least one chunk
            MNS_CUDA_TRY(cudaMemsetAsync(w.changed, 0, 4, s));
            resync_kernel<<<grid_for(r.nchunks, 128), 128, 0, s>>>(r, ein, eout, w.starts, w.changed);
            MNS_CUDA_TRY(cudaGetLastError());
            int changed = 0;
            MNS_CUDA_TRY(cudaMemcpyAsync(&changed, w.changed, 4, cudaMemcpyDeviceToHost, s));
            MNS_CUDA_TRY(cudaStreamSynchronize(s));
            std::swap(ein, eout);
            if (!changed) break;
        }
        // token list
        const long long nwords = (body + 63) / 64;
        popc_kernel<<<grid_for(nwords, 256), 256, 0, s>>>(w.bitmap, nwords, w.wcnt);
        MNS_CUDA_TRY(cudaGetLastError());
        if (scan(w.wcnt, w.wbase, nwords, w, &w.totals[0], s)) return -1;
        MNS_CUDA_TRY(cudaMemcpyAsync(&ntok, &w.totals[0], 8, cudaMemcpyDeviceToHost, s));
        MNS_CUDA_TRY(cudaStreamSynchronize(s));
        MNS_CHECK_ARG(ntok <= w.maxtok, "token count overflow");
        token_list_kernel<<<grid_for(nwords, 256), 256, 0, s>>>(w.bitmap, nwords, w.wbase, w.tokpos);
        MNS_CUDA_TRY(cudaGetLastError());
    }
    if (ntok > 0) {
        token_info_kernel<<<grid_for(ntok, 256), 256, 0, s>>>(r, w.tokpos, ntok, w.area, w.nleaf);
        MNS_CUDA_TRY(cudaGetLastError());
        if (scan(w.area, w.cell0, ntok, w, &w.totals[1], s)) return -1;
        if (scan(w.nleaf, w.leaf0, ntok, w, &w.totals[2], s)) return -1;
        EmitParams e{n_roots * 64, pw / 16, records, capacity, root_offsets, d_count,
                     reinterpret_cast<long long *>(d_status)};
        emit_kernel<<<grid_for(ntok, 256), 256, 0, s>>>(r, e, w.tokpos, w.cell0, w.leaf0, ntok);
        MNS_CUDA_TRY(cudaGetLastError());
    }
    return 0;
}

}  // namespace mns
