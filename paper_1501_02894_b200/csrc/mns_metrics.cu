// Device metrics for the rate-distortion sweep (bench.py:39-79 rd_sweep):
//   * exact squared error of two uint8 images -- the numerator of metrics.py:16-31 mse/psnr
//     (an integer < 2^16 per pixel, so the uint64 sum is exact; the host divides once);
//   * the leaf tallies of a packed code -- encoder.py:135-142 level_counts / phase2_count.

#include "mns_common.cuh"

namespace mns {
namespace {

constexpr unsigned FULL = 0xffffffffu;

// one CTA row of threads per image row stripe; 16 pixels per thread per step
__global__ void sse_kernel(const uint8_t *a, int64_t pa, const uint8_t *b, int64_t pb, int W, int H,
                           unsigned long long *out) {
    unsigned long long acc = 0;
    for (int y = blockIdx.y; y < H; y += gridDim.y) {
        const uint8_t *ra = a + (ptrdiff_t)y * pa, *rb = b + (ptrdiff_t)y * pb;
        for (int x = (blockIdx.x * blockDim.x + threadIdx.x); x < W; x += gridDim.x * blockDim.x) {
            const int d = (int)ra[x] - (int)rb[x];
            acc += (unsigned long long)(d * d);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// out[0..3] = leaves per level 1..4, out[4] = phase-2 leaves (warp-aggregated atomics)
__global__ void code_stats_kernel(const uint64_t *rec, long long n, unsigned long long *out) {
    unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const uint64_t r = rec[i];
        const int lv = (int)((r >> MNS_REC_LEVEL_SHIFT) & 3);
#pragma unroll
        for (int k = 0; k < 4; k++) c[k] += lv == k;
        const int p2 = (int)((r >> MNS_REC_PHASE2_SHIFT) & 1);
        c[4] += p2;
        c[5] += lv == 3 || (lv == 2 && p2);  // leaves painted as 2x2 units (level 4, level-3 quadrants)
    }
#pragma unroll
    for (int k = 0; k < 6; k++) {
        unsigned long long v = c[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&out[k], v);
    }
}

// per range: offset (dx, dy) = domain centre - range centre (cli.py:98-104 samples of
// encoder.py:249-309), dense marginal and joint counts (bench.py:119-127 offset_histogram)
__global__ void offset_hist_kernel(const int32_t *dom, long long n, int ndx, int step, int B, int rpr, int ox, int oy,
                                   int jw, int *hx, int *hy, int *joint) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int d = dom[i];
        const int dx = (d % ndx) * step + B - ((int)(i % rpr) * B + B / 2);
        const int dy = (d / ndx) * step + B - ((int)(i / rpr) * B + B / 2);
        atomicAdd(&hx[dx + ox], 1);
        atomicAdd(&hy[dy + oy], 1);
        atomicAdd(&joint[(long long)(dy + oy) * jw + (dx + ox)], 1);
    }
}

}  // namespace

int offset_histogram(const int32_t *dom, int64_t n_ranges, int W, int H, int B, int step, int32_t *hist_x,
                     int32_t *hist_y, int32_t *joint, cudaStream_t stream) {
    MNS_CHECK_ARG(B > 0 && step > 0 && W >= 2 * B && H >= 2 * B && W % B == 0 && H % B == 0, "bad search geometry");
    MNS_CHECK_ARG(n_ranges == (int64_t)(W / B) * (H / B), "n_ranges must be (W/B)*(H/B)");
    const int ox = W, oy = H, jw = 2 * W + 1, jh = 2 * H + 1;
    MNS_CUDA_TRY(cudaMemsetAsync(hist_x, 0, (size_t)jw * 4, stream));
    MNS_CUDA_TRY(cudaMemsetAsync(hist_y, 0, (size_t)jh * 4, stream));
    MNS_CUDA_TRY(cudaMemsetAsync(joint, 0, (size_t)jw * jh * 4, stream));
    const int ndx = (W - 2 * B) / step + 1;
    const long long blocks = (n_ranges + 255) / 256 < 1184 ? (n_ranges + 255) / 256 : 1184;
    offset_hist_kernel<<<(unsigned)(blocks > 0 ? blocks : 1), 256, 0, stream>>>(dom, n_ranges, ndx, step, B, W / B, ox,
                                                                                 oy, jw, hist_x, hist_y, joint);
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

int image_sse(const uint8_t *a, int64_t pitch_a, const uint8_t *b, int64_t pitch_b, int W, int H, uint64_t *out,
              cudaStream_t stream) {
    MNS_CHECK_ARG(W > 0 && H > 0 && pitch_a >= W && pitch_b >= W, "bad image geometry");
    MNS_CUDA_TRY(cudaMemsetAsync(out, 0, 8, stream));
    const dim3 grid((unsigned)((W + 255) / 256 < 8 ? (W + 255) / 256 : 8), (unsigned)(H < 1024 ? H : 1024));
    sse_kernel<<<grid, 256, 0, stream>>>(a, pitch_a, b, pitch_b, W, H, reinterpret_cast<unsigned long long *>(out));
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

int code_stats(const uint64_t *records, int64_t n, int64_t *out6, cudaStream_t stream) {
    MNS_CHECK_ARG(n >= 0, "negative record count");
    MNS_CUDA_TRY(cudaMemsetAsync(out6, 0, 6 * 8, stream));
    if (n == 0) return 0;
    const long long blocks = (n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184;
    code_stats_kernel<<<(unsigned)blocks, 256, 0, stream>>>(records, n, reinterpret_cast<unsigned long long *>(out6));
    MNS_CUDA_TRY(cudaGetLastError());
    return 0;
}

}  // namespace mns
