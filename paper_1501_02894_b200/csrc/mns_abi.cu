// extern "C" boundary of libmns_b200.so (include/mns_b200.h): argument checks,
// thread-local error strings, and dispatch to the sm_100a kernels.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>

#include "mns_common.cuh"
#include "mns_tma.cuh"

namespace mns {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

double sqrt_bound(double E) {
    if (!(E < INFINITY)) return INFINITY;
    double x = E * E;
    while (x > 0.0 && sqrt(x) > E) x = nextafter(x, 0.0);
    while (sqrt(nextafter(x, INFINITY)) <= E) x = nextafter(x, INFINITY);
    return x;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !ptr) {
            set_error("cuTensorMapEncodeTiled unavailable");
            return nullptr;
        }
        fn = (EncodeTiledFn)ptr;
    }
    return fn;
}

static int encode_tmap_impl(CUtensorMap *map, CUtensorMapDataType dtype, const void *base, uint64_t width,
                            uint64_t height, uint64_t row_bytes, uint32_t box_w, uint32_t box_h,
                            CUtensorMapSwizzle swz) {
    const EncodeTiledFn fn = encode_tiled_fn();
    if (!fn) return -1;
    const cuuint64_t dims[2] = {width, height};
    const cuuint64_t strides[1] = {row_bytes};
    const cuuint32_t box[2] = {box_w, box_h};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(map, dtype, 2, const_cast<void *>(base), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
        return -1;
    }
    return 0;
}

int encode_tmap_3d(CUtensorMap *map, CUtensorMapDataType dtype, const void *base, uint64_t d0, uint64_t d1,
                   uint64_t d2, uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box0, uint32_t box1,
                   uint32_t box2) {
    const EncodeTiledFn fn = encode_tiled_fn();
    if (!fn) return -1;
    const cuuint64_t dims[3] = {d0, d1, d2};
    const cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
    const cuuint32_t box[3] = {box0, box1, box2};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = fn(map, dtype, 3, const_cast<void *>(base), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled (3d) failed (%d)", (int)r);
        return -1;
    }
    return 0;
}

int encode_tmap_2d(CUtensorMap *map, CUtensorMapDataType dtype, int, const void *base, uint64_t width,
                   uint64_t height, uint64_t row_bytes, uint32_t box_w, uint32_t box_h) {
    return encode_tmap_impl(map, dtype, base, width, height, row_bytes, box_w, box_h, CU_TENSOR_MAP_SWIZZLE_NONE);
}

int encode_tmap_2d_swizzled(CUtensorMap *map, CUtensorMapDataType dtype, const void *base, uint64_t width,
                            uint64_t height, uint64_t row_bytes, uint32_t box_w, uint32_t box_h) {
    return encode_tmap_impl(map, dtype, base, width, height, row_bytes, box_w, box_h, CU_TENSOR_MAP_SWIZZLE_128B);
}

int encode_workspace_bytes(int width, int n_images, int rr0, int rr1, int64_t *bytes);
int encode_quadtree(const uint8_t *img, int W, int H, int64_t pitch, int64_t image_stride, int n_images, int rr0,
                    int rr1, const mns_enc_cfg *cfg, uint64_t *records, int64_t capacity, int32_t *root_offsets,
                    int64_t *d_count, uint32_t *unit_map, void *workspace, int64_t workspace_bytes,
                    cudaStream_t stream, cudaStream_t cstream);
int build_unit_map(const uint64_t *records, const int32_t *root_offsets, int W, int rr0, int rr1, uint32_t *unit_map,
                   cudaStream_t stream);
int build_block_map(const uint64_t *records, const int32_t *root_offsets, int W, int rr0, int rr1,
                    uint16_t *block_map, cudaStream_t stream);
int try_node(const uint8_t *img, int W, int H, int64_t pitch, int x, int y, int level, int phase,
             const mns_enc_cfg *cfg, uint64_t *d_rec, double *d_rms, cudaStream_t stream);
int decode_workspace_bytes(int W, int H, int64_t *bytes);
int decode_pass_lattice(const uint16_t *block_map, int umap_r0, int W, int H, int rr0, int rr1, const float *cur,
                        float init, float *nxt, uint8_t *out, int *err, cudaStream_t stream);
int decode_flat_lattice(const uint16_t *block_map, int umap_r0, int W, int H, int rr0, int rr1, float init, float *nxt,
                        uint8_t *out, cudaStream_t stream);
int decode_quadtree_lattice(const uint64_t *records, const int32_t *root_offsets, int W, int H, int iters, float init,
                            float *lat_ping, float *lat_pong, uint8_t *out, int32_t *err, void *workspace,
                            int64_t workspace_bytes, cudaStream_t stream);
int decode_umap_lattice(const uint16_t *umap, int W, int H, int iters, float init, float *lat_ping, float *lat_pong,
                        uint8_t *out, int32_t *err, cudaStream_t stream);
int decode_quadtree(const uint64_t *records, const int32_t *root_offsets, int W, int H, int iters,
                    double stop_delta, float init, float *ping, float *pong, uint8_t *out, int32_t *d_iters_done,
                    void *workspace, int64_t workspace_bytes, cudaStream_t stream);
int decode_unit_map(const uint32_t *unit_map, int W, int H, int iters, double stop_delta, float init, float *ping,
                    float *pong, uint8_t *out, int32_t *d_iters_done, void *workspace, int64_t workspace_bytes,
                    cudaStream_t stream);
int decode_sweep(const uint32_t *unit_map, int W, int H, int rr0, int rr1, const float *cur, float init,
                 float *nxt, uint8_t *out, int *state, double stop_delta, cudaStream_t stream);
int decode_sweep2(const uint32_t *unit_map, int umap_r0, int W, int H, int rr0, int rr1, const float *cur, float init,
                  float *nxt, uint8_t *out, cudaStream_t stream);
int decode_units(const int32_t *ux, const int32_t *uy, const int32_t *usize, const int32_t *udx,
                 const int32_t *udy, const float *us, const float *uo, int64_t n, int W, int H, int iters,
                 double stop_delta, float init, float *ping, float *pong, uint8_t *out, int32_t *d_iters_done,
                 void *workspace, int64_t workspace_bytes, cudaStream_t stream);
int decode_step_f64(const int32_t *ux, const int32_t *uy, const int32_t *usize, const int32_t *udx,
                    const int32_t *udy, const double *us, const double *uo, int64_t n, int W, int H,
                    const double *cur, double *out, cudaStream_t stream);
int decode_f64(const int32_t *ux, const int32_t *uy, const int32_t *usize, const int32_t *udx, const int32_t *udy,
               const double *us, const double *uo, int64_t n, int W, int H, int iters, double stop_delta,
               double init, double *ping, double *pong, uint8_t *out, int32_t *d_iters_done, void *workspace,
               int64_t workspace_bytes, cudaStream_t st);
int records_to_units(const uint64_t *records, int64_t n, int W, int H, int32_t *ux, int32_t *uy, int32_t *usize,
                     int32_t *udx, int32_t *udy, double *us, double *uo, cudaStream_t st);
int decode_f64_sweep(const int32_t *ux, const int32_t *uy, const int32_t *usize, const int32_t *udx,
                     const int32_t *udy, const double *us, const double *uo, int64_t n, int W, const double *cur,
                     double *nxt, int64_t *state, cudaStream_t st);
int decode_f64_decide(int64_t *state, double stop_delta, cudaStream_t st);
int decode_f64_finalize(const double *ping, const double *pong, const int64_t *state, int W, int y0, int y1,
                        uint8_t *out, int32_t *iters_done, cudaStream_t st);
int search_workspace_bytes(int W, int H, int B, int step, int n_iso, int64_t *bytes);
int full_search(const uint8_t *img, int W, int H, int B, int step, int n_iso, int r0, int r1, int32_t *out_dom,
                int8_t *out_iso, uint8_t *out_o, uint8_t *out_code, void *ws, int64_t ws_bytes, cudaStream_t st);
int local_search(const uint8_t *img, int W, int H, int radius, int n_iso, int32_t *out_dx, int32_t *out_dy,
                 int8_t *out_iso, uint8_t *out_o, uint8_t *out_code, cudaStream_t st);
int local_search_workspace_bytes(int W, int H, int radius, int n_iso, int64_t *bytes);
int local_search_ws(const uint8_t *img, int W, int H, int radius, int n_iso, int32_t *out_dx, int32_t *out_dy,
                    int8_t *out_iso, uint8_t *out_o, uint8_t *out_code, void *ws, int64_t ws_bytes, cudaStream_t st);
int stream_workspace_bytes(int64_t n, int64_t *bytes);
int write_stream(const uint64_t *records, int64_t n, int ow, int oh, int pw, int ph, int mns, int t2, uint8_t *out,
                 int64_t cap, int64_t *d_bits, void *ws, int64_t ws_bytes, cudaStream_t st);

int image_sse(const uint8_t *a, int64_t pitch_a, const uint8_t *b, int64_t pitch_b, int W, int H, uint64_t *out,
              cudaStream_t stream);
int read_stream_workspace_bytes(int64_t nbytes, int64_t *bytes);
int read_stream(const uint8_t *data, int64_t nbytes, int mns, int t2, int pw, int ph, uint64_t *records,
                int64_t capacity, int32_t *root_offsets, int64_t *d_count, int64_t *d_status, void *workspace,
                int64_t workspace_bytes, cudaStream_t s);
int code_stats(const uint64_t *records, int64_t n, int64_t *out6, cudaStream_t stream);
int offset_histogram(const int32_t *dom, int64_t n_ranges, int W, int H, int B, int step, int32_t *hist_x,
                     int32_t *hist_y, int32_t *joint, cudaStream_t stream);

}  // namespace mns

#define GUARD(call)                                                   \
    try {                                                             \
        return call;                                              \
    } catch (...) {                                                   \
        mns::set_error("unexpected C++ exception");                   \
        return -3;                                                    \
    }

extern "C" {

const char *mns_last_error(void) { return mns::g_err; }
int mns_version(void) { return 1; }

int mns_read_stream_workspace_bytes(int64_t n_bytes, int64_t *bytes) {
    GUARD(mns::read_stream_workspace_bytes(n_bytes, bytes));
}

int mns_read_stream(const uint8_t *data, int64_t n_bytes, int32_t mns, int32_t technique2, int32_t padded_w,
                    int32_t padded_h, uint64_t *records, int64_t capacity, int32_t *root_offsets, int64_t *d_count,
                    int64_t *d_status, void *workspace, int64_t workspace_bytes, void *stream) {
    GUARD(mns::read_stream(data, n_bytes, mns, technique2, padded_w, padded_h, records, capacity, root_offsets,
                           d_count, d_status, workspace, workspace_bytes, (cudaStream_t)stream));
}

int mns_image_sse(const uint8_t *a, int64_t pitch_a, const uint8_t *b, int64_t pitch_b, int32_t width, int32_t height,
                  uint64_t *d_sse, void *stream) {
    GUARD(mns::image_sse(a, pitch_a, b, pitch_b, width, height, d_sse, (cudaStream_t)stream));
}

int mns_code_stats(const uint64_t *records, int64_t n_records, int64_t *d_out6, void *stream) {
    GUARD(mns::code_stats(records, n_records, d_out6, (cudaStream_t)stream));
}

int mns_offset_histogram(const int32_t *dom, int64_t n_ranges, int32_t width, int32_t height, int32_t range_size,
                         int32_t step, int32_t *hist_x, int32_t *hist_y, int32_t *joint, void *stream) {
    GUARD(mns::offset_histogram(dom, n_ranges, width, height, range_size, step, hist_x, hist_y, joint,
                                (cudaStream_t)stream));
}

int mns_encode_workspace_bytes(int32_t width, int32_t n_images, int32_t rr0, int32_t rr1, int64_t *bytes) {
    GUARD(mns::encode_workspace_bytes(width, n_images, rr0, rr1, bytes));
}

int mns_encode_quadtree(const uint8_t *img, int32_t width, int32_t height, int64_t pitch, int64_t image_stride,
                        int32_t n_images, int32_t rr0, int32_t rr1, const mns_enc_cfg *cfg, uint64_t *records,
                        int64_t capacity, int32_t *root_offsets, int64_t *d_count, uint32_t *unit_map,
                        void *workspace, int64_t workspace_bytes, void *stream) {
    GUARD(mns::encode_quadtree(img, width, height, pitch, image_stride, n_images, rr0, rr1, cfg, records, capacity,
                               root_offsets, d_count, unit_map, workspace, workspace_bytes, (cudaStream_t)stream,
                               (cudaStream_t)stream));
}

int mns_encode_quadtree_split(const uint8_t *img, int32_t width, int32_t height, int64_t pitch, int64_t image_stride,
                              int32_t n_images, int32_t rr0, int32_t rr1, const mns_enc_cfg *cfg, uint64_t *records,
                              int64_t capacity, int32_t *root_offsets, int64_t *d_count, uint32_t *unit_map,
                              void *workspace, int64_t workspace_bytes, void *stream, void *compact_stream) {
    GUARD(mns::encode_quadtree(img, width, height, pitch, image_stride, n_images, rr0, rr1, cfg, records, capacity,
                               root_offsets, d_count, unit_map, workspace, workspace_bytes, (cudaStream_t)stream,
                               (cudaStream_t)compact_stream));
}

int mns_try_node(const uint8_t *img, int32_t width, int32_t height, int64_t pitch, int32_t x, int32_t y, int32_t level,
                 int32_t phase, const mns_enc_cfg *cfg, uint64_t *record, double *rms, void *stream) {
    GUARD(mns::try_node(img, width, height, pitch, x, y, level, phase, cfg, record, rms, (cudaStream_t)stream));
}

int mns_build_unit_map(const uint64_t *records, const int32_t *root_offsets, int32_t width, int32_t root_row_begin,
                       int32_t root_row_end, uint32_t *unit_map, void *stream) {
    GUARD(mns::build_unit_map(records, root_offsets, width, root_row_begin, root_row_end, unit_map,
                              (cudaStream_t)stream));
}

int mns_build_block_map(const uint64_t *records, const int32_t *root_offsets, int32_t width, int32_t root_row_begin,
                        int32_t root_row_end, uint16_t *block_map, void *stream) {
    GUARD(mns::build_block_map(records, root_offsets, width, root_row_begin, root_row_end, block_map,
                               (cudaStream_t)stream));
}

int mns_decode_workspace_bytes(int32_t width, int32_t height, int64_t *bytes) {
    GUARD(mns::decode_workspace_bytes(width, height, bytes));
}

int mns_decode_quadtree(const uint64_t *records, const int32_t *root_offsets, int32_t width, int32_t height,
                        int32_t iters, double stop_delta, float initial_value, float *ping, float *pong,
                        uint8_t *out, int32_t *d_iters_done, void *workspace, int64_t workspace_bytes,
                        void *stream) {
    GUARD(mns::decode_quadtree(records, root_offsets, width, height, iters, stop_delta, initial_value, ping, pong,
                               out, d_iters_done, workspace, workspace_bytes, (cudaStream_t)stream));
}

int mns_decode_unit_map(const uint32_t *unit_map, int32_t width, int32_t height, int32_t iters, double stop_delta,
                        float initial_value, float *ping, float *pong, uint8_t *out, int32_t *d_iters_done,
                        void *workspace, int64_t workspace_bytes, void *stream) {
    GUARD(mns::decode_unit_map(unit_map, width, height, iters, stop_delta, initial_value, ping, pong, out,
                               d_iters_done, workspace, workspace_bytes, (cudaStream_t)stream));
}

int mns_decode_sweep(const uint32_t *unit_map, int32_t width, int32_t height, int32_t root_row_begin,
                     int32_t root_row_end, const float *cur, float initial_value, float *nxt, uint8_t *out,
                     int32_t *state, double stop_delta, void *stream) {
    GUARD(mns::decode_sweep(unit_map, width, height, root_row_begin, root_row_end, cur, initial_value, nxt, out,
                            state, stop_delta, (cudaStream_t)stream));
}

int mns_decode_sweep2(const uint32_t *unit_map, int32_t unit_map_row_begin, int32_t width, int32_t height,
                      int32_t root_row_begin, int32_t root_row_end, const float *cur, float initial_value, float *nxt,
                      uint8_t *out, void *stream) {
    GUARD(mns::decode_sweep2(unit_map, unit_map_row_begin, width, height, root_row_begin, root_row_end, cur,
                             initial_value, nxt, out, (cudaStream_t)stream));
}

int mns_decode_pass_lattice(const uint16_t *block_map, int32_t block_map_row_begin, int32_t width, int32_t height,
                            int32_t root_row_begin, int32_t root_row_end, const float *cur_lattice, float initial_value,
                            float *nxt_lattice, uint8_t *out, int32_t *d_error, void *stream) {
    GUARD(mns::decode_pass_lattice(block_map, block_map_row_begin, width, height, root_row_begin, root_row_end,
                                   cur_lattice, initial_value, nxt_lattice, out, d_error, (cudaStream_t)stream));
}

int mns_decode_flat_lattice(const uint16_t *block_map, int32_t block_map_row_begin, int32_t width, int32_t height,
                            int32_t root_row_begin, int32_t root_row_end, float initial_value, float *nxt_lattice,
                            uint8_t *out, void *stream) {
    GUARD(mns::decode_flat_lattice(block_map, block_map_row_begin, width, height, root_row_begin, root_row_end,
                                   initial_value, nxt_lattice, out, (cudaStream_t)stream));
}

int mns_decode_quadtree_lattice(const uint64_t *records, const int32_t *root_offsets, int32_t width, int32_t height,
                                int32_t iters, float initial_value, float *lat_ping, float *lat_pong, uint8_t *out,
                                int32_t *d_error, void *workspace, int64_t workspace_bytes, void *stream) {
    GUARD(mns::decode_quadtree_lattice(records, root_offsets, width, height, iters, initial_value, lat_ping, lat_pong,
                                       out, d_error, workspace, workspace_bytes, (cudaStream_t)stream));
}

int mns_decode_unit_map_lattice(const uint16_t *block_map, int32_t width, int32_t height, int32_t iters,
                                float initial_value, float *lat_ping, float *lat_pong, uint8_t *out, int32_t *d_error,
                                void *workspace, int64_t workspace_bytes, void *stream) {
    (void)workspace;
    (void)workspace_bytes;
    GUARD(mns::decode_umap_lattice(block_map, width, height, iters, initial_value, lat_ping, lat_pong, out, d_error,
                                   (cudaStream_t)stream));
}

int mns_decode_units(const int32_t *ux, const int32_t *uy, const int32_t *usize, const int32_t *udx,
                     const int32_t *udy, const float *us, const float *uo, int64_t n_units, int32_t width,
                     int32_t height, int32_t iters, double stop_delta, float initial_value, float *ping,
                     float *pong, uint8_t *out, int32_t *d_iters_done, void *workspace, int64_t workspace_bytes,
                     void *stream) {
    GUARD(mns::decode_units(ux, uy, usize, udx, udy, us, uo, n_units, width, height, iters, stop_delta,
                            initial_value, ping, pong, out, d_iters_done, workspace, workspace_bytes,
                            (cudaStream_t)stream));
}

int mns_decode_step_f64(const int32_t *ux, const int32_t *uy, const int32_t *usize, const int32_t *udx,
                        const int32_t *udy, const double *us, const double *uo, int64_t n_units, int32_t width,
                        int32_t height, const double *cur, double *out, void *stream) {
    GUARD(mns::decode_step_f64(ux, uy, usize, udx, udy, us, uo, n_units, width, height, cur, out,
                               (cudaStream_t)stream));
}

int mns_decode_f64(const int32_t *ux, const int32_t *uy, const int32_t *usize, const int32_t *udx,
                   const int32_t *udy, const double *us, const double *uo, int64_t n_units, int32_t width,
                   int32_t height, int32_t max_iters, double stop_delta, double initial_value, double *ping,
                   double *pong, uint8_t *out, int32_t *d_iters_done, void *workspace, int64_t workspace_bytes,
                   void *stream) {
    GUARD(mns::decode_f64(ux, uy, usize, udx, udy, us, uo, n_units, width, height, max_iters, stop_delta,
                          initial_value, ping, pong, out, d_iters_done, workspace, workspace_bytes,
                          (cudaStream_t)stream));
}

int mns_records_to_units(const uint64_t *records, int64_t n_records, int32_t width, int32_t height, int32_t *ux,
                         int32_t *uy, int32_t *usize, int32_t *udx, int32_t *udy, double *us, double *uo,
                         void *stream) {
    GUARD(mns::records_to_units(records, n_records, width, height, ux, uy, usize, udx, udy, us, uo,
                                (cudaStream_t)stream));
}

int mns_decode_f64_sweep(const int32_t *ux, const int32_t *uy, const int32_t *usize, const int32_t *udx,
                         const int32_t *udy, const double *us, const double *uo, int64_t n_units, int32_t width,
                         const double *cur, double *nxt, int64_t *state, void *stream) {
    GUARD(mns::decode_f64_sweep(ux, uy, usize, udx, udy, us, uo, n_units, width, cur, nxt, state,
                                (cudaStream_t)stream));
}

int mns_decode_f64_decide(int64_t *state, double stop_delta, void *stream) {
    GUARD(mns::decode_f64_decide(state, stop_delta, (cudaStream_t)stream));
}

int mns_decode_f64_finalize(const double *ping, const double *pong, const int64_t *state, int32_t width,
                            int32_t row_begin, int32_t row_end, uint8_t *out, int32_t *d_iters_done, void *stream) {
    GUARD(mns::decode_f64_finalize(ping, pong, state, width, row_begin, row_end, out, d_iters_done,
                                   (cudaStream_t)stream));
}

int mns_search_workspace_bytes(int32_t width, int32_t height, int32_t B, int32_t step, int32_t n_iso,
                               int64_t *bytes) {
    GUARD(mns::search_workspace_bytes(width, height, B, step, n_iso, bytes));
}

int mns_full_search(const uint8_t *img, int32_t width, int32_t height, int32_t B, int32_t step, int32_t n_iso,
                    int32_t range_begin, int32_t range_end, int32_t *out_dom, int8_t *out_iso, uint8_t *out_o,
                    uint8_t *out_code, void *workspace, int64_t workspace_bytes, void *stream) {
    GUARD(mns::full_search(img, width, height, B, step, n_iso, range_begin, range_end, out_dom, out_iso, out_o,
                           out_code, workspace, workspace_bytes, (cudaStream_t)stream));
}

int mns_local_search(const uint8_t *img, int32_t width, int32_t height, int32_t radius, int32_t n_iso,
                     int32_t *out_dx, int32_t *out_dy, int8_t *out_iso, uint8_t *out_o, uint8_t *out_code,
                     void *stream) {
    GUARD(mns::local_search(img, width, height, radius, n_iso, out_dx, out_dy, out_iso, out_o, out_code,
                            (cudaStream_t)stream));
}

int mns_local_search_workspace_bytes(int32_t width, int32_t height, int32_t radius, int32_t n_iso, int64_t *bytes) {
    GUARD(mns::local_search_workspace_bytes(width, height, radius, n_iso, bytes));
}

int mns_local_search_tc(const uint8_t *img, int32_t width, int32_t height, int32_t radius, int32_t n_iso,
                        int32_t *out_dx, int32_t *out_dy, int8_t *out_iso, uint8_t *out_o, uint8_t *out_code,
                        void *workspace, int64_t workspace_bytes, void *stream) {
    GUARD(mns::local_search_ws(img, width, height, radius, n_iso, out_dx, out_dy, out_iso, out_o, out_code, workspace,
                               workspace_bytes, (cudaStream_t)stream));
}

int mns_stream_workspace_bytes(int64_t n_records, int64_t *bytes) {
    GUARD(mns::stream_workspace_bytes(n_records, bytes));
}

int mns_write_stream(const uint64_t *records, int64_t n_records, int32_t orig_w, int32_t orig_h, int32_t padded_w,
                     int32_t padded_h, int32_t mns, int32_t technique2, uint8_t *out, int64_t out_capacity,
                     int64_t *d_bits, void *workspace, int64_t workspace_bytes, void *stream) {
    GUARD(mns::write_stream(records, n_records, orig_w, orig_h, padded_w, padded_h, mns, technique2, out,
                            out_capacity, d_bits, workspace, workspace_bytes, (cudaStream_t)stream));
}

}  // extern "C"
