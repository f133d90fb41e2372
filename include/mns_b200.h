/*
 * mns_b200.h -- C ABI of libmns_b200.so, the B200 (sm_100a) implementation of the
 * MNS fractal coder's data-parallel core (arXiv 1501.02894; reference package
 * `mnscodec`, /root/reference/pkg/src/mnscodec).
 *
 * The reference has no native layer: its "plugin boundary" is the set of
 * module-level Python functions re-exported by mnscodec/__init__.py:9-53.
 * Each entry point below is what a maintainer binds (ctypes) in place of one
 * of those functions; the Python mirror paper_1501_02894_b200/codec.py does
 * exactly that and keeps the reference's signatures and error messages.
 *
 * Conventions
 *   - All buffers are caller-owned DEVICE pointers (e.g. torch tensors'
 *     data_ptr()); `stream` is a cudaStream_t cast to void* (NULL = legacy
 *     default stream).  Calls are asynchronous and stream-ordered; the library
 *     keeps no pointers after returning and holds no mutable global state.
 *   - Images are uint8, row-major, already padded (pad_to_multiple,
 *     image.py:123-132, is host work): width/height multiples of 16 for the
 *     quadtree, of B for the search baselines.
 *   - Return value: 0 on success, negative on a CUDA/argument error; the
 *     message is available from mns_last_error() (thread-local).  Reference
 *     ValueErrors are raised by the Python layer before any native call.
 *   - Transform codes travel as packed 64-bit leaf records (mns_record.h).
 */
#ifndef MNS_B200_H
#define MNS_B200_H

#include <stdint.h>

#include "mns_record.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Encoder knobs: mirror of EncoderConfig (encoder.py:52-76) plus the root-level
 * extension (root_level = 2: every 16x16 root is forced to split once, the
 * "8->4" quadtree of BASELINE configs 1 and 3). */
typedef struct {
    double e[3];      /* e1, e2, e3 (RMS tolerances of levels 1..3; +inf allowed) */
    double mean_tol;  /* phase-2 gate */
    int32_t mns;      /* 1: mode "mns"; 0: mode "no_search" */
    int32_t root_level;
    int32_t n_iso;    /* 1 (0): the reference; 8: phase 1 also tries the 8 isometries of the co-centred
                         domain (extension, BASELINE configs[1]; records carry the isometry, MNS_REC_ISO_SHIFT) */
    int32_t map_form; /* the decoder map mns_encode_quadtree emits into unit_map (mns_record.h):
                         0 = unit map (32 words per root), 1 = block map (8 words per root; the lattice decoders) */
} mns_enc_cfg;

/* Replaces: encoder.encode_quadtree (encoder.py:215-246) for n_images images of
 * identical size stacked at image_stride bytes, restricted to the root rows
 * [root_row_begin, root_row_end) of each image (strip sharding; pass 0 and
 * height/16 for whole images).  `img` points at row 0 of image 0 even when only
 * rows [root_row_begin*16 - 16, root_row_end*16 + 16) are resident (the rest is
 * never read).
 *
 * Output: packed records in reference DFS order (images, then roots in raster
 * order, then TL,TR,BL,BR pre-order), root_offsets[i] = index of the first
 * record of root i (roots of the processed rows, image-major, raster order;
 * n_roots + 1 entries, the last = total), *d_count = total records (device).
 * capacity must be >= 64 * n_roots.  unit_map (optional) receives the decoder's
 * map in cfg->map_form: the unit map (32 words per root) or the block map (8).  Workspace: mns_encode_workspace_bytes (64
 * staged record slots per root + the compaction scan state; two kernels: the
 * encoder, whose CTAs never wait on one another, then the scan + compaction). */
int mns_encode_workspace_bytes(int32_t width, int32_t n_images, int32_t root_row_begin, int32_t root_row_end,
                               int64_t *bytes);
int mns_encode_quadtree(const uint8_t *img, int32_t width, int32_t height, int64_t pitch, int64_t image_stride,
                        int32_t n_images, int32_t root_row_begin, int32_t root_row_end, const mns_enc_cfg *cfg,
                        uint64_t *records, int64_t capacity, int32_t *root_offsets, int64_t *d_count,
                        uint32_t *unit_map, void *workspace, int64_t workspace_bytes, void *stream);

/* Replaces: encoder.try_phase1 / try_phase2 (encoder.py:145-212), exported by
 * mnscodec/__init__.py:31-32: one node decision at (x, y) of size 32 >> level
 * (phase 1: levels 1..4, phase 2: levels 1..3).  *record (device) = the packed
 * leaf record, 0 on rejection; *rms (device) = the reference's rms -- phase 1:
 * rms_error of the quantised fit, phase 2: the worst chosen quadrant rms, or
 * +inf on rejection -- replayed in numpy's fp64 evaluation order (bit-exact).
 * One single-CTA launch; the image needs a 2(32 >> level) square co-centred
 * domain (phase 1). */
int mns_try_node(const uint8_t *img, int32_t width, int32_t height, int64_t pitch, int32_t x, int32_t y, int32_t level,
                 int32_t phase, const mns_enc_cfg *cfg, uint64_t *record, double *rms, void *stream);

/* The same with the record compaction (the second kernel) on compact_stream,
 * ordered after the encoder by an event: the unit map is complete when `stream`
 * reaches this point, the records / root_offsets / d_count only when
 * compact_stream does (so a decoder on `stream` overlaps the compaction).  The
 * workspace stays in use until compact_stream passes the compaction. */
int mns_encode_quadtree_split(const uint8_t *img, int32_t width, int32_t height, int64_t pitch, int64_t image_stride,
                              int32_t n_images, int32_t root_row_begin, int32_t root_row_end, const mns_enc_cfg *cfg,
                              uint64_t *records, int64_t capacity, int32_t *root_offsets, int64_t *d_count,
                              uint32_t *unit_map, void *workspace, int64_t workspace_bytes, void *stream,
                              void *compact_stream);

/* Decoder unit map (mns_record.h) of a record array grouped by root: 32 uint32
 * words (64 cells) per root of the root rows [root_row_begin, root_row_end).
 * mns_encode_quadtree emits the same map directly when unit_map != NULL.
 * mns_build_block_map: the block map (16 uint16 per root), as map_form = 1 emits it. */
int mns_build_unit_map(const uint64_t *records, const int32_t *root_offsets, int32_t width, int32_t root_row_begin,
                       int32_t root_row_end, uint32_t *unit_map, void *stream);
int mns_build_block_map(const uint64_t *records, const int32_t *root_offsets, int32_t width, int32_t root_row_begin,
                        int32_t root_row_end, uint16_t *block_map, void *stream);

/* Replaces: decoder.decode / decode_step (decoder.py:37-77) for quadtree codes.
 * One Jacobi sweep per iteration over an fp32 raster (ping/pong, width*height
 * floats each).  Records must be grouped by root with root_offsets (as
 * mns_encode_quadtree emits); leaf order inside a root is free, as in the
 * reference (decoder.py:8-10).  After `iters` sweeps (early stop when
 * stop_delta > 0 and max|delta| < stop_delta; *d_iters_done receives the count)
 * the raster is rounded floor(x+0.5), clipped to [0,255] into out (width*height
 * bytes, padded; the caller crops).  The final raster is in ping when
 * iters_done is even, else in pong -- except when out != NULL and stop_delta == 0:
 * then sweeps run two per pass (mns_decode_sweep2) and only out is defined. */
int mns_decode_workspace_bytes(int32_t width, int32_t height, int64_t *bytes);
int mns_decode_quadtree(const uint64_t *records, const int32_t *root_offsets, int32_t width, int32_t height,
                        int32_t iters, double stop_delta, float initial_value, float *ping, float *pong,
                        uint8_t *out, int32_t *d_iters_done, void *workspace, int64_t workspace_bytes,
                        void *stream);
/* mns_decode_unit_map: mns_decode_quadtree from the unit map of every root row (as
 * mns_encode_quadtree emits it with map_form = 0, or mns_build_unit_map builds it), skipping the map
 * build; workspace >= 64 bytes. */
int mns_decode_unit_map(const uint32_t *unit_map, int32_t width, int32_t height, int32_t iters, double stop_delta,
                        float initial_value, float *ping, float *pong, uint8_t *out, int32_t *d_iters_done,
                        void *workspace, int64_t workspace_bytes, void *stream);

/* One Jacobi sweep over the root rows [root_row_begin, root_row_end) (strip
 * sharding: the multi-GPU decoder exchanges 16-row halos between sweeps).
 * cur / nxt / out are bases of the FULL image (row 0) even when only rows
 * [16*root_row_begin - 16, 16*root_row_end + 16) are resident; the unit map is
 * local to the strip's roots.  cur holds values in [0, 255] (every sweep's
 * output does; the clip is elided when it provably cannot bind).  cur may be NULL on the first sweep: the flat
 * start raster of initial_value is implied (no fill pass).  nxt may be NULL when
 * out (uint8, rounded) is given: the fused final sweep.  state: 4 int32 zeroed
 * before the first sweep (early-stop bookkeeping when stop_delta > 0). */
int mns_decode_sweep(const uint32_t *unit_map, int32_t width, int32_t height, int32_t root_row_begin,
                     int32_t root_row_end, const float *cur, float initial_value, float *nxt, uint8_t *out,
                     int32_t *state, double stop_delta, void *stream);

/* Two sweeps t -> t+2 in one pass (stop_delta == 0 only): raster t is read once,
 * t+2 written once, t+1 stays on chip.  Rows [16*root_row_begin - 32,
 * 16*root_row_end + 32) of cur must be resident (32-row halo; exchanged once per
 * pass on the multi-GPU decoder).  unit_map holds the root rows starting at
 * unit_map_row_begin, which must cover [root_row_begin - 1, root_row_end + 1)
 * clipped to the image.  cur NULL = flat start raster, else values in [0, 255];
 * exactly one of nxt (fp32)
 * and out (rounded uint8, final pass) is non-NULL.  Same result as two
 * mns_decode_sweep calls. */
int mns_decode_sweep2(const uint32_t *unit_map, int32_t unit_map_row_begin, int32_t width, int32_t height,
                      int32_t root_row_begin, int32_t root_row_end, const float *cur, float initial_value, float *nxt,
                      uint8_t *out, void *stream);

/* Lattice-state decoding for codes WITHOUT 2x2 units (every leaf side >= 4, e.g.
 * the 16->8->4 quadtree, e3 = inf).  Such a code reads the previous raster only
 * through its even 2x2-sum lattice (image.py:160-171 downsample_mean2 order), so
 * the state between passes is that lattice: (height/2) rows of width/2 floats,
 * each row de-interleaved (the width/4 even lattice columns, then the odd ones),
 * a quarter of the raster's bytes with bit-identical values -- the decoded image
 * equals the raster path's bit for bit.  *d_error (device int32, zeroed by the
 * caller) is set to 1 if a 2x2 unit is met (the output is then undefined; use
 * the raster path).
 *
 * The lattice decoders read the BLOCK map (mns_record.h: one descriptor per 4x4
 * block, 16 uint16 per root; a quarter of the unit map's bytes), with the same
 * root-row conventions as the unit map of mns_decode_sweep2.
 *
 * mns_decode_pass_lattice: two sweeps t -> t+2 (as mns_decode_sweep2; lattice
 * rows [8*root_row_begin - 16, 8*root_row_end + 16) of cur_lattice resident,
 * 16-byte aligned; cur_lattice NULL = flat start; exactly one of nxt_lattice
 * and out).  mns_decode_flat_lattice: the single first sweep from the flat
 * raster, written as lattice (odd sweep counts; nxt_lattice) or, for a one-sweep
 * decode, as the rounded uint8 image (out; exactly one of the two).
 * mns_decode_quadtree_lattice:
 * the whole decode (stop_delta = 0) into the uint8 image, as mns_decode_quadtree
 * with out != NULL; lat_ping / lat_pong hold (height/2)*(width/2) floats each. */
int mns_decode_pass_lattice(const uint16_t *block_map, int32_t block_map_row_begin, int32_t width, int32_t height,
                            int32_t root_row_begin, int32_t root_row_end, const float *cur_lattice, float initial_value,
                            float *nxt_lattice, uint8_t *out, int32_t *d_error, void *stream);
int mns_decode_flat_lattice(const uint16_t *block_map, int32_t block_map_row_begin, int32_t width, int32_t height,
                            int32_t root_row_begin, int32_t root_row_end, float initial_value, float *nxt_lattice,
                            uint8_t *out, void *stream);
int mns_decode_quadtree_lattice(const uint64_t *records, const int32_t *root_offsets, int32_t width, int32_t height,
                                int32_t iters, float initial_value, float *lat_ping, float *lat_pong, uint8_t *out,
                                int32_t *d_error, void *workspace, int64_t workspace_bytes, void *stream);
/* mns_decode_unit_map_lattice: mns_decode_quadtree_lattice from the block map of every root row (as
 * mns_encode_quadtree emits it with map_form = 1), skipping the map build; workspace >= 64 bytes. */
int mns_decode_unit_map_lattice(const uint16_t *block_map, int32_t width, int32_t height, int32_t iters,
                                float initial_value, float *lat_ping, float *lat_pong, uint8_t *out, int32_t *d_error,
                                void *workspace, int64_t workspace_bytes, void *stream);

/* Generic painted units (decoder.py:32-34 _paint): destination square (x, y, size),
 * domain origin (dx, dy) of the 2*size domain, map (s, o).  usize = side | isometry << 8: the
 * isometry extension paints d_t(i, j) = d(src_t(i, j)) (0 = identity, the reference).  Used for search-
 * baseline codes whose domains are explicit (BaselinePayload) and for arbitrary
 * leaf orders.  Units are SoA arrays of length n_units. */
int mns_decode_units(const int32_t *ux, const int32_t *uy, const int32_t *usize, const int32_t *udx,
                     const int32_t *udy, const float *us, const float *uo, int64_t n_units, int32_t width,
                     int32_t height, int32_t iters, double stop_delta, float initial_value, float *ping,
                     float *pong, uint8_t *out, int32_t *d_iters_done, void *workspace, int64_t workspace_bytes,
                     void *stream);

/* One sweep on a caller-provided fp64 raster, bit-exact with decoder.decode_step
 * (numpy evaluation order emulated; for parity tests and debugging). */
int mns_decode_step_f64(const int32_t *ux, const int32_t *uy, const int32_t *usize, const int32_t *udx,
                        const int32_t *udy, const double *us, const double *uo, int64_t n_units, int32_t width,
                        int32_t height, const double *cur, double *out, void *stream);

/* Replaces: decoder.decode (decoder.py:66-77) EXACTLY, including the early stop: every sweep is
 * the bit-exact fp64 step above, the sweep's max|nxt - current| is an exact fp64 max, and the
 * stop test `delta < stop_delta` runs on the device (later sweeps are no-ops), so the sweep count
 * and the uint8 image (clip(floor(x + 0.5))) equal the reference's bit for bit.  Used for
 * stop_delta > 0 (the default DecodeConfig); the fp32 decoders serve stop_delta = 0.  ping/pong:
 * fp64 [height][width]; *d_iters_done = sweeps run; workspace >= 64 bytes (with 32..63 bytes the
 * one-launch path for small images is not taken).  Images of up to 2^21 pixels decode in ONE
 * cooperative launch (fill, sweeps, stop decisions, uint8 image), larger ones in a launch chain. */
int mns_decode_f64(const int32_t *ux, const int32_t *uy, const int32_t *usize, const int32_t *udx,
                   const int32_t *udy, const double *us, const double *uo, int64_t n_units, int32_t width,
                   int32_t height, int32_t max_iters, double stop_delta, double initial_value, double *ping,
                   double *pong, uint8_t *out, int32_t *d_iters_done, void *workspace, int64_t workspace_bytes,
                   void *stream);

/* The building blocks of mns_decode_f64 for strip sharding (decoder.py:70-75 per rank, the delta
 * all-reduced between mns_decode_f64_sweep and mns_decode_f64_decide).  state: int64[4] zeroed by
 * the caller ([0] converged, [1] sweeps done, [2] the sweep's max|delta| as fp64 bits).  cur/nxt
 * may be "virtual global" base pointers (row 0 of the image) of resident strips.
 * mns_records_to_units expands n packed records into 4n unit slots (decoder.py:48-59): slot i is
 * record i's first unit (the leaf itself, or quadrant 0 of a phase-2 record), slots n + 3i .. + 2
 * its quadrants 1..3; unused slots get size 0 and are skipped.  The order of a unit list does not
 * matter to the sweeps (units are disjoint); this one keeps the live units of a mostly phase-1
 * code dense. */
int mns_records_to_units(const uint64_t *records, int64_t n_records, int32_t width, int32_t height, int32_t *ux,
                         int32_t *uy, int32_t *usize, int32_t *udx, int32_t *udy, double *us, double *uo,
                         void *stream);
int mns_decode_f64_sweep(const int32_t *ux, const int32_t *uy, const int32_t *usize, const int32_t *udx,
                         const int32_t *udy, const double *us, const double *uo, int64_t n_units, int32_t width,
                         const double *cur, double *nxt, int64_t *state, void *stream);
int mns_decode_f64_decide(int64_t *state, double stop_delta, void *stream);
int mns_decode_f64_finalize(const double *ping, const double *pong, const int64_t *state, int32_t width,
                            int32_t row_begin, int32_t row_end, uint8_t *out, int32_t *d_iters_done, void *stream);

/* Replaces: encoder.encode_full_search (encoder.py:249-309).  Ranges: the
 * non-overlapping B x B blocks of the B-padded raster in raster order (range
 * ids [range_begin, range_end) -- range sharding).  Domain pool: every 2B x 2B
 * block on a stride-`step` lattice, raster order, x n_iso isometries (1 = the
 * reference; 8 = extension, order documented in DESIGN.md).  Per range:
 * out_dom = domain index, out_iso, out_o = o_byte, out_code = s_code, with the
 * reference's tie-break (lowest domain index, then isometry).  B in {4, 8}
 * runs on the tcgen05 tensor-core path; B in {2, 16} on CUDA cores. */
int mns_search_workspace_bytes(int32_t width, int32_t height, int32_t B, int32_t step, int32_t n_iso,
                               int64_t *bytes);
int mns_full_search(const uint8_t *img, int32_t width, int32_t height, int32_t B, int32_t step, int32_t n_iso,
                    int32_t range_begin, int32_t range_end, int32_t *out_dom, int8_t *out_iso, uint8_t *out_o,
                    uint8_t *out_code, void *workspace, int64_t workspace_bytes, void *stream);

/* Replaces: encoder.encode_local_search (encoder.py:312-347); radius 4 and n_iso 1 are the
 * reference (81 candidates), other radii (up to 32) and n_iso = 8 (the isometries of
 * mns_full_search, ties to the lowest candidate then isometry) are the extension.  Outputs the
 * winning domain origin (and isometry; out_iso may be NULL) per 8x8 range of the 8-padded raster. */
int mns_local_search(const uint8_t *img, int32_t width, int32_t height, int32_t radius, int32_t n_iso,
                     int32_t *out_dx, int32_t *out_dy, int8_t *out_iso, uint8_t *out_o, uint8_t *out_code,
                     void *stream);

/* The same local search as a windowed GEMM on the tcgen05 full-search pipeline: only the (range
 * tile, domain tile) pairs that meet some window are multiplied, elements outside a row's window are
 * masked, and the winners are decided by the same exact keys (bit-identical to mns_local_search).
 * Workspace: mns_local_search_workspace_bytes.  MNS_LOCAL_CUDA_CORES=1 in the environment routes to
 * the CUDA-core kernel (A/B checks). */
int mns_local_search_workspace_bytes(int32_t width, int32_t height, int32_t radius, int32_t n_iso, int64_t *bytes);
int mns_local_search_tc(const uint8_t *img, int32_t width, int32_t height, int32_t radius, int32_t n_iso,
                        int32_t *out_dx, int32_t *out_dy, int8_t *out_iso, uint8_t *out_o, uint8_t *out_code,
                        void *workspace, int64_t workspace_bytes, void *stream);

/* Packed .mns bitstream (bitstream.py:130-205) of a record array: per-leaf
 * widths, exclusive scan, MSB-first scatter.  out must hold
 * 4*ceil((104 + 33n)/32) bytes; *d_bits receives the exact bit count
 * (stream_bit_count, bitstream.py:282-300). */
int mns_stream_workspace_bytes(int64_t n_records, int64_t *bytes);
int mns_write_stream(const uint64_t *records, int64_t n_records, int32_t orig_w, int32_t orig_h, int32_t padded_w,
                     int32_t padded_h, int32_t mns, int32_t technique2, uint8_t *out, int64_t out_capacity,
                     int64_t *d_bits, void *workspace, int64_t workspace_bytes, void *stream);

/* .mns reader (bitstream.py:208-279 read_stream) for the leaf body of a
 * container whose 13-byte header the caller has validated (mns / technique2 flags, padded
 * dimensions).  Parallel token parse (per-chunk exit tables); writes records in DFS order (capacity >=
 * 64 * n_roots), root_offsets[n_roots + 1] and *d_count.  d_status[0] = first format error
 * as a key (bit position << 16 | code << 8 | a << 4 | b; -1 = none; codes: 1 level-a leaf
 * inside a level-b node, 2 quartet interrupted by a level-a id, 3 negative-zero delta,
 * 4 truncated), d_status[1] = bit position after the final leaf (-1 if the stream ended
 * before every root was tiled).  Trailing / padding checks are the caller's.  Asynchronous
 * (no host round trip). */
int mns_read_stream_workspace_bytes(int64_t n_bytes, int64_t *bytes);
int mns_read_stream(const uint8_t *data, int64_t n_bytes, int32_t mns, int32_t technique2, int32_t padded_w,
                    int32_t padded_h, uint64_t *records, int64_t capacity, int32_t *root_offsets, int64_t *d_count,
                    int64_t *d_status, void *workspace, int64_t workspace_bytes, void *stream);

/* Rate-distortion metrics on device (bench.py:39-79 rd_sweep):
 * exact sum of squared differences of two W x H uint8 images (metrics.py:16-31
 * mse = sse / (W*H)), and the leaf tallies of a record array (encoder.py:135-142):
 * out6 = {level-1, level-2, level-3, level-4 leaves, phase-2 leaves, leaves painted
 * as 2x2 units (level 4 and level-3 phase 2: a code with none can be decoded on
 * lattice state, mns_decode_pass_lattice)}. */
int mns_image_sse(const uint8_t *a, int64_t pitch_a, const uint8_t *b, int64_t pitch_b, int32_t width, int32_t height,
                  uint64_t *d_sse, void *stream);
int mns_code_stats(const uint64_t *records, int64_t n_records, int64_t *d_out6, void *stream);

/* Domain-offset histogram of a full-search result (bench.py:119-127 offset_histogram
 * over the samples of encoder.py:249-309): offset = domain centre - range centre
 * of each of the (W/B)*(H/B) ranges; dense int32 counts hist_x[dx + W] (2W+1),
 * hist_y[dy + H] (2H+1) and joint[(dy + H)*(2W+1) + dx + W]. */
int mns_offset_histogram(const int32_t *dom, int64_t n_ranges, int32_t width, int32_t height, int32_t range_size,
                         int32_t step, int32_t *hist_x, int32_t *hist_y, int32_t *joint, void *stream);

const char *mns_last_error(void);
int mns_version(void);

#ifdef __cplusplus
}
#endif

#endif
