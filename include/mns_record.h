/* Packed 64-bit transform-code leaf record shared by the CUDA library and the
 * CPU oracle (test infrastructure).  One record = one reference `LeafRecord`
 * of a no_search / mns code (reference: pkg/src/mnscodec/encoder.py:79-117).
 *
 *   bits  0..14  x / 2          (range x, 15 bits; padded width <= 65534)
 *   bits 15..29  y / 2
 *   bits 30..31  level - 1      (1..4 -> 0..3; block size = 32 >> level)
 *   bit  32      phase2 flag    (Phase2Payload when set, Phase1Payload else)
 *   bits 33..40  o_byte         (u8)
 *   phase 1:  bits 41..43  s_code (0..7)
 *   phase 2:  bits 41..46  delta0 (6-bit two's complement, |d| <= 31)
 *             bits 47..52  delta1
 *             bits 53..58  delta2
 *             bits 59..62  s_bits (TL, TR, BL, BR -> bit 59, 60, 61, 62)
 *   bit 63 reserved (0)
 */
#ifndef MNS_RECORD_H
#define MNS_RECORD_H

#include <stdint.h>

#define MNS_REC_X_SHIFT 0
#define MNS_REC_Y_SHIFT 15
#define MNS_REC_LEVEL_SHIFT 30
#define MNS_REC_PHASE2_SHIFT 32
#define MNS_REC_O_SHIFT 33
#define MNS_REC_PAYLOAD_SHIFT 41
/* extension: the isometry (0..7, 0 = identity) of a phase-1 leaf's domain (n_iso = 8 encodes) */
#define MNS_REC_ISO_SHIFT 44

#ifdef __CUDACC__
#define MNS_REC_INLINE __host__ __device__ static inline
#else
#define MNS_REC_INLINE static inline
#endif

MNS_REC_INLINE uint64_t mns_rec_phase1(int x, int y, int level, int o_byte, int s_code) {
    return ((uint64_t)(x >> 1) << MNS_REC_X_SHIFT) | ((uint64_t)(y >> 1) << MNS_REC_Y_SHIFT) |
           ((uint64_t)(level - 1) << MNS_REC_LEVEL_SHIFT) | ((uint64_t)(o_byte & 0xFF) << MNS_REC_O_SHIFT) |
           ((uint64_t)(s_code & 7) << MNS_REC_PAYLOAD_SHIFT);
}

MNS_REC_INLINE uint64_t mns_rec_phase2(int x, int y, int level, int o_byte, int d0, int d1, int d2, int s_bits) {
    return ((uint64_t)(x >> 1) << MNS_REC_X_SHIFT) | ((uint64_t)(y >> 1) << MNS_REC_Y_SHIFT) |
           ((uint64_t)(level - 1) << MNS_REC_LEVEL_SHIFT) | ((uint64_t)1 << MNS_REC_PHASE2_SHIFT) |
           ((uint64_t)(o_byte & 0xFF) << MNS_REC_O_SHIFT) |
           ((uint64_t)(d0 & 63) << 41) | ((uint64_t)(d1 & 63) << 47) | ((uint64_t)(d2 & 63) << 53) |
           ((uint64_t)(s_bits & 15) << 59);
}

/* Unit map (decoder input): one uint16 per 2x2 cell of every 16x16 root, 64 per
 * root in Morton (= DFS) order, roots in raster order.  A cell names the painted
 * unit covering it (decoder.py:48-62: a phase-1 leaf, or one quadrant of a
 * phase-2 leaf):
 *   bits  0..3   contrast index: 0..7 phase-1 code k (s = -0.875 + 0.25k);
 *                8 + 2*(level-1) + bit for a phase-2 quadrant (CONTRAST_SETS)
 *   bits  4..13  luminance target + 32 (phase-2 targets span -31..286)
 *   bits 14..15  log2(unit side) - 1 (side 2, 4, 8, 16)
 * The unit's origin is the cell position rounded down to the side; its domain is
 * the co-centred one (image.py:174-187).
 *
 * Block map (lattice decoders): one uint16 per 4x4 block, 16 per root in Morton
 * order, = the unit-map descriptor of the block's first cell.  A unit of side
 * >= 4 is aligned to its side, so it covers whole blocks and the four cells of a
 * block share its descriptor; a block holding 2x2 units carries side bits 0
 * (the lattice decoders flag it). */
MNS_REC_INLINE uint16_t mns_unit_desc(int s_index, int target, int side_log2) {
    return (uint16_t)((s_index & 15) | ((target + 32) << 4) | ((side_log2 - 1) << 14));
}

/* Descriptor of the unit covering root-relative pixel (px, py) (even) of leaf record r. */
MNS_REC_INLINE uint16_t mns_unit_of_record(uint64_t r, int rx, int ry, int px, int py) {
    const int x = (int)((r >> MNS_REC_X_SHIFT) & 0x7FFF) * 2 - rx, y = (int)((r >> MNS_REC_Y_SHIFT) & 0x7FFF) * 2 - ry;
    const int level = (int)((r >> MNS_REC_LEVEL_SHIFT) & 3) + 1;
    const int lg = 5 - level; /* side = 32 >> level */
    const int o = (int)((r >> MNS_REC_O_SHIFT) & 0xFF);
    if (!((r >> MNS_REC_PHASE2_SHIFT) & 1)) return mns_unit_desc((int)((r >> MNS_REC_PAYLOAD_SHIFT) & 7), o, lg);
    const int h = 1 << (lg - 1);
    const int q = ((py - y) >= h ? 2 : 0) + ((px - x) >= h ? 1 : 0);
    int d[3];
    for (int j = 0; j < 3; j++) {
        const int f = (int)((r >> (41 + 6 * j)) & 63);
        d[j] = f >= 32 ? f - 64 : f;
    }
    const int t = q < 3 ? o + d[q] : o - (d[0] + d[1] + d[2]);
    const int bit = (int)((r >> (59 + q)) & 1);
    return mns_unit_desc(8 + 2 * (level - 1) + bit, t, lg - 1);
}

/* Both descriptors of the horizontally adjacent cells (px, py) and (px + 2, py) (px a multiple of
 * 4) of one leaf record r of side >= 4, packed low | high << 16: the record's fields are decoded
 * once (the encoder's emission, a lane's two cells). */
MNS_REC_INLINE uint32_t mns_unit_pair_of_record(uint64_t r, int rx, int ry, int px, int py) {
    const int level = (int)((r >> MNS_REC_LEVEL_SHIFT) & 3) + 1;
    const int lg = 5 - level;
    const int o = (int)((r >> MNS_REC_O_SHIFT) & 0xFF);
    if (!((r >> MNS_REC_PHASE2_SHIFT) & 1)) {
        const uint32_t d = mns_unit_desc((int)((r >> MNS_REC_PAYLOAD_SHIFT) & 7), o, lg);
        return d | (d << 16);
    }
    const int x = (int)((r >> MNS_REC_X_SHIFT) & 0x7FFF) * 2 - rx, y = (int)((r >> MNS_REC_Y_SHIFT) & 0x7FFF) * 2 - ry;
    const int h = 1 << (lg - 1);
    const int qy = (py - y) >= h ? 2 : 0;
    int d[3];
    for (int j = 0; j < 3; j++) {
        const int f = (int)((r >> (41 + 6 * j)) & 63);
        d[j] = f >= 32 ? f - 64 : f;
    }
    uint32_t out = 0;
    for (int c = 0; c < 2; c++) {
        const int q = qy + ((px + 2 * c - x) >= h ? 1 : 0);
        const int t = q < 3 ? o + d[q] : o - (d[0] + d[1] + d[2]);
        const int bit = (int)((r >> (59 + q)) & 1);
        out |= (uint32_t)mns_unit_desc(8 + 2 * (level - 1) + bit, t, lg - 1) << (16 * c);
    }
    return out;
}

#endif
