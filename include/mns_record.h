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

#endif
