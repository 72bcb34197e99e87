/*
 * mec_synth.h -- device-side synthetic input generator (bench / test helper,
 * not part of the MEC method).  It evaluates, in its own CUDA kernel, the
 * same counter-based formula as the host generator synth/__init__.py:
 *
 *   z = splitmix64(seed ^ (tensor_id << 56) ^ (index_offset + i))
 *   GRID8  : v = (int8)(z >> 56) / 128        (exact in bf16)
 *   GRID11 : v = ((z >> 53) - 1024) / 1024    (exact in tf32)
 *   FULL24 : v = ((z >> 40) - 2^23) / 2^23
 *
 * and stores v as bf16 (out_dtype = MEC_DTYPE_BF16, round-to-nearest-even,
 * exact for GRID8) or fp32 (MEC_DTYPE_TF32).  `dst` is a device pointer of
 * `count` elements owned by the caller; the fill is enqueued on `stream`.
 * Returns MEC_ERR_INVALID_ARG for a NULL dst, negative count or bad kind.
 */
#ifndef MEC_SYNTH_H
#define MEC_SYNTH_H
#include "mec.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { MEC_SYNTH_GRID8 = 0, MEC_SYNTH_GRID11 = 1, MEC_SYNTH_FULL24 = 2 } mec_synth_kind_t;

mec_status_t mec_synth_fill(void* dst, int64_t count, uint64_t seed, int tensor_id,
                            uint64_t index_offset, int kind, mec_dtype_t out_dtype,
                            void* stream);

/* L2 flush helper, on `stream`: overwrites the first half of the device
 * scratch buffer `scratch` (`bytes` >= 4x the L2 size), then reads its second
 * half.  The write evicts everything the previous step left in L2; the read
 * then evicts the write's own dirty lines (their write-back happens here, not
 * inside the next timed step), so the timed step starts with an L2 holding
 * only clean lines of `scratch`.  MEC_ERR_INVALID_ARG for a NULL scratch. */
mec_status_t mec_l2_flush(void* scratch, size_t bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif
