/*
 * prng_sinks.h -- built-in sinks for prng_generate() (the paper's `out` block, P:164,
 * P:169), usable directly as the `sink` argument with the matching `user` struct.
 *
 *  prng_sink_null   -- discards the data.  The paper's measurements redirect stdout to
 *                      the null device, so this is the benchmark sink.
 *  prng_sink_copy   -- copies each iteration row into a caller-owned host array
 *                      dst[(k - iter_offset) * dst_pitch + (gid - gid_offset)].
 *                      Returns nonzero (abort), writing nothing, if an iteration of
 *                      the batch falls outside [iter_offset, iter_offset + iters) or a
 *                      gid outside [gid_offset, gid_offset + dst_pitch).
 *  prng_sink_digest -- folds each iteration row into xor_out[k - iter_offset] ^= XOR(row),
 *                      sum_out[k - iter_offset] += SUM(row) and (if wsum_out != NULL)
 *                      wsum_out[k - iter_offset] += SUM over gids g of (2 g + 1) row[g]
 *                      (mod 2^64, g the GLOBAL gid: a position-weighted fold that changes
 *                      when outputs swap places); all folds are associative, so per-rank
 *                      digests combine by XOR / + across gid shards (the large-run parity
 *                      check).  The caller zero-initialises the arrays.
 */
#ifndef PRNG_B200_SINKS_H
#define PRNG_B200_SINKS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct prng_copy_sink {
    uint64_t *dst;          /* host array, >= iters * dst_pitch u64 */
    uint64_t dst_pitch;     /* u64 elements per iteration row        */
    uint64_t iter_offset;   /* iteration stored in row 0             */
    uint64_t iters;         /* rows available                        */
    uint64_t gid_offset;    /* gid stored in column 0                */
} prng_copy_sink_t;

typedef struct prng_digest_sink {
    uint64_t *xor_out;      /* [iters], zero-initialised by the caller */
    uint64_t *sum_out;      /* [iters], zero-initialised by the caller */
    uint64_t iter_offset;
    uint64_t iters;
    uint64_t *wsum_out;     /* [iters] or NULL, zero-initialised by the caller */
} prng_digest_sink_t;

int prng_sink_null(void *user, uint64_t iter_begin, uint32_t iters, uint64_t gid_begin, uint64_t count,
                   const uint64_t *data);
int prng_sink_copy(void *user, uint64_t iter_begin, uint32_t iters, uint64_t gid_begin, uint64_t count,
                   const uint64_t *data);
int prng_sink_digest(void *user, uint64_t iter_begin, uint32_t iters, uint64_t gid_begin, uint64_t count,
                     const uint64_t *data);

#ifdef __cplusplus
}
#endif
#endif /* PRNG_B200_SINKS_H */
