/*
 * prng_probes.h -- same-box roofline probes (SURVEY.md §8(d) "Denominators"), exported by
 * libprng_probes.so, a library of its own next to libprng_b200.so.
 *
 * Measurement infrastructure for bench.py, not the hot path: the probes run the memory
 * system and the host link with the kernels and copies below, and report GB/s.  They share
 * no code with the generator (libprng_b200.so) and never touch a prng_t handle.  Each call
 * allocates its buffer on the current CUDA device, times `reps` runs after one warm-up, and
 * frees the buffer.  A return value < 0 means a CUDA error (allocation, launch or sync).
 */
#ifndef PRNG_PROBES_H
#define PRNG_PROBES_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same-box denominators, for bench.py: each returns GB/s or < 0 on
 * error; `bytes` is the buffer size.  The store kernels write pseudo-random
 * (incompressible) data, like the generator. */
double prng_probe_memset_gbs(uint64_t bytes, int reps);  /* cudaMemsetAsync (copy engine), best of reps */
/* The same fill repeated `reps` times back to back, timed as one interval (sustained,
 * power-capped write rate of the fill engine). */
double prng_probe_memset_sustained_gbs(uint64_t bytes, int reps);
double prng_probe_store_gbs(uint64_t bytes, int reps);   /* persistent grid-stride 32-B store sweep */
/* One-shot grid of 128-thread CTAs, each writing one contiguous 16 KiB chunk with 32-B
 * stores (a framework fill kernel's structure): the fastest SM write pattern measured. */
double prng_probe_fill_gbs(uint64_t bytes, int reps);
/* Pinned (or pageable) cudaMemcpyAsync D2H over `nstreams` streams, best of `reps`. */
double prng_probe_d2h_gbs(uint64_t bytes, int reps, int pinned, int nstreams);
/* `reps` pinned D2H copies back to back timed as one interval: each rank's sustained share
 * of the host links when all ranks of a node run it at once (bench.py, N > 1). */
double prng_probe_d2h_sustained_gbs(uint64_t bytes, int reps);

#ifdef __cplusplus
}
#endif
#endif /* PRNG_PROBES_H */
