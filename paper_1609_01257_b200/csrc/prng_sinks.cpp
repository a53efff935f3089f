// prng_sinks.cpp -- the built-in sinks of include/prng_sinks.h (the paper's `out`).
#include <cstdint>
#include <cstring>

#include "../../include/prng_sinks.h"

extern "C" {

// ---------------------------------------------------------------------------- built-in sinks
int prng_sink_null(void *, uint64_t, uint32_t, uint64_t, uint64_t, const uint64_t *) { return 0; }

int prng_sink_copy(void *user, uint64_t iter_begin, uint32_t iters, uint64_t gid_begin, uint64_t count,
                   const uint64_t *data) {
    prng_copy_sink_t *c = (prng_copy_sink_t *)user;
    // the batch's gid columns must fit the caller's rows: [gid_offset, gid_offset + dst_pitch)
    if (gid_begin < c->gid_offset || gid_begin - c->gid_offset > c->dst_pitch ||
        count > c->dst_pitch - (gid_begin - c->gid_offset))
        return 1;
    // ... and its iterations the caller's rows: [iter_offset, iter_offset + iters)
    if (iter_begin < c->iter_offset || iter_begin - c->iter_offset > c->iters ||
        iters > c->iters - (iter_begin - c->iter_offset))
        return 1;
    for (uint32_t t = 0; t < iters; ++t) {
        const uint64_t k = iter_begin + t;
        std::memcpy(c->dst + (k - c->iter_offset) * c->dst_pitch + (gid_begin - c->gid_offset), data + t * count,
                    count * sizeof(uint64_t));
    }
    return 0;
}

int prng_sink_digest(void *user, uint64_t iter_begin, uint32_t iters, uint64_t gid_begin, uint64_t count,
                     const uint64_t *data) {
    prng_digest_sink_t *d = (prng_digest_sink_t *)user;
    for (uint32_t t = 0; t < iters; ++t) {
        const uint64_t k = iter_begin + t;
        if (k < d->iter_offset || k - d->iter_offset >= d->iters) return 1;
        uint64_t x = 0, s = 0, w = 0;
        const uint64_t *row = data + (uint64_t)t * count;
        for (uint64_t j = 0; j < count; ++j) {
            x ^= row[j];
            s += row[j];
            w += (2 * (gid_begin + j) + 1) * row[j];
        }
        d->xor_out[k - d->iter_offset] ^= x;
        d->sum_out[k - d->iter_offset] += s;
        if (d->wsum_out) d->wsum_out[k - d->iter_offset] += w;
    }
    return 0;
}

}  // extern "C"
