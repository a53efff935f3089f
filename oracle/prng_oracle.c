/*
 * prng_oracle.c -- CPU ORACLE for the massive-PRNG hot path of
 * Fachada et al., "cf4ocl: a C framework for OpenCL" (arXiv 1609.01257), §5.
 *
 * THIS FILE IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *   Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 *   `--impl reference` legs may load, call or execute anything under oracle/.
 *   The CUDA product path (paper_1609_01257_b200/) shares no code, header,
 *   table or constant generator with this file and never calls it.
 *
 * It is the plain, slow, obviously correct definition of what the hot path
 * computes: single-threaded, scalar, flat loops, no blocking / fusion /
 * reordering beyond what the definition states.  Citations:
 *   P:<line> §<sec>  = /root/reference/PAPER.md line, section
 *   S:<line> <op>    = /root/reference/SPEC.md line, operation
 *   A<n>             = the reading adopted in DESIGN.md §3
 *
 * The definition:
 *   wang32(x)   = Wang's 32-bit integer hash ("[wang1997inthash]", A1)
 *   fmix64(z)   = 64-bit finaliser used only to premix the seed (A4)
 *   seed64(g,s) = (wang32(g ^ lo32(fmix64 s)) << 32)
 *               |  wang32(g ^ 0x9E3779B9 ^ hi32(fmix64 s)),  0 -> 1   (A2, A3, A4)
 *   xs(x)       = x ^= x<<13; x ^= x>>7; x ^= x<<17    (Marsaglia xor64, A5)
 *   out[0][g]   = seed64(g, s)                          ("first batch ... seeds", A6)
 *   out[k][g]   = xs(out[k-1][g]),  k = 1 .. numiter-1  (A6)
 *   stream      = for k: for g: 8 little-endian bytes of out[k][g]; 8*n*i bytes (Eq. 1; A8)
 *
 * Every function here is pinned by tests/test_oracle_pins.py against values
 * the paper, the cited sources or mathematics fix.
 */
#include <stdint.h>
#include <stdlib.h>

#define ORC_OK 0
#define ORC_EINVAL -1
#define ORC_ENOMEM -3

/* A1: Wang's 32-bit multiplicative integer hash, steps in the order of S:464:
 *   x = (x ^ 61) ^ (x >> 16); x = x * 9; x = x ^ (x >> 4);
 *   x = x * 0x27d4eb2d;       x = x ^ (x >> 15)      -- wrapping u32. */
uint32_t orc_wang32(uint32_t x)
{
    x = (x ^ 61u) ^ (x >> 16);
    x = x * 9u;
    x = x ^ (x >> 4);
    x = x * 0x27d4eb2du;
    x = x ^ (x >> 15);
    return x;
}

/* A4: seed premix (no paper counterpart: the paper's init kernel takes no seed,
 * P:252).  64-bit finaliser; fmix64(0) = 0 so seed 0 is the paper. */
uint64_t orc_fmix64(uint64_t z)
{
    z ^= z >> 33;
    z *= 0xff51afd7ed558ccdull;
    z ^= z >> 33;
    z *= 0xc4ceb9fe1a85ec53ull;
    z ^= z >> 33;
    return z;
}

/* a1 / P:173 "applying a hash function to the global ID of the associated
 * work-items"; A2 (two 32-bit hashes -> one 64-bit state), A3 (0 -> 1),
 * A4 (seed premix XORed into the hash keys). */
uint64_t orc_seed64(uint32_t gid, uint64_t seed)
{
    uint64_t m = orc_fmix64(seed);
    uint32_t a = (uint32_t)m;
    uint32_t b = (uint32_t)(m >> 32);
    uint64_t hi = (uint64_t)orc_wang32(gid ^ a);
    uint64_t lo = (uint64_t)orc_wang32(gid ^ 0x9E3779B9u ^ b);
    uint64_t st = (hi << 32) | lo;
    if (st == 0)
        st = 1;
    return st;
}

/* a2 / P:177 "a simple Xorshift PRNG [marsaglia2003xorshift]"; A5 triple
 * (13, 7, 17), left-right-left, on u64; A7 output = the new state. */
uint64_t orc_xorshift64(uint64_t x)
{
    x ^= x << 13;
    x ^= x >> 7;
    x ^= x << 17;
    return x;
}

/* Random-access form of the same definition: out[k][g] = xs^k(seed64(g, s)).
 * O(k) per value; used to check sampled outputs of large runs. */
uint64_t orc_sample(uint32_t gid, uint64_t k, uint64_t seed)
{
    uint64_t x = orc_seed64(gid, seed);
    for (uint64_t t = 0; t < k; ++t)
        x = orc_xorshift64(x);
    return x;
}

static int orc_check(uint64_t numrn, uint64_t numiter, uint64_t gid_begin, uint64_t count)
{
    /* A12: 1 <= numrn <= 2^32 (gid is a cl_uint), numiter >= 1. */
    if (numrn < 1 || numrn > (1ull << 32) || numiter < 1)
        return ORC_EINVAL;
    if (gid_begin > numrn || count > numrn - gid_begin)
        return ORC_EINVAL;
    return ORC_OK;
}

/* The flat loop of the definition (A6, A8): for k in 0..numiter-1,
 * for g in [gid_begin, gid_begin+count): s[g] = k ? xs(s[g]) : seed64(g, seed);
 * out[k*count + (g-gid_begin)] = s[g].  `out` holds numiter*count u64 (the host
 * is little-endian, so the array's bytes ARE the stream, A8). */
int orc_stream(uint64_t numrn, uint64_t numiter, uint64_t seed,
               uint64_t gid_begin, uint64_t count, uint64_t *out)
{
    int rc = orc_check(numrn, numiter, gid_begin, count);
    if (rc != ORC_OK)
        return rc;
    if (count == 0)
        return ORC_OK;
    uint64_t *s = (uint64_t *)malloc(count * sizeof(uint64_t));
    if (!s)
        return ORC_ENOMEM;
    for (uint64_t k = 0; k < numiter; ++k) {
        for (uint64_t j = 0; j < count; ++j) {
            uint32_t g = (uint32_t)(gid_begin + j);
            if (k == 0)
                s[j] = orc_seed64(g, seed);
            else
                s[j] = orc_xorshift64(s[j]);
            out[k * count + j] = s[j];
        }
    }
    free(s);
    return ORC_OK;
}

/* The same flat loop, folding each iteration's `count` outputs instead of storing them
 * (the large-run parity digests, SURVEY.md §8(c) "Parity procedure"), with every output
 * optional (NULL = not wanted):
 *   xor_out[k]  = XOR over g of out[k][g]
 *   sum_out[k]  = SUM over g of out[k][g]                mod 2^64
 *   wsum_out[k] = SUM over g of (2*g + 1) * out[k][g]    mod 2^64, g the GLOBAL gid --
 *                 position-weighted, so it changes when outputs swap places (the XOR and
 *                 the sum do not); the odd weights make each term a bijection of out[k][g]
 *   last_out[j] = out[numiter-1][gid_begin + j]          (the final state of the loop)
 * xor / sum / wsum hold numiter words, last_out count words. */
int orc_digest(uint64_t numrn, uint64_t numiter, uint64_t seed,
               uint64_t gid_begin, uint64_t count,
               uint64_t *xor_out, uint64_t *sum_out, uint64_t *wsum_out,
               uint64_t *last_out)
{
    int rc = orc_check(numrn, numiter, gid_begin, count);
    if (rc != ORC_OK)
        return rc;
    uint64_t *s = (uint64_t *)malloc((count ? count : 1) * sizeof(uint64_t));
    if (!s)
        return ORC_ENOMEM;
    for (uint64_t k = 0; k < numiter; ++k) {
        uint64_t fx = 0, fs = 0, fw = 0;
        for (uint64_t j = 0; j < count; ++j) {
            uint64_t gid = gid_begin + j;
            uint32_t g = (uint32_t)gid;
            if (k == 0)
                s[j] = orc_seed64(g, seed);
            else
                s[j] = orc_xorshift64(s[j]);
            fx ^= s[j];
            fs += s[j];
            fw += (2 * gid + 1) * s[j];
        }
        if (xor_out)
            xor_out[k] = fx;
        if (sum_out)
            sum_out[k] = fs;
        if (wsum_out)
            wsum_out[k] = fw;
    }
    if (last_out)
        for (uint64_t j = 0; j < count; ++j)
            last_out[j] = s[j];
    free(s);
    return ORC_OK;
}

/* NEXT-3 / A19: xorshift64*-style output scrambling on the same recurrence -- the emitted
 * value is the state times Vigna's xorshift64* multiplier M32 = 2685821657736338717
 * (0x2545F4914F6CDD1D), mod 2^64; P:177 (limitation 1) and P:358 ("a more complex PRNG
 * could probably be used instead").  Same flat loop as orc_stream. */
#define ORC_STAR_MUL 0x2545F4914F6CDD1Dull

uint64_t orc_star(uint64_t x) { return x * ORC_STAR_MUL; }

int orc_stream_star(uint64_t numrn, uint64_t numiter, uint64_t seed, uint64_t gid_begin, uint64_t count,
                    uint64_t *out)
{
    int rc = orc_check(numrn, numiter, gid_begin, count);
    if (rc != ORC_OK)
        return rc;
    if (count == 0)
        return ORC_OK;
    uint64_t *s = (uint64_t *)malloc(count * sizeof(uint64_t));
    if (!s)
        return ORC_ENOMEM;
    for (uint64_t k = 0; k < numiter; ++k) {
        for (uint64_t j = 0; j < count; ++j) {
            uint32_t g = (uint32_t)(gid_begin + j);
            if (k == 0)
                s[j] = orc_seed64(g, seed);
            else
                s[j] = orc_xorshift64(s[j]);
            out[k * count + j] = orc_star(s[j]);
        }
    }
    free(s);
    return ORC_OK;
}
