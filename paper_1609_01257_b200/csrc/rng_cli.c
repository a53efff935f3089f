/*
 * rng_b200 -- NEXT-1: the paper's example program on the B200 path (§5).
 *
 *   rng_b200 n i [--seed S] [--mode O2|O1|O3|S0|S1] [--batch T] [--device D]
 *                [--star] [--start K] [--profile] [--export FILE]
 *
 * "a standalone program which outputs random numbers in binary format to the standard
 * output ... The program accepts two parameters: a) n, the quantity of 64-bit (8-byte)
 * random values to generate per iteration; and, b) i, the number of iterations"
 * (P:151).  Exactly N = 8*n*i bytes (Eq. 1) of little-endian u64 go to stdout,
 * iteration-major (A8); everything else (usage, errors, the Fig. 3 profile summary with
 * --profile) goes to stderr, so the stream stays pipeable, e.g.
 *   ./rng_b200 16777216 10000 | dieharder -g 200 -a
 * The `out` block is the sink below: write(2) of each pinned batch while the next
 * batch is copied D2H and generated (host dual buffer, P:177 limitation 2).
 * Exit status: 0 ok, 1 runtime error (incl. a closed pipe), 2 usage error.
 */
#include <errno.h>
#include <signal.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include "prng.h"

static void usage(FILE *f) {
    fprintf(f,
            "usage: rng_b200 n i [--seed S] [--mode O2|O1|O3|S0|S1] [--batch T] [--device D]\n"
            "                [--star] [--start K] [--profile] [--export FILE]\n"
            "  --start K  resume: emit iterations K .. K+i-1 (GF(2) jump-ahead, no replay)\n"
            "  --star  xorshift64*-scrambled output (state * 0x2545F4914F6CDD1D)\n"
            "  n  64-bit random values per iteration (1 .. 2^32)\n"
            "  i  iterations (>= 1); writes 8*n*i bytes to stdout\n");
}

static int parse_u64(const char *s, uint64_t *out) {
    char *end = NULL;
    errno = 0;
    unsigned long long v = strtoull(s, &end, 0);
    if (errno || !end || *end || s[0] == '-') return -1;
    *out = (uint64_t)v;
    return 0;
}

/* `out`: write the batch to stdout (fd 1), retrying short writes. */
static int sink_stdout(void *user, uint64_t iter_begin, uint32_t iters, uint64_t gid_begin, uint64_t count,
                       const uint64_t *data) {
    (void)user;
    (void)iter_begin;
    (void)gid_begin;
    const char *p = (const char *)data;
    size_t left = (size_t)iters * (size_t)count * sizeof(uint64_t);
    while (left) {
        ssize_t w = write(1, p, left);
        if (w < 0) {
            if (errno == EINTR) continue;
            return 1; /* EPIPE etc.: abort generation */
        }
        p += w;
        left -= (size_t)w;
    }
    return 0;
}

int main(int argc, char **argv) {
    uint64_t n = 0, iters = 0, seed = 0, batch = 0, start = 0;
    int mode = PRNG_MODE_OVERLAP2, device = -1, profile = 0, npos = 0, star = 0;
    const char *export_path = NULL;
    for (int a = 1; a < argc; ++a) {
        const char *s = argv[a];
        if (!strcmp(s, "-h") || !strcmp(s, "--help")) {
            usage(stderr);
            return 0;
        } else if (!strcmp(s, "--seed") && a + 1 < argc) {
            if (parse_u64(argv[++a], &seed)) return usage(stderr), 2;
        } else if (!strcmp(s, "--start") && a + 1 < argc) {
            if (parse_u64(argv[++a], &start)) return usage(stderr), 2;
        } else if (!strcmp(s, "--batch") && a + 1 < argc) {
            if (parse_u64(argv[++a], &batch)) return usage(stderr), 2;
        } else if (!strcmp(s, "--device") && a + 1 < argc) {
            device = atoi(argv[++a]);
        } else if (!strcmp(s, "--mode") && a + 1 < argc) {
            const char *m = argv[++a];
            if (!strcmp(m, "S0")) mode = PRNG_MODE_SERIAL;
            else if (!strcmp(m, "S1")) mode = PRNG_MODE_PAGEABLE;
            else if (!strcmp(m, "O1")) mode = PRNG_MODE_OVERLAP1;
            else if (!strcmp(m, "O2")) mode = PRNG_MODE_OVERLAP2;
            else if (!strcmp(m, "O3")) mode = PRNG_MODE_ZEROCOPY;
            else return usage(stderr), 2;
        } else if (!strcmp(s, "--star")) {
            star = 1;
        } else if (!strcmp(s, "--profile")) {
            profile = 1;
        } else if (!strcmp(s, "--export") && a + 1 < argc) {
            export_path = argv[++a];
            profile = 1;
        } else if (s[0] != '-' && npos < 2) {
            if (parse_u64(s, npos == 0 ? &n : &iters)) return usage(stderr), 2;
            ++npos;
        } else {
            return usage(stderr), 2;
        }
    }
    if (npos != 2 || n < 1 || n > (1ull << 32) || iters < 1) {
        usage(stderr);
        return 2;
    }
    signal(SIGPIPE, SIG_IGN); /* a closed pipe surfaces as EPIPE -> sink abort */

    prng_err_t err = {0, {0}};
    prng_t *h = prng_create_range(n, seed, 0, n, device, &err);
    if (!h) {
        fprintf(stderr, "rng_b200: %s: %s\n", prng_strerror(err.code), err.msg);
        return 1;
    }
    int rc = prng_set_option(h, PRNG_OPT_MODE, mode, &err);
    if (!rc) rc = prng_set_option(h, PRNG_OPT_BATCH_ITERS, (int64_t)batch, &err);
    if (!rc) rc = prng_set_option(h, PRNG_OPT_PROFILE, profile, &err);
    if (!rc) rc = prng_set_option(h, PRNG_OPT_OUTPUT, star, &err);
    /* profiled runs keep the paper's separate init kernel, so the chart shows it (Fig. 5) */
    if (!rc && profile) rc = prng_set_option(h, PRNG_OPT_FUSED_SEED, 0, &err);
    if (!rc) rc = start ? prng_seek(h, start, &err) : prng_init(h, &err);
    if (!rc) rc = prng_generate(h, iters, sink_stdout, NULL, &err);
    if (rc) {
        fprintf(stderr, "rng_b200: %s: %s\n", prng_strerror(rc), err.msg);
        prng_destroy(h);
        return 1;
    }
    if (profile) {
        uint64_t ne = 0;
        double wall = 0;
        prng_prof_events(h, 0, NULL, NULL, NULL, &ne, &wall, &err);
        uint32_t *ids = (uint32_t *)malloc((ne ? ne : 1) * sizeof(uint32_t));
        double *st = (double *)malloc((ne ? ne : 1) * sizeof(double));
        double *en = (double *)malloc((ne ? ne : 1) * sizeof(double));
        if (ids && st && en && !prng_prof_events(h, ne, ids, st, en, &ne, &wall, &err)) {
            uint64_t len = 0;
            prng_prof_summary(ne, ids, st, en, PRNG_EV_NAMES, NULL, wall, PRNG_PROF_AGG_SORT_TIME | PRNG_PROF_SORT_DESC,
                              PRNG_PROF_OVERLAP_SORT_DURATION | PRNG_PROF_SORT_DESC, NULL, 0, &len, NULL);
            char *buf = (char *)malloc(len + 1);
            if (buf && !prng_prof_summary(ne, ids, st, en, PRNG_EV_NAMES, NULL, wall,
                                          PRNG_PROF_AGG_SORT_TIME | PRNG_PROF_SORT_DESC,
                                          PRNG_PROF_OVERLAP_SORT_DURATION | PRNG_PROF_SORT_DESC, buf, len + 1, &len,
                                          &err))
                fputs(buf, stderr);
            free(buf);
            if (export_path && prng_prof_export(ne, ids, st, en, PRNG_EV_NAMES, NULL, NULL, export_path, &err))
                fprintf(stderr, "rng_b200: export: %s\n", err.msg);
        }
        free(ids);
        free(st);
        free(en);
    }
    prng_destroy(h);
    return 0;
}
