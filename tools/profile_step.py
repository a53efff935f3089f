#!/usr/bin/env python3
"""One bench step (prng_init + prng_generate(numiter), device only) with a fixed kernel
variant and no autotune -- a short target for ncu (--replay-mode application)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_01257_b200 as P  # noqa: E402

n = int(os.environ.get("PRNG_N", 1 << 24))
it = int(os.environ.get("PRNG_ITERS", 1000))
h = P.prng_create(n, 0)
P.prng_set_option(h, P.PRNG_OPT_KERNEL, int(os.environ.get("PRNG_KERNEL", 0)))
P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, int(os.environ.get("PRNG_SLOTS", 0)))
P.prng_set_option(h, P.PRNG_OPT_PIECE_ORDER, int(os.environ.get("PRNG_ORDER", 0)))
P.prng_set_option(h, P.PRNG_OPT_EPOCH_ITERS, int(os.environ.get("PRNG_EPOCH", 0)))
P.prng_init(h)
P.prng_generate(h, it)
P.prng_destroy(h)
