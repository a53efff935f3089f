#!/usr/bin/env python3
"""Round-2 probe target for ncu --print-metric-instances values: one bench-shape step of the
generator (2^24 x ITERS, the default "auto" kernel) and one run of the one-shot fill kernel
(prng_probe_fill_gbs, 8 GiB), so the per-DRAM-channel activity of the two can be compared."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1609_01257_b200 as P  # noqa: E402

it = int(os.environ.get("PRNG_ITERS", 200))
h = P.prng_create(1 << 24, 0)
P.prng_init(h)
P.prng_generate(h, it)
P.prng_destroy(h)
print("fill", P.prng_probe_fill_gbs(8 << 30, 1))
