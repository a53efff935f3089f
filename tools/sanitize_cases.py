#!/usr/bin/env python3
"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck): every kernel
family (natural order with the .aligned / non-.aligned barrier, ping-pong loop,
time-parallel jump-ahead, epoch order, the anti-absorption substitution, star output,
zero-copy), checked against the oracle.  Run from the repo root on a GPU box:
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_1609_01257_b200 as P  # noqa: E402

names = [P.prng_kernel_variant_name(i) for i in range(P.prng_kernel_variants())]
cases = [  # (n, iters, variant, mode, output, device-ring slots, PRNG_OPT_EPOCH_ITERS)
    (1000, 600, "v2n4s1", P.PRNG_MODE_OVERLAP2, 0, 1000, 0),  # time-parallel chunks
    (1000, 600, "v2n4s1", P.PRNG_MODE_OVERLAP2, 0, 16, 0),    # wrapping ring: epoch order, E = 16
    (1003, 9, "v4n4s1", P.PRNG_MODE_OVERLAP1, 1, 16, 0),      # star output, ragged n
    (4100, 7, "v4n4s1p", P.PRNG_MODE_SERIAL, 0, 16, 0),       # ping-pong hot loop
    (4096, 6, "v2n4s1", P.PRNG_MODE_ZEROCOPY, 0, 16, 0),      # zero-copy
    (70001, 40, "auto", P.PRNG_MODE_OVERLAP2, 1, 16, 7),      # forced epochs, star, ragged
    (1 << 20, 70, "auto", P.PRNG_MODE_OVERLAP2, 0, 64, 0),    # anti-absorption: v2n32s1
    (300000, 9, "v4n8s1a", P.PRNG_MODE_OVERLAP2, 0, 16, 0),   # .aligned barrier in uniform rounds
    (300000, 9, "v4n16s1", P.PRNG_MODE_OVERLAP2, 1, 16, 0),   # wide pieces, ragged last piece
    (3000, 9, "auto", P.PRNG_MODE_OVERLAP2, 0, 16, 0),        # auto -> v2n2s1 (small handle), ragged
    (4100, 700, "auto", P.PRNG_MODE_OVERLAP2, 1, 1000, 0),    # time-parallel at 8 warps/SM, v2n2s1, star
    (20000, 300, "v4n4s1p", P.PRNG_MODE_ZEROCOPY, 0, 300, 0), # time-parallel (>= 3 chunks of >= 48), O3
]
# a1 is fused into the first batch launch by default (seeds computed in registers); these
# cases also run with the separate seed kernel (PRNG_OPT_FUSED_SEED 0), and every other case
# reads the state between prng_init and the device-only generate (the pending seeds are
# then materialised by seed_kernel and the launch does not seed)
cases = [c + (1, 1) for c in cases] + [
    (70001, 40, "auto", P.PRNG_MODE_OVERLAP2, 1, 16, 7, 0, 1),   # separate a1: epochs, star
    (1000, 600, "v2n4s1", P.PRNG_MODE_OVERLAP2, 0, 1000, 0, 0, 1),  # separate a1: time-parallel
    (4100, 7, "v4n4s1p", P.PRNG_MODE_SERIAL, 0, 16, 0, 0, 1),    # separate a1: ping-pong
    # one-shot grids (PRNG_OPT_ONE_SHOT 2): one piece per warp, 4-warp CTAs, many waves
    (300007, 9, "v4n8s1a", P.PRNG_MODE_OVERLAP2, 0, 16, 0, 1, 2),  # ragged last CTA / piece
    (200001, 7, "v2n32s1", P.PRNG_MODE_OVERLAP1, 1, 16, 0, 0, 2),  # wide pieces, star, separate a1
]
bad = 0
for ci, (n, it, v, mode, out, slots, epoch, fused, one_shot) in enumerate(cases):
    h = P.prng_create(n, 3)
    P.prng_set_option(h, P.PRNG_OPT_FUSED_SEED, fused)
    P.prng_set_option(h, P.PRNG_OPT_ONE_SHOT, one_shot)
    P.prng_set_option(h, P.PRNG_OPT_KERNEL, names.index(v))
    P.prng_set_option(h, P.PRNG_OPT_OUTPUT, out)
    P.prng_set_option(h, P.PRNG_OPT_MODE, mode)
    P.prng_set_option(h, P.PRNG_OPT_BATCH_ITERS, 0 if it > 100 else 2)
    P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, slots)
    P.prng_set_option(h, P.PRNG_OPT_EPOCH_ITERS, epoch)
    buf = np.zeros((it, n), np.uint64)
    P.prng_init(h)
    P.prng_generate(h, it, P.SINK_COPY, P.CopySink(buf.ctypes.data_as(P.P64), n, 0, it, 0))
    want = oracle.stream_star(n, it, 3) if out else oracle.stream(n, it, 3)
    ok = np.array_equal(buf, want)
    P.prng_init(h)
    if ci % 2:
        ok = ok and np.array_equal(P.prng_read_state(h, n), oracle.stream(n, 1, 3)[0])  # materialised seeds
    P.prng_generate(h, it)  # device only through the ring
    ok = ok and np.array_equal(P.prng_read_state(h, n), oracle.stream(n, it, 3)[-1])
    vid, e = P.prng_last_launch(h)
    grid_one_shot = P.prng_last_grid(h)[3]
    P.prng_destroy(h)
    print(n, it, v, mode, out, slots, epoch, "fused", fused, "one_shot", grid_one_shot, "ran", names[vid], "E", e, "ok" if ok else "MISMATCH", flush=True)
    bad += not ok
sys.exit(1 if bad else 0)
