#!/usr/bin/env python3
"""Round-2 probe: where the ~25-35 us floor of a small-n prng_init + prng_generate goes
(profiles/r2_fig4.md).  Per cell: GPU time (CUDA events on the gen stream) of init alone,
generate alone, and both; host time of the calls (non-blocking); best of 20."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402

torch.cuda.set_device(0)
gen, cop = torch.cuda.Stream(), torch.cuda.Stream()
h = P.prng_create(1 << 24, 0)
for _ in range(50):
    P.prng_init(h)
    P.prng_generate(h, 200)
P.prng_destroy(h)


def best_of(fn, reps=20):
    bg, bh = 1e30, 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(gen)
        t0 = time.perf_counter()
        fn()
        t1 = time.perf_counter()
        e1.record(gen)
        torch.cuda.synchronize()
        bg = min(bg, e0.elapsed_time(e1) * 1e3)
        bh = min(bh, (t1 - t0) * 1e6)
    return round(bg, 1), round(bh, 1)


for lg in (12, 14, 16, 18):
    for it in (1, 100, 1000):
        h = P.prng_create(1 << lg, 0)
        P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
        for blocking in (1, 0):
            P.prng_set_option(h, P.PRNG_OPT_BLOCKING, blocking)
            P.prng_init(h)
            P.prng_generate(h, it)
            torch.cuda.synchronize()
            gi, hi = best_of(lambda: P.prng_init(h))
            gg, hg = best_of(lambda: P.prng_generate(h, it))
            gb, hb = best_of(lambda: (P.prng_init(h), P.prng_generate(h, it)))
            vid, ep = P.prng_last_launch(h)
            print(json.dumps({"n": f"2^{lg}", "i": it, "blocking": blocking, "kernel": P.prng_kernel_variant_name(vid),
                              "gpu_us": {"init": gi, "generate": gg, "both": gb},
                              "host_us": {"init": hi, "generate": hg, "both": hb},
                              "gbs_both": round(8 * (1 << lg) * it / (gb * 1e-6) / 1e9, 1)}), flush=True)
        P.prng_destroy(h)
