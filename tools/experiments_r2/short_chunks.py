#!/usr/bin/env python3
"""Round-2 probe: time-parallel chunks for SHORT launches (i < 256, where the auto rule does
not chunk).  Forced PRNG_OPT_CHUNK_ITERS L vs auto, device-only, prng_init + prng_generate
non-blocking, GPU time by CUDA events, best of 20, a1 fused (the default)."""
import json
import os
import sys

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
names = [P.prng_kernel_variant_name(i) for i in range(P.prng_kernel_variants())]
for lg in (10, 12, 14, 16):
    for it in (50, 100, 200, 300):
        for kn in ("auto", "v2n2s1"):
            row = {}
            for L in (0, 6, 8, 12, 16, 25, 32, 50, 64, 100):
                if L and L >= it:
                    continue
                h = P.prng_create(1 << lg, 0)
                P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
                P.prng_set_option(h, P.PRNG_OPT_BLOCKING, 0)
                P.prng_set_option(h, P.PRNG_OPT_KERNEL, names.index(kn))
                P.prng_set_option(h, P.PRNG_OPT_CHUNK_ITERS, L)
                P.prng_init(h)
                P.prng_generate(h, it)
                torch.cuda.synchronize()
                best = 1e30
                for _ in range(20):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    e0.record(gen)
                    P.prng_init(h)
                    P.prng_generate(h, it)
                    e1.record(gen)
                    torch.cuda.synchronize()
                    best = min(best, e0.elapsed_time(e1) * 1e3)
                P.prng_destroy(h)
                row[L] = round(best, 1)
            print(json.dumps({"n": f"2^{lg}", "i": it, "kernel": kn, "us_by_chunk": row}), flush=True)
