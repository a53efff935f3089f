#!/usr/bin/env python3
"""Round-2 probe: small-n cells (device-only, prng_init + prng_generate non-blocking, CUDA
events, best of 20) for an A/B of the shortest time-parallel chunk (run once per build)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else ""
torch.cuda.set_device(0)
gen, cop = torch.cuda.Stream(), torch.cuda.Stream()
h = P.prng_create(1 << 24, 0)
for _ in range(50):
    P.prng_init(h)
    P.prng_generate(h, 200)
P.prng_destroy(h)
for lg in (10, 12, 13, 14, 15, 16):
    for it in (100, 200, 300, 500, 1000, 3000, 10000):
        h = P.prng_create(1 << lg, 0)
        P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
        P.prng_set_option(h, P.PRNG_OPT_BLOCKING, 0)
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
        vid, ep = P.prng_last_launch(h)
        P.prng_destroy(h)
        print(json.dumps({"build": tag, "n": f"2^{lg}", "i": it, "us": round(best, 1),
                          "gbs": round(8 * (1 << lg) * it / (best * 1e-6) / 1e9, 1),
                          "kernel": P.prng_kernel_variant_name(vid)}), flush=True)
