#!/usr/bin/env python3
"""Round-2 experiment: small-numrn cells of the Fig. 4 grid (time-parallel chunks) with
larger grids (PRNG_OPT_GRID_WARPS) -- does the per-warp store rate bound them?"""
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
for lg, it in [(12, 10000), (14, 10000), (14, 1000), (16, 1000), (16, 10000), (18, 1000), (12, 1000), (16, 100)]:
    n = 1 << lg
    for gw, ch in [(g, c) for g in (0, 1184) for c in (0, 32, 64, 128)]:
        h = P.prng_create(n, 0)
        P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
        P.prng_set_option(h, P.PRNG_OPT_GRID_WARPS, gw)
        P.prng_set_option(h, P.PRNG_OPT_CHUNK_ITERS, ch)
        P.prng_init(h)
        P.prng_generate(h, it)
        best = 1e30
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(gen)
            P.prng_init(h)
            P.prng_generate(h, it)
            e1.record(gen)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        ids, s, e, _ = (None, None, None, None)
        vid, ep = P.prng_last_launch(h)
        print(json.dumps({"n": f"2^{lg}", "i": it, "grid_warps": gw, "chunk": ch, "ms": round(best, 4),
                          "gbs": round(8 * n * it / (best * 1e-3) / 1e9, 1), "kernel": P.prng_kernel_variant_name(vid)}),
              flush=True)
        P.prng_destroy(h)
