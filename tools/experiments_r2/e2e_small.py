#!/usr/bin/env python3
"""Round-2 probe: end-to-end per-call cost at small n (host wall clock around prng_init +
prng_generate(SINK_NULL), mode O2, and prng_generate_host into a pinned array), best of 20.
argv[1]: tag; argv[2] (optional): path of the libprng_b200.so to load (A/B of two builds)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
tag = sys.argv[1] if len(sys.argv) > 1 else ""
import paper_1609_01257_b200 as P  # noqa: E402
if len(sys.argv) > 2:
    os.environ["PRNG_B200_NO_BUILD"] = "1"
    P.LIB = os.path.abspath(sys.argv[2])
import numpy as np  # noqa: E402
import torch  # noqa: E402

torch.cuda.set_device(0)
for lg in (10, 12, 14, 16, 18):
    for it in (1, 10, 100, 1000):
        n = 1 << lg
        h = P.prng_create(n, 0)
        P.prng_init(h)
        P.prng_generate(h, it, P.SINK_NULL)
        best = 1e30
        for _ in range(20):
            t = time.perf_counter()
            P.prng_init(h)
            P.prng_generate(h, it, P.SINK_NULL)
            best = min(best, time.perf_counter() - t)
        arr = torch.empty((it, n), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
        P.prng_init(h)
        P.prng_generate_host(h, it, arr, n, it)
        bh = 1e30
        for _ in range(20):
            t = time.perf_counter()
            P.prng_init(h)
            P.prng_generate_host(h, it, arr, n, it)
            bh = min(bh, time.perf_counter() - t)
        P.prng_destroy(h)
        print(json.dumps({"build": tag, "n": f"2^{lg}", "i": it, "o2_us": round(best * 1e6, 1),
                          "o2_gbs": round(8 * n * it / best / 1e9, 2), "host_us": round(bh * 1e6, 1),
                          "host_gbs": round(8 * n * it / bh / 1e9, 2)}), flush=True)
