#!/usr/bin/env python3
"""Round-2 probe: warps per SM of natural-order launches at mid n (2^16..2^22 x 100..1000),
where a launch may be latency-bound rather than DRAM-bound (copy of tp_warps.py).
PRNG_OPT_GRID_WARPS = W * SMs (the TP rule then cuts min(W*SMs / pieces, iters / 48)
chunks) for W = 8 (the auto rule's), 16, 24, 32; device-only, non-blocking, CUDA events,
best of 10, two interleaved rounds.  A light warm-up keeps the GPU below its power cap."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402

torch.cuda.set_device(0)
sms = torch.cuda.get_device_properties(0).multi_processor_count
gen, cop = torch.cuda.Stream(), torch.cuda.Stream()
h = P.prng_create(1 << 20, 0)
t0 = time.perf_counter()
while time.perf_counter() - t0 < 0.3:
    P.prng_init(h)
    P.prng_generate(h, 100)
P.prng_destroy(h)
res = {}
for rnd in range(2):
    for lg in (16, 17, 18, 19, 20, 21, 22):
        for it in (100, 300, 1000):
            for W in (0, 8, 12, 16):
                h = P.prng_create(1 << lg, 0)
                P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
                P.prng_set_option(h, P.PRNG_OPT_BLOCKING, 0)
                P.prng_set_option(h, P.PRNG_OPT_GRID_WARPS, W * sms)
                P.prng_init(h)
                P.prng_generate(h, it)
                torch.cuda.synchronize()
                best = 1e30
                for _ in range(10):
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
                res.setdefault((lg, it, W), []).append(round(best, 1))
for (lg, it, W), v in res.items():
    print(json.dumps({"n": f"2^{lg}", "i": it, "warps_per_sm": W or 4, "us": v,
                      "gbs": round(8 * (1 << lg) * it / (min(v) * 1e-6) / 1e9)}))
