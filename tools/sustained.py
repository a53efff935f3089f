#!/usr/bin/env python3
"""Sustained (power-capped) device-only throughput of several (variant, grid warps, CTA
warps) configurations at the bench shape (numrn = 2^24 x 1000 per launch), interleaved
rounds so thermal / power drift hits all of them alike; NVML SM clock per round.

    python tools/sustained.py "v4n8s1a:0:0,v4n8s1a:1184:8" [rounds] [reps]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402
from bench import Clocks  # noqa: E402

cfgs = [c.split(":") for c in (sys.argv[1] if len(sys.argv) > 1 else "v4n8s1a:0:0,v4n4s1:0:0").split(",")]
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 4
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 100
torch.cuda.set_device(0)
gen, cop = torch.cuda.Stream(), torch.cuda.Stream()
allv = [P.prng_kernel_variant_name(i) for i in range(P.prng_kernel_variants())]
n, it = 1 << 24, 1000
h = P.prng_create(n, 0)
P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
P.prng_set_option(h, P.PRNG_OPT_BLOCKING, 0)
res = {":".join(c): [] for c in cfgs}
for r in range(rounds):
    for c in cfgs:
        name, gw, cw = c[0], int(c[1]), int(c[2])
        P.prng_set_option(h, P.PRNG_OPT_KERNEL, allv.index(name))
        P.prng_set_option(h, P.PRNG_OPT_GRID_WARPS, gw)
        P.prng_set_option(h, P.PRNG_OPT_CTA_WARPS, cw)
        P.prng_init(h)
        P.prng_generate(h, it)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with Clocks(0) as clk:
            e0.record(gen)
            for _ in range(reps):
                P.prng_init(h)
                P.prng_generate(h, it)
            e1.record(gen)
            torch.cuda.synchronize()
        s = clk.summary()
        ran, ep = P.prng_last_launch(h)
        res[":".join(c)].append((8 * n * it * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9, s["sm_mhz"],
                                 allv[ran], ep))
for k, v in res.items():
    print(json.dumps({"config": k, "median_gbs": round(statistics.median(x[0] for x in v), 1),
                      "min": round(min(x[0] for x in v), 1), "max": round(max(x[0] for x in v), 1),
                      "sm_mhz": [x[1] for x in v], "ran": v[0][2], "epoch": v[0][3]}))
P.prng_destroy(h)
