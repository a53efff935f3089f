#!/usr/bin/env python3
"""Sustained (power-capped) device-only throughput of a few kernel variants, interleaved
rounds so thermal / power drift hits all of them alike.  numrn = 2^24 x 1000 per launch."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["v2n4s1", "v4n8s1", "v4n12s1", "v4n16s1"]
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 6
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
torch.cuda.set_device(0)
gen, cop = torch.cuda.Stream(), torch.cuda.Stream()
allv = [P.prng_kernel_variant_name(i) for i in range(P.prng_kernel_variants())]
n, it = 1 << 24, 1000
hs = {}
for nm in names:
    h = P.prng_create(n, 0)
    P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
    P.prng_set_option(h, P.PRNG_OPT_KERNEL, allv.index(nm))
    P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, 128)  # 16 GiB each (4 handles share the GPU)
    P.prng_init(h)
    P.prng_generate(h, it)
    hs[nm] = h
res = {nm: [] for nm in names}
for r in range(rounds):
    for nm in names:
        h = hs[nm]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(gen)
        for _ in range(reps):
            P.prng_init(h)
            P.prng_generate(h, it)
        e1.record(gen)
        torch.cuda.synchronize()
        res[nm].append(8 * n * it * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9)
for nm in names:
    print(json.dumps({"variant": nm, "median_gbs": round(statistics.median(res[nm]), 1),
                      "min": round(min(res[nm]), 1), "max": round(max(res[nm]), 1)}))
