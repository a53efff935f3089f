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

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["v4n8s1a", "v4n4s1"]
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
    # 512 slots = 64 GiB per handle: the live set (512 x 592 warps x >= 1 KiB) clears 2 x L2,
    # so no rewrite is absorbed in L2 (profiles/r1_l2_absorption.md; round 1 used 128 slots,
    # 16 GiB, whose rewrites were partly absorbed).  Two handles fit in HBM.
    P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, 512)
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
for h in hs.values():
    P.prng_destroy(h)
# the fill engine sustained over a comparable time (~4 s of 32 GiB fills), for reference
print(json.dumps({"variant": "cudaMemsetAsync (sustained)",
                  "gbs": round(P.prng_probe_memset_sustained_gbs(32 << 30, 900), 1)}))
