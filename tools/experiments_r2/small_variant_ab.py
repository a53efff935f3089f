#!/usr/bin/env python3
"""Round-2 A/B on one box: "auto" (v4n4s1p below 2^21) vs v2n2s1 (64-gid pieces) for small
numrn, time-parallel on (default), interleaved rounds, device-only (CUDA events around
prng_init + prng_generate, best of 5 per round)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402

torch.cuda.set_device(0)
gen, cop = torch.cuda.Stream(), torch.cuda.Stream()
names = [P.prng_kernel_variant_name(i) for i in range(P.prng_kernel_variants())]
h = P.prng_create(1 << 24, 0)
for _ in range(50):
    P.prng_init(h)
    P.prng_generate(h, 200)
P.prng_destroy(h)
cells = [(lg, it) for lg in (10, 12, 13, 14, 15, 16) for it in (100, 300, 1000, 10000)]
res = {}
for rnd in range(3):
    for lg, it in cells:
        for kn in ("auto", "v4n4s1p", "v2n2s1"):
            h = P.prng_create(1 << lg, 0)
            P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
            P.prng_set_option(h, P.PRNG_OPT_KERNEL, names.index(kn))
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
            P.prng_destroy(h)
            res.setdefault((lg, it, kn), []).append(round(best * 1e3, 1))
for k, v in res.items():
    print(json.dumps({"n": f"2^{k[0]}", "i": k[1], "kernel": k[2], "us": v,
                      "gbs": round(8 * (1 << k[0]) * k[1] / (min(v) * 1e-6) / 1e9)}))
