#!/usr/bin/env python3
"""Round-2 A/B on one box: time-parallel on / off for the small-n Fig. 4 cells, interleaved
rounds (device-only, CUDA events around prng_init + prng_generate, best of 5 per round)."""
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
cells = [(12, 1000), (12, 10000), (14, 1000), (14, 10000), (16, 1000), (16, 10000), (16, 300)]
hs = {}
for lg, it in cells:
    for tp in (0, 1):
        h = P.prng_create(1 << lg, 0)
        P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
        P.prng_set_option(h, P.PRNG_OPT_TIME_PARALLEL, tp)
        hs[(lg, it, tp)] = h
res = {}
for rnd in range(3):
    for (lg, it, tp), h in hs.items():
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
        res.setdefault((lg, it, tp), []).append(8 * (1 << lg) * it / (best * 1e-3) / 1e9)
for k, v in res.items():
    print(json.dumps({"n": f"2^{k[0]}", "i": k[1], "time_parallel": k[2], "gbs": [round(x) for x in v]}))
