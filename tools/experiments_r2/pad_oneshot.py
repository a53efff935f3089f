#!/usr/bin/env python3
"""Round-2 probe: ring pitch padding (PRNG_OPT_RING_PAD) on the one-shot grid at the bench
shape -- consecutive CTAs write consecutive slots' columns, so the slot pitch (128 MiB, a
power of two, unpadded) decides which DRAM banks they hit together.  Burst (best of 5 after
15 warm-up launches) and 40-launch sustained, 3 interleaved rounds."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402

torch.cuda.set_device(0)
gen, cop = torch.cuda.Stream(), torch.cuda.Stream()
n, it = 1 << 24, 1000
pads = (0, 32, 256, 1024, 4096, 12288, 65536)
res = {}
for rnd in range(3):
    for pad in pads:
        h = P.prng_create(n, 0)
        P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
        P.prng_set_option(h, P.PRNG_OPT_RING_PAD, pad)
        P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, 480)
        P.prng_set_option(h, P.PRNG_OPT_BLOCKING, 0)
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 0.4:  # past the post-allocation slow phase
            P.prng_init(h)
            P.prng_generate(h, it)
            torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(gen)
            P.prng_init(h)
            P.prng_generate(h, it)
            e1.record(gen)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(gen)
        for _ in range(40):
            P.prng_init(h)
            P.prng_generate(h, it)
        e1.record(gen)
        torch.cuda.synchronize()
        res.setdefault(pad, []).append((round(8 * n * it / (min(ts) * 1e-3) / 1e9),
                                        round(8 * n * it * 40 / (e0.elapsed_time(e1) * 1e-3) / 1e9),
                                        P.prng_last_grid(h)[3]))
        P.prng_destroy(h)
for pad, v in res.items():
    print(json.dumps({"pad_u64": pad, "burst_best_gbs": [x[0] for x in v], "sustained40_gbs": [x[1] for x in v],
                      "one_shot": v[0][2]}))
