#!/usr/bin/env python3
"""Round-2 probe: end to end (mode O2, null sink, 2^24 x 1000 = config 3) with the one-shot
grid (PRNG_OPT_ONE_SHOT 1, auto) vs the persistent grid (0) for the batch launches,
interleaved rounds, host wall clock per call; plus prng_generate_host."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402

torch.cuda.set_device(0)
n, it = 1 << 24, 1000
hs = {}
for mode in (0, 1):
    h = P.prng_create(n, 0)
    P.prng_set_option(h, P.PRNG_OPT_ONE_SHOT, mode)
    P.prng_init(h)
    P.prng_generate(h, 8, P.SINK_NULL)
    hs[mode] = h
arr = torch.empty((4, n), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
res = {}
for rnd in range(3):
    for mode in (0, 1):
        h = hs[mode]
        P.prng_init(h)
        t = time.perf_counter()
        P.prng_generate(h, it, P.SINK_NULL)
        dt = time.perf_counter() - t
        P.prng_init(h)
        t = time.perf_counter()
        P.prng_generate_host(h, 400, arr, n, 4)
        dh = time.perf_counter() - t
        res.setdefault(mode, []).append((8 * n * it / dt / 1e9, 8 * n * 400 / dh / 1e9, P.prng_last_grid(h)))
for mode, v in res.items():
    print(json.dumps({"one_shot": mode, "o2_gbs": [round(x[0], 2) for x in v], "host_gbs": [round(x[1], 2) for x in v],
                      "grid": v[0][2]}))
print(json.dumps({"d2h_probe_gbs": P.prng_probe_d2h_gbs(1 << 30, 5, True, 1)}))
