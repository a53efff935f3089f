#!/usr/bin/env python3
"""Round-2 probe: the library's one-shot grid (PRNG_OPT_ONE_SHOT 2 = always, where the form
allows) vs the persistent grid (0) by shape, to place the auto threshold (kOneShotMinWaves);
device-only, default ring, auto kernel, 3 interleaved rounds, best / median of 5 launches;
then the bench step sustained (2 x 100 launches each) with auto (1) vs 0."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402
from bench import Clocks  # noqa: E402

torch.cuda.set_device(0)
gen, cop = torch.cuda.Stream(), torch.cuda.Stream()


def run(n, it, mode, reps):
    h = P.prng_create(n, 0)
    P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
    P.prng_set_option(h, P.PRNG_OPT_ONE_SHOT, mode)
    P.prng_set_option(h, P.PRNG_OPT_BLOCKING, 0)
    # warm-up: >= 10 launches and >= 0.3 s (the first launches after a ring allocation are
    # slow, profiles/r2_fig4.md "bimodal cells")
    t0 = time.perf_counter()
    k = 0
    while k < 10 or time.perf_counter() - t0 < 0.3:
        P.prng_init(h)
        P.prng_generate(h, it)
        torch.cuda.synchronize()
        k += 1
    ts = []
    with Clocks(0) as clk:
        for _ in range(reps if reps <= 5 else 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(gen)
            for _ in range(1 if reps <= 5 else reps):
                P.prng_init(h)
                P.prng_generate(h, it)
            e1.record(gen)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / (1 if reps <= 5 else reps))
    grid = P.prng_last_grid(h)
    vid, ep = P.prng_last_launch(h)
    P.prng_destroy(h)
    gbs = [8 * n * it / (t * 1e-3) / 1e9 for t in ts]
    return max(gbs), statistics.median(gbs), grid, P.prng_kernel_variant_name(vid), ep, clk.summary()["sm_mhz"]


res = {}
for rnd in range(3):
    for lg in (19, 20, 21, 22, 23, 24):
        for it in (100, 1000):
            for mode in (0, 2):
                b, m, grid, v, ep, mhz = run(1 << lg, it, mode, 5)
                res.setdefault((lg, it, mode), []).append((round(b), round(m), grid[3], v, ep, mhz))
for (lg, it, mode), v in res.items():
    print(json.dumps({"n": f"2^{lg}", "i": it, "one_shot": mode, "best_gbs": [x[0] for x in v],
                      "median_gbs": [x[1] for x in v], "ran_one_shot": v[0][2], "kernel": v[0][3], "epoch": v[0][4],
                      "sm_mhz": [x[5] for x in v]}), flush=True)
for rnd in range(2):
    for mode in (1, 0):
        b, m, grid, v, ep, mhz = run(1 << 24, 1000, mode, 100)
        print(json.dumps({"sustained": True, "n": "2^24", "i": 1000, "one_shot": mode, "gbs": round(b),
                          "grid": grid, "kernel": v, "sm_mhz": mhz}), flush=True)
