#!/usr/bin/env python3
"""Round-2 probe (gpu_m37.sh experimental build): one-shot grids with the resident CTAs per
SM capped by dynamic shared memory (env PRNG_EXP_SMEM, set per process by the script),
vs the persistent grid; burst (best / median of 5 after >= 0.3 s warm-up) per shape, and the
bench step sustained (100 launches)."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402
from bench import Clocks  # noqa: E402

tag = sys.argv[1]
mode = int(sys.argv[2])
torch.cuda.set_device(0)
gen, cop = torch.cuda.Stream(), torch.cuda.Stream()
for lg, it, reps in ((22, 1000, 5), (23, 1000, 5), (24, 100, 5), (24, 1000, 5), (24, 1000, 100)):
    n = 1 << lg
    h = P.prng_create(n, 0)
    P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
    P.prng_set_option(h, P.PRNG_OPT_ONE_SHOT, mode)
    P.prng_set_option(h, P.PRNG_OPT_BLOCKING, 0)
    t0 = time.perf_counter()
    k = 0
    while k < 10 or time.perf_counter() - t0 < 0.3:
        P.prng_init(h)
        P.prng_generate(h, it)
        torch.cuda.synchronize()
        k += 1
    ts = []
    with Clocks(0) as clk:
        for _ in range(5 if reps == 5 else 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(gen)
            for _ in range(1 if reps == 5 else reps):
                P.prng_init(h)
                P.prng_generate(h, it)
            e1.record(gen)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / (1 if reps == 5 else reps))
    grid = P.prng_last_grid(h)
    P.prng_destroy(h)
    g = [8 * n * it / (t * 1e-3) / 1e9 for t in ts]
    print(json.dumps({"cfg": tag, "n": f"2^{lg}", "i": it, "reps": reps, "best": round(max(g)),
                      "median": round(statistics.median(g)), "grid": grid, "sm_mhz": clk.summary()["sm_mhz"]}),
          flush=True)
