#!/usr/bin/env python3
"""Round-2 probe: which variant on the one-shot grid (PRNG_OPT_ONE_SHOT 2, 3 CTAs/SM) by
shape -- v4n4s1p (1 KiB per warp-iteration), v4n8s1a (2 KiB), v4n16s1 (4 KiB) -- against
"auto"; >= 0.3 s warm-up, best / median of 5, 3 interleaved rounds."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402

torch.cuda.set_device(0)
gen, cop = torch.cuda.Stream(), torch.cuda.Stream()
names = [P.prng_kernel_variant_name(i) for i in range(P.prng_kernel_variants())]
res = {}
for rnd in range(3):
    for lg in (20, 21, 22, 23, 24):
        for it in (100, 1000):
            for kn, os_ in (("auto", 1), ("v4n4s1p", 2), ("v4n8s1a", 2), ("v4n16s1", 2)):
                n = 1 << lg
                h = P.prng_create(n, 0)
                P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
                P.prng_set_option(h, P.PRNG_OPT_KERNEL, names.index(kn))
                P.prng_set_option(h, P.PRNG_OPT_ONE_SHOT, os_)
                P.prng_set_option(h, P.PRNG_OPT_BLOCKING, 0)
                t0 = time.perf_counter()
                k = 0
                while k < 10 or time.perf_counter() - t0 < 0.3:
                    P.prng_init(h)
                    P.prng_generate(h, it)
                    torch.cuda.synchronize()
                    k += 1
                ts = []
                for _ in range(5):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(gen)
                    P.prng_init(h)
                    P.prng_generate(h, it)
                    e1.record(gen)
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
                vid, _ = P.prng_last_launch(h)
                grid = P.prng_last_grid(h)
                P.prng_destroy(h)
                g = [8 * n * it / (t * 1e-3) / 1e9 for t in ts]
                res.setdefault((lg, it, kn), []).append((round(max(g)), round(statistics.median(g)), names[vid], grid[3]))
for (lg, it, kn), v in res.items():
    print(json.dumps({"n": f"2^{lg}", "i": it, "cfg": kn, "best": [x[0] for x in v], "median": [x[1] for x in v],
                      "ran": v[0][2], "one_shot": v[0][3]}))
