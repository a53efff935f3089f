#!/usr/bin/env python3
"""Round-2 probe (needs the gpu_m33.sh experimental build, which lifts the one-wave cap on
PRNG_OPT_GRID_WARPS): persistent one-wave grid (the library's default) vs a one-shot
multi-wave grid (GRID_WARPS = every unit, one unit per warp, CTAs of CTA_WARPS warps,
dispatched in order by the hardware) over shapes, device-only through the default 64 GiB
ring, 3 interleaved rounds, best / median of 5 launches per round (GB/s)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402

torch.cuda.set_device(0)
gen, cop = torch.cuda.Stream(), torch.cuda.Stream()
names = [P.prng_kernel_variant_name(i) for i in range(P.prng_kernel_variants())]
# (log2 n, iters, [(label, variant, grid_warps, cta_warps)])
NPT = {"v4n8s1a": 8, "v4n4s1p": 4, "v4n16s1": 16, "v2n32s1": 32, "v4n8s1": 8}


def oneshot(v, n, cw=4):
    return (f"oneshot-{v}-c{cw}", v, -(-n // (32 * NPT[v])), cw)


cells = []
for lg, it in ((20, 1000), (22, 100), (22, 1000), (24, 100), (24, 1000), (25, 1000), (26, 1000), (27, 200)):
    n = 1 << lg
    cfg = [("auto", "auto", 0, 0)]
    big = "v4n8s1a" if lg >= 21 else "v4n4s1p"
    cfg.append(oneshot(big, n))
    if lg >= 25:
        cfg += [("persist-v4n16s1", "v4n16s1", 0, 0), oneshot("v4n16s1", n), ("persist-v2n32s1", "v2n32s1", 0, 0),
                oneshot("v2n32s1", n)]
    cells.append((lg, it, cfg))
res = {}
for rnd in range(3):
    for lg, it, cfg in cells:
        n = 1 << lg
        for label, v, gw, cw in cfg:
            h = P.prng_create(n, 0)
            P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
            P.prng_set_option(h, P.PRNG_OPT_KERNEL, names.index(v))
            P.prng_set_option(h, P.PRNG_OPT_GRID_WARPS, gw)
            P.prng_set_option(h, P.PRNG_OPT_CTA_WARPS, cw)
            P.prng_set_option(h, P.PRNG_OPT_BLOCKING, 0)
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
            vid, ep = P.prng_last_launch(h)
            P.prng_destroy(h)
            res.setdefault((lg, it, label), []).append((8 * n * it / (min(ts) * 1e-3) / 1e9,
                                                        8 * n * it / (statistics.median(ts) * 1e-3) / 1e9,
                                                        names[vid], ep))
for (lg, it, label), v in res.items():
    print(json.dumps({"n": f"2^{lg}", "i": it, "cfg": label, "best_gbs": [round(x[0]) for x in v],
                      "median_gbs": [round(x[1]) for x in v], "ran": v[0][2], "epoch": v[0][3]}))
