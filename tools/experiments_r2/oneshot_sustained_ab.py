#!/usr/bin/env python3
"""Round-2 probe: the bench step sustained (100 launches per round, 4 interleaved rounds) on
the one-shot grid with v4n8s1a (the default) vs v4n4s1p / v4n16s1, and the 5-launch burst
after each; NVML SM clock per round."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402
from bench import Clocks  # noqa: E402

torch.cuda.set_device(0)
gen, cop = torch.cuda.Stream(), torch.cuda.Stream()
names = [P.prng_kernel_variant_name(i) for i in range(P.prng_kernel_variants())]
n, it = 1 << 24, 1000
hs = {}
for kn in ("v4n8s1a", "v4n4s1p", "v4n16s1"):
    h = P.prng_create(n, 0)
    P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
    P.prng_set_option(h, P.PRNG_OPT_KERNEL, names.index(kn))
    P.prng_set_option(h, P.PRNG_OPT_BLOCKING, 0)
    for _ in range(15):
        P.prng_init(h)
        P.prng_generate(h, it)
    torch.cuda.synchronize()
    hs[kn] = h
res = {}
for rnd in range(4):
    for kn, h in hs.items():
        time.sleep(1.0)  # let the power controller settle between configurations
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        with Clocks(0) as clk:
            e[0].record(gen)
            for k in range(100):
                if k == 5:
                    e[1].record(gen)
                P.prng_init(h)
                P.prng_generate(h, it)
            e[2].record(gen)
            torch.cuda.synchronize()
        burst = 8 * n * it * 5 / (e[0].elapsed_time(e[1]) * 1e-3) / 1e9
        sust = 8 * n * it * 100 / (e[0].elapsed_time(e[2]) * 1e-3) / 1e9
        res.setdefault(kn, []).append((round(burst), round(sust), clk.summary()["sm_mhz"], P.prng_last_grid(h)[3]))
for kn, v in res.items():
    print(json.dumps({"variant": kn, "first5_gbs": [x[0] for x in v], "sustained100_gbs": [x[1] for x in v],
                      "sm_mhz": [x[2] for x in v], "one_shot": v[0][3]}))
