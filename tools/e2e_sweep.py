#!/usr/bin/env python3
"""End-to-end throughput sweep (GPU box): modes x batch T x host memory kind, null sink.

    python tools/e2e_sweep.py [--numrn 16777216] [--numiter 200]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--numrn", type=int, default=1 << 24)
    ap.add_argument("--numiter", type=int, default=200)
    ap.add_argument("--modes", default="3,4")
    ap.add_argument("--batches", default="1,2,4,8")
    ap.add_argument("--hostmem", default="0,1,2")
    ap.add_argument("--kernel", type=int, default=0)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for mode in [int(x) for x in a.modes.split(",")]:
        for T in [int(x) for x in a.batches.split(",")]:
            for hm in ([0] if mode == 4 else [int(x) for x in a.hostmem.split(",")]):
                h = P.prng_create(a.numrn, 0)
                P.prng_set_option(h, P.PRNG_OPT_MODE, mode)
                P.prng_set_option(h, P.PRNG_OPT_BATCH_ITERS, T)
                P.prng_set_option(h, P.PRNG_OPT_HOST_MEM, hm)
                P.prng_set_option(h, P.PRNG_OPT_KERNEL, a.kernel)
                P.prng_init(h)
                P.prng_generate(h, 2 * T, P.SINK_NULL)  # allocate + warm
                best = 0
                for _ in range(2):
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    P.prng_init(h)
                    P.prng_generate(h, a.numiter, P.SINK_NULL)
                    dt = time.perf_counter() - t0
                    best = max(best, 8 * a.numrn * a.numiter / dt / 1e9)
                P.prng_destroy(h)
                print(json.dumps({"mode": mode, "T": T, "host_mem": hm, "gbs": round(best, 2)}), flush=True)
    print(json.dumps({"probe_d2h_pinned": P.prng_probe_d2h_gbs(1 << 30, 5, True, 1),
                      "probe_d2h_pinned_4GiB": P.prng_probe_d2h_gbs(4 << 30, 3, True, 1)}), flush=True)


if __name__ == "__main__":
    main()
