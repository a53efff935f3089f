#!/usr/bin/env python3
"""NEXT-4: the paper's Fig. 4 grid (n = 2^12, 2^14, ..., 2^24; i = 10^2, 10^3, 10^4;
P:334-335) on the B200 path: device-only and end-to-end throughput per (n, i), plus the
launch/host overhead visible at small n ("a larger n masks the ... overhead").

    python tools/fig4_grid.py [--e2e-cap-gb 20] > fig4.jsonl
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
    ap.add_argument("--e2e-cap-gb", type=float, default=20.0)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    gen, cop = torch.cuda.Stream(), torch.cuda.Stream()
    # ramp the clocks up first (a small first case would otherwise run at idle clocks)
    h = P.prng_create(1 << 24, 0)
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 1.0:
        P.prng_init(h)
        P.prng_generate(h, 200)
    P.prng_destroy(h)
    rows = {}
    # pass 1: device only (CUDA events around init + generate, best of 5 after a warm-up),
    # through the default 64 GiB rotating ring (every byte reaches DRAM; small runs pay
    # fresh-page TLB walks) and through a 256-slot ring (small runs stay in L2: labelled)
    for lg in range(12, 25, 2):
      for ring in (0, 256):
        n = 1 << lg
        h = P.prng_create(n, 0)
        P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
        P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, ring)
        if ring:  # the labelled L2-resident diagnostic: keep the natural order (no
            P.prng_set_option(h, P.PRNG_OPT_EPOCH_ITERS, -1)  # anti-absorption rule)
        for it in (100, 1000, 10000):
            nbytes = 8 * n * it
            P.prng_init(h)
            P.prng_generate(h, it)
            best = None
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(gen)
                P.prng_init(h)
                P.prng_generate(h, it)
                e1.record(gen)
                torch.cuda.synchronize()
                best = min(best or 1e30, e0.elapsed_time(e1))
            key = "device" if ring == 0 else "device_ring256"
            rows.setdefault((lg, it), {"n": f"2^{lg}", "i": it, "bytes": nbytes})
            vid, ep = P.prng_last_launch(h)
            rows[(lg, it)].update({f"{key}_ms": best, f"{key}_gbs": nbytes / (best * 1e-3) / 1e9,
                                   f"{key}_kernel": P.prng_kernel_variant_name(vid) + (f"/E{ep}" if ep else "")})
        P.prng_destroy(h)
    # pass 2: end to end (host wall clock, null sink), bounded total bytes
    for lg in range(12, 25, 2):
        n = 1 << lg
        h = P.prng_create(n, 0)
        for it in (100, 1000, 10000):
            nbytes = 8 * n * it
            if nbytes > a.e2e_cap_gb * 1e9:
                continue
            P.prng_init(h)
            P.prng_generate(h, min(it, 4), P.SINK_NULL)  # allocate the pinned halves
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            P.prng_init(h)
            P.prng_generate(h, it, P.SINK_NULL)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            rows[(lg, it)].update({"e2e_ms": dt * 1e3, "e2e_gbs": nbytes / dt / 1e9})
        P.prng_destroy(h)
    for k in sorted(rows):
        print(json.dumps(rows[k]), flush=True)


if __name__ == "__main__":
    main()
