#!/usr/bin/env python3
"""Round-2 probe: the bimodal small-n timings (e.g. 2^14 x 10^4 reads 205 or 270 us).
Per launch: CUDA-event time, the NVML SM clock just after, and the ring slot the launch
started at; default rotating 64 GiB ring vs a ring of exactly `iters` slots (same addresses
every run)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import pynvml as N  # noqa: E402
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402

N.nvmlInit()
nv = N.nvmlDeviceGetHandleByIndex(0)
torch.cuda.set_device(0)
gen, cop = torch.cuda.Stream(), torch.cuda.Stream()
for lg, it in ((14, 10000), (12, 10000), (15, 10000)):
    for ring in (0, it):
        h = P.prng_create(1 << lg, 0)
        P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
        P.prng_set_option(h, P.PRNG_OPT_BLOCKING, 0)
        P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, ring)
        P.prng_init(h)
        P.prng_generate(h, it)
        torch.cuda.synchronize()
        us, clk, slot0 = [], [], []
        for _ in range(30):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(gen)
            P.prng_init(h)
            P.prng_generate(h, it)
            e1.record(gen)
            torch.cuda.synchronize()
            us.append(round(e0.elapsed_time(e1) * 1e3, 1))
            clk.append(N.nvmlDeviceGetClockInfo(nv, N.NVML_CLOCK_SM))
            slot0.append(P.prng_device_ring(h)[3])
            time.sleep(0.002)
        P.prng_destroy(h)
        print(json.dumps({"n": f"2^{lg}", "i": it, "ring_slots": ring or "auto (64 GiB rotating)", "us": us,
                          "sm_mhz": clk, "iter0_slot": slot0}), flush=True)
