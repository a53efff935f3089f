#!/usr/bin/env python3
"""Drift diagnostic (GPU box): run the traced variant v2n4s1t and report how far CTAs drift
apart in iterations while they sweep the ring."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
torch.cuda.set_device(0)
names = [P.prng_kernel_variant_name(i) for i in range(P.prng_kernel_variants())]
kv = names.index("v2n4s1t")
h = P.prng_create(n, 0)
P.prng_set_option(h, P.PRNG_OPT_KERNEL, kv)
ctas = 148
npieces = (n + 127) // 128
warps = 592
rounds = (npieces + warps - 1) // warps
per_round = (iters + 63) // 64
buf = torch.zeros(ctas * rounds * per_round + 1024, dtype=torch.int64, device="cuda")
P.prng_set_option(h, P.PRNG_OPT_TRACE_PTR, buf.data_ptr())
P.prng_init(h)
P.prng_generate(h, iters)
P.prng_init(h)
buf.zero_()
t0 = torch.cuda.Event(enable_timing=True)
t1 = torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
P.prng_generate(h, iters)
torch.cuda.synchronize()
tr = buf[: ctas * rounds * per_round].cpu().numpy().reshape(ctas, rounds, per_round).astype(np.float64)
P.prng_destroy(h)
valid = tr > 0
t_start = tr[valid].min()
tr = np.where(valid, tr - t_start, np.nan)
total_ns = np.nanmax(tr)
bytes_total = 8 * n * iters
ns_per_iter_cta = total_ns / (rounds * iters)   # a CTA's average time per iteration
spread = np.nanmax(tr, axis=0) - np.nanmin(tr, axis=0)     # [round, sample] spread across CTAs
out = {"n": n, "iters": iters, "rounds": rounds, "total_ms": total_ns / 1e6,
       "gbs": bytes_total / total_ns, "ns_per_iteration": ns_per_iter_cta,
       "spread_ns_median": float(np.nanmedian(spread)), "spread_ns_p90": float(np.nanpercentile(spread, 90)),
       "spread_iters_median": float(np.nanmedian(spread) / ns_per_iter_cta),
       "spread_iters_p90": float(np.nanpercentile(spread, 90) / ns_per_iter_cta),
       "spread_iters_max": float(np.nanmax(spread) / ns_per_iter_cta)}
# how many distinct slots are being written at one instant: at a global time t, each CTA is
# at (round, iteration); count distinct iterations mod ring among CTAs
print(json.dumps(out))
