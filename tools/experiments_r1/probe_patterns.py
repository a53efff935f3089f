#!/usr/bin/env python3
"""Research probe: SM store patterns over 32 GiB (GB/s), to see what the HBM write path
rewards.  See prngk::store_pattern_kernel for the modes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402

torch.cuda.set_device(0)
L = P.lib()
B = 32 << 30
for mode in (0, 1, 2, 3):
    for wpc, cps in ((4, 1), (8, 1), (4, 2), (8, 2), (8, 4)):
        print(f"mode {mode} warps/CTA {wpc} CTAs/SM {cps}: {L.prng_probe_store_mode_gbs(B, 3, mode, wpc, cps, 1):.0f}",
              flush=True)
for slots in (256, 512, 4096):
    for wpc, cps in ((4, 1), (8, 1), (2, 2)):
        print(f"mode 4 slots {slots} warps/CTA {wpc} CTAs/SM {cps}: "
              f"{L.prng_probe_store_mode_gbs(B, 3, 4, wpc, cps, slots):.0f}", flush=True)
print(f"memset: {P.prng_probe_memset_gbs(B, 3):.0f}")
