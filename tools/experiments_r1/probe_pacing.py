#!/usr/bin/env python3
"""Research probe: does pacing SM stores (dependent ALU work between them) raise the HBM
write rate?  mode 100+k = grid-stride 16-B stores with k xorshift steps between stores."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402

torch.cuda.set_device(0)
L = P.lib()
B = 32 << 30
for k in (0, 1, 2, 4, 6, 8, 12, 16):
    for wpc, cps in ((4, 1), (8, 1), (8, 2), (8, 4)):
        print(f"pace {k} warps/CTA {wpc} CTAs/SM {cps}: {L.prng_probe_store_mode_gbs(B, 3, 100 + k, wpc, cps, 1):.0f}",
              flush=True)
