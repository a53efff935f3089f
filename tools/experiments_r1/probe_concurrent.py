#!/usr/bin/env python3
"""Research probe: SM stores + copy-engine D2D concurrently -- do the write paths add up?"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402

torch.cuda.set_device(0)
L = P.lib()
for sm_gib, ce_gib, chunk_mib, w in ((24, 8, 32, 4), (24, 8, 32, 8), (20, 12, 32, 4), (28, 4, 32, 4), (24, 8, 8, 4)):
    a, b = ctypes.c_double(), ctypes.c_double()
    tot = L.prng_probe_concurrent_gbs(sm_gib << 30, ce_gib << 30, chunk_mib << 20, w, 2, ctypes.byref(a), ctypes.byref(b))
    print(f"SM {sm_gib} GiB ({w} warps/SM) + CE {ce_gib} GiB ({chunk_mib} MiB src): combined {tot:.0f} GB/s; "
          f"SM alone {a.value:.0f}, CE alone {b.value:.0f}", flush=True)
print(f"memset 32 GiB: {P.prng_probe_memset_gbs(32 << 30, 2):.0f}")
