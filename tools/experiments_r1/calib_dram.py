#!/usr/bin/env python3
"""Run each write path once on known bytes, for an ncu dram__bytes_write calibration:
cudaMemsetAsync 4 GiB, the 32-B store probe 4 GiB, and one batch-kernel launch of
numrn x numiter (device only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1609_01257_b200 as P  # noqa: E402

torch.cuda.set_device(0)
print("memset GB/s", P.prng_probe_memset_gbs(4 << 30, 1))
print("store GB/s", P.prng_probe_store_gbs(4 << 30, 1))
n, it = 1 << 24, int(sys.argv[1]) if len(sys.argv) > 1 else 32
h = P.prng_create(n, 0)
P.prng_init(h)
P.prng_generate(h, it)
P.prng_destroy(h)
print("batch kernel bytes", 8 * n * it)
