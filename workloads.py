"""Seeded synthetic workloads shared by tests/ and bench.py.

Holds NONE of the method's arithmetic: only the shapes of BASELINE.json's configs, the
seeds, and seeded (numpy) choices of which outputs to sample.  The method's input is just
(numrn, numiter, seed) -- the paper's program takes n and i on the command line
 -- so "synthetic input" here means those integers, shaped like the paper's
defaults, plus the seed (reading A4).
"""
from __future__ import annotations

import numpy as np

SEED_PERF = 0                      # seed 0 == the paper (no seed argument; A4)
SEED_PARITY = 0x0123456789ABCDEF   # a nonzero seed exercising the A4 premix

# BASELINE.json "configs" (index = position in that list).
CONFIGS = {
    "c1": dict(numrn=1024, numiter=8, mode="parity"),
    "c2": dict(numrn=1 << 24, numiter=1000, mode="device"),
    "c3": dict(numrn=1 << 24, numiter=1000, mode="e2e"),
    "c4": dict(numrn=1 << 28, numiter=1000, mode="device"),   # sharded over 2/4/8 GPUs
    "c5": dict(numrn=1 << 28, numiter=100, mode="e2e"),       # sharded over 8 GPUs
}

# Parity grid of SPEC.md S:499 / S:582 (n, i) in {1, 7, 256, 4096} x {1, 2, 8, 16},
# plus ragged shapes that do not divide any tile / warp / vector width.
SPEC_GRID_N = (1, 7, 256, 4096)
SPEC_GRID_I = (1, 2, 8, 16)
RAGGED_N = (1, 2, 3, 31, 33, 63, 65, 127, 129, 1000, 1023, 1025, 4097, 65535, 100003)


def sample_points(numrn: int, numiter: int, nsamples: int, rng_seed: int = 1234,
                  gid_begin: int = 0, count: int | None = None):
    """Seeded uniform (gid, k) sample inside [gid_begin, gid_begin+count) x [0, numiter),
    always including the four corners (first/last gid x first/last iteration)."""
    if count is None:
        count = numrn - gid_begin
    r = np.random.default_rng(rng_seed)
    g = r.integers(gid_begin, gid_begin + count, size=nsamples, dtype=np.int64)
    k = r.integers(0, numiter, size=nsamples, dtype=np.int64)
    cg = np.array([gid_begin, gid_begin + count - 1] * 2, dtype=np.int64)
    ck = np.array([0, 0, numiter - 1, numiter - 1], dtype=np.int64)
    return np.concatenate([cg, g]), np.concatenate([ck, k])


def shard_range(numrn: int, rank: int, world: int):
    """Contiguous gid range of `rank` out of `world`: [floor(r n/P), floor((r+1) n/P))."""
    b = (rank * numrn) // world
    e = ((rank + 1) * numrn) // world
    return b, e - b
