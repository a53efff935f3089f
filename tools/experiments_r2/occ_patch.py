#!/usr/bin/env python3
"""Experimental build patch (gpu_m37.sh): one-shot launches take PRNG_EXP_SMEM bytes of
dynamic shared memory (unused), to cap the resident CTAs per SM; and the one-shot rule is
forced by PRNG_OPT_ONE_SHOT 2 in the probe.  Never committed to the library."""
import sys
p = sys.argv[1]
s = open(p).read()
old = "    fn<<<(unsigned)blocks, (unsigned)(32 * wpb), 0, s>>>(a);"
new = """    size_t exp_smem = 0;
    if (oneshot && std::getenv("PRNG_EXP_SMEM")) {
        exp_smem = (size_t)std::atoll(std::getenv("PRNG_EXP_SMEM"));
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)exp_smem);
    }
    fn<<<(unsigned)blocks, (unsigned)(32 * wpb), exp_smem, s>>>(a);"""
assert old in s
s = s.replace(old, new)
open(p, "w").write(s)
