"""Build libprng_b200.so (the hot path's C ABI) and libprng_probes.so (bench.py's same-box
roofline probes) in-tree with nvcc for sm_100a (no JIT, no torch extension cache)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# PRNG_B200_CHECKED=1: the test-only checked build (device bounds checks that trap,
# -DPRNG_CHECKED, prng_kernels.cuh) in libprng_b200_checked.so; the package then loads it.
CHECKED = os.environ.get("PRNG_B200_CHECKED") == "1"
DEFAULT_LIB = os.path.join(PKG, "libprng_b200.so")
CHECKED_LIB = os.path.join(PKG, "libprng_b200_checked.so")
LIB = CHECKED_LIB if CHECKED else DEFAULT_LIB
SOURCES = [os.path.join(CSRC, f) for f in
           ("prng_engine.cu", "prng_pipeline.cu", "prng_prof.cpp", "prng_sinks.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, "prng_kernels.cuh"), os.path.join(CSRC, "engine_internal.h"),
                  os.path.join(ROOT, "include", "prng.h"), os.path.join(ROOT, "include", "prng_sinks.h")]
PROBES_LIB = os.path.join(PKG, "libprng_probes.so")
PROBES_SOURCES = [os.path.join(CSRC, "prng_probes.cu")]
PROBES_DEPS = PROBES_SOURCES + [os.path.join(ROOT, "include", "prng_probes.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2,-Wall",
    "-Xptxas", "-v",
    "-shared",
]


def needs_build(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(d) > t for d in DEPS)


CLI_SRC = os.path.join(CSRC, "rng_cli.c")
CLI = os.path.join(PKG, "bin", "rng_b200")


def build_cli(force: bool = False) -> str:
    """The paper's example program (NEXT-1), linked against libprng_b200.so."""
    if not force and os.path.exists(CLI) and os.path.getmtime(CLI) >= max(
            os.path.getmtime(CLI_SRC), os.path.getmtime(LIB), os.path.getmtime(os.path.join(ROOT, "include", "prng.h"))):
        return CLI
    os.makedirs(os.path.dirname(CLI), exist_ok=True)
    tmp = CLI + f".tmp{os.getpid()}"
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-D_POSIX_C_SOURCE=200809L", "-I", os.path.join(ROOT, "include"),
           "-o", tmp, CLI_SRC, "-L", PKG, "-l:libprng_b200.so", "-Wl,-rpath,$ORIGIN/.."]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"gcc failed ({r.returncode}): {' '.join(cmd)}")
    os.replace(tmp, CLI)
    return CLI


def build_probes(force: bool = False) -> str:
    """libprng_probes.so: measurement probes only, no code shared with libprng_b200.so."""
    if not force and os.path.exists(PROBES_LIB) and all(
            os.path.getmtime(d) <= os.path.getmtime(PROBES_LIB) for d in PROBES_DEPS):
        return PROBES_LIB
    tmp = PROBES_LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", tmp, *PROBES_SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed ({r.returncode}): {' '.join(cmd)}")
    os.replace(tmp, PROBES_LIB)
    return PROBES_LIB


def build(force: bool = False, verbose: bool = False, checked: bool = CHECKED, probes: bool = True) -> str:
    """The hot-path library (checked: its bounds-checked test build) and the probes."""
    if probes:
        build_probes(force)
    lib = CHECKED_LIB if checked else DEFAULT_LIB
    if not force and not needs_build(lib):
        if not checked:
            build_cli()
        return lib
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *NVCC_FLAGS, *(["-DPRNG_CHECKED"] if checked else []), "-I", os.path.join(ROOT, "include"), "-o",
           tmp, *SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed ({r.returncode}): {' '.join(cmd)}")
    if not checked:
        with open(os.path.join(CSRC, "ptxas_info.txt"), "w") as f:
            f.write(r.stderr)
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, lib)
    if not checked:  # the CLI links the default library
        build_cli(force=True)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
