"""CPU oracle for the massive-PRNG hot path (arXiv 1609.01257 §5) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The CUDA product path
(``paper_1609_01257_b200``) never imports it and shares no code with it.

``prng_oracle.c`` holds the plain definition (see its header for citations);
this module only compiles it with gcc and marshals arguments through ctypes.
``prof.py`` holds the profiler-arithmetic definitions.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "prng_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
# "plain, slow": -O2, scalar, no intrinsics, single-threaded.
CFLAGS = ["-O2", "-std=c99", "-fPIC", "-shared"]

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle/prng_oracle.c -> oracle/liboracle.so (gcc)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.run(["gcc", *CFLAGS, "-o", tmp, _SRC], check=True)
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        u32, u64, i32 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
        p64 = ctypes.POINTER(ctypes.c_uint64)
        L.orc_wang32.argtypes, L.orc_wang32.restype = [u32], u32
        L.orc_fmix64.argtypes, L.orc_fmix64.restype = [u64], u64
        L.orc_seed64.argtypes, L.orc_seed64.restype = [u32, u64], u64
        L.orc_xorshift64.argtypes, L.orc_xorshift64.restype = [u64], u64
        L.orc_sample.argtypes, L.orc_sample.restype = [u32, u64, u64], u64
        L.orc_stream.argtypes, L.orc_stream.restype = [u64, u64, u64, u64, u64, p64], i32
        L.orc_digest.argtypes, L.orc_digest.restype = [u64, u64, u64, u64, u64, p64, p64, p64, p64], i32
        L.orc_star.argtypes, L.orc_star.restype = [u64], u64
        L.orc_stream_star.argtypes, L.orc_stream_star.restype = [u64, u64, u64, u64, u64, p64], i32
        _lib = L
    return _lib


def _p64(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def wang32(x: int) -> int:
    return lib().orc_wang32(x & 0xFFFFFFFF)


def fmix64(z: int) -> int:
    return lib().orc_fmix64(z & 0xFFFFFFFFFFFFFFFF)


def seed64(gid: int, seed: int = 0) -> int:
    return lib().orc_seed64(gid & 0xFFFFFFFF, seed & 0xFFFFFFFFFFFFFFFF)


def xorshift64(x: int) -> int:
    return lib().orc_xorshift64(x & 0xFFFFFFFFFFFFFFFF)


def sample(gid: int, k: int, seed: int = 0) -> int:
    """out[k][gid] via the random-access form xs^k(seed64(gid, seed))."""
    return lib().orc_sample(gid & 0xFFFFFFFF, k, seed & 0xFFFFFFFFFFFFFFFF)


def stream(numrn: int, numiter: int, seed: int = 0, gid_begin: int = 0, count: int | None = None) -> np.ndarray:
    """The whole output, shape [numiter, count] uint64 (iteration-major, gid ascending)."""
    if count is None:
        count = numrn - gid_begin
    out = np.empty((numiter, count), dtype=np.uint64)
    rc = lib().orc_stream(numrn, numiter, seed & 0xFFFFFFFFFFFFFFFF, gid_begin, count, _p64(out))
    if rc != 0:
        raise ValueError(f"orc_stream rc={rc}")
    return out


def stream_bytes(numrn: int, numiter: int, seed: int = 0) -> bytes:
    """The byte stream of Eq. 1 (8*n*i little-endian bytes, A8)."""
    return stream(numrn, numiter, seed).astype("<u8").tobytes()


def digest(numrn: int, numiter: int, seed: int = 0, gid_begin: int = 0, count: int | None = None):
    """Per-iteration (xor, sum mod 2^64) folds of the outputs: two uint64[numiter] arrays."""
    r = folds(numrn, numiter, seed, gid_begin, count)
    return r["xor"], r["sum"]


def folds(numrn: int, numiter: int, seed: int = 0, gid_begin: int = 0, count: int | None = None,
          last: bool = False) -> dict:
    """One pass of the flat loop: per-iteration xor, sum and gid-weighted sum
    (sum of (2 g + 1) out[k][g] mod 2^64, g global) as uint64[numiter] arrays, plus
    (last=True) the final iteration out[numiter-1][gid_begin:gid_begin+count]."""
    if count is None:
        count = numrn - gid_begin
    x = np.empty(numiter, dtype=np.uint64)
    s = np.empty(numiter, dtype=np.uint64)
    w = np.empty(numiter, dtype=np.uint64)
    lo = np.empty(count if last else 0, dtype=np.uint64)
    rc = lib().orc_digest(numrn, numiter, seed & 0xFFFFFFFFFFFFFFFF, gid_begin, count, _p64(x), _p64(s), _p64(w),
                          _p64(lo) if last else None)
    if rc != 0:
        raise ValueError(f"orc_digest rc={rc}")
    out = {"xor": x, "sum": s, "wsum": w}
    if last:
        out["last"] = lo
    return out


def star(x: int) -> int:
    """NEXT-3 output scrambler (A19): x * 0x2545F4914F6CDD1D mod 2^64."""
    return lib().orc_star(x & 0xFFFFFFFFFFFFFFFF)


def stream_star(numrn: int, numiter: int, seed: int = 0, gid_begin: int = 0, count: int | None = None) -> np.ndarray:
    """NEXT-3: the scrambled stream, shape [numiter, count] uint64."""
    if count is None:
        count = numrn - gid_begin
    out = np.empty((numiter, count), dtype=np.uint64)
    rc = lib().orc_stream_star(numrn, numiter, seed & 0xFFFFFFFFFFFFFFFF, gid_begin, count, _p64(out))
    if rc != 0:
        raise ValueError(f"orc_stream_star rc={rc}")
    return out
