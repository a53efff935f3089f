"""B200-native massive-PRNG hot path of arXiv 1609.01257 §5 (cf4ocl's example application).

Thin Python binding of the C ABI in ``include/prng.h`` / ``include/prng_sinks.h``: the
functions below carry the same names and only marshal arguments (ctypes) -- every step of
the path runs in the sm_100a kernels and the C++ engine of ``libprng_b200.so``.  There is
no CPU fallback: if the library is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from ._build import LIB, PROBES_LIB, build as _build_lib

__all__ = [
    "PrngError", "lib", "probes_lib", "prng_create", "prng_create_range", "prng_destroy", "prng_get_range", "prng_init",
    "prng_generate", "prng_generate_device", "prng_generate_host", "prng_seek", "prng_device_ring", "prng_read_slot",
    "prng_read_state", "prng_set_option", "prng_get_option", "prng_set_streams",
    "prng_strerror", "prng_prof_events", "prng_prof_calc", "prng_event_name",
    "prng_kernel_variants", "prng_kernel_variant_name", "prng_last_launch", "prng_autotune", "prng_probe_memset_gbs",
    "prng_probe_store_gbs", "prng_probe_fill_gbs", "prng_probe_d2h_gbs",
    "prng_probe_d2h_sustained_gbs", "SINK_NULL", "SINK_COPY", "SINK_DIGEST",
    "CopySink", "DigestSink", "SINK_FN",
    "PRNG_OPT_MODE", "PRNG_OPT_BATCH_ITERS", "PRNG_OPT_RING_SLOTS", "PRNG_OPT_PROFILE",
    "PRNG_OPT_KERNEL", "PRNG_OPT_GRID_WARPS", "PRNG_OPT_RING_PAD", "PRNG_OPT_HOST_MEM", "PRNG_OPT_CHUNK_ITERS",
    "PRNG_OPT_PIECE_ORDER", "PRNG_OPT_EPOCH_ITERS", "PRNG_OPT_FUSED_SEED", "PRNG_OPT_ONE_SHOT", "prng_last_grid", "PRNG_MODE_ZEROCOPY", "PRNG_MODE_SERIAL", "PRNG_MODE_PAGEABLE",
    "PRNG_MODE_OVERLAP1", "PRNG_MODE_OVERLAP2", "EV_NAMES",
]

# ---------------------------------------------------------------- constants (include/prng.h)
PRNG_OK, PRNG_EINVAL, PRNG_ESTATE, PRNG_ENOMEM, PRNG_ECUDA, PRNG_ESINK = 0, -1, -2, -3, -4, -5
PRNG_OPT_MODE, PRNG_OPT_BATCH_ITERS, PRNG_OPT_RING_SLOTS = 1, 2, 3
PRNG_OPT_PROFILE, PRNG_OPT_KERNEL, PRNG_OPT_GRID_WARPS, PRNG_OPT_RING_PAD, PRNG_OPT_HOST_MEM = 4, 5, 6, 7, 8
PRNG_OPT_OUTPUT, PRNG_OPT_TIME_PARALLEL, PRNG_OPT_BLOCKING, PRNG_OPT_CTA_WARPS = 10, 11, 12, 13
PRNG_OPT_CHUNK_ITERS, PRNG_OPT_PIECE_ORDER, PRNG_OPT_EPOCH_ITERS, PRNG_OPT_FUSED_SEED = 14, 15, 16, 17
PRNG_OPT_ONE_SHOT = 18
PRNG_MODE_SERIAL, PRNG_MODE_PAGEABLE, PRNG_MODE_OVERLAP1, PRNG_MODE_OVERLAP2, PRNG_MODE_ZEROCOPY = 0, 1, 2, 3, 4
EV_NAMES = ("INIT_KERNEL", "RNG_KERNEL", "READ_BUFFER", "OUT")

u64, u32, i32, i64, dbl = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_int64, ctypes.c_double
vp = ctypes.c_void_p
P64 = ctypes.POINTER(ctypes.c_uint64)
P32 = ctypes.POINTER(ctypes.c_uint32)
PD = ctypes.POINTER(ctypes.c_double)


class prng_err_t(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int), ("msg", ctypes.c_char * 256)]


class CopySink(ctypes.Structure):
    _fields_ = [("dst", P64), ("dst_pitch", u64), ("iter_offset", u64), ("iters", u64), ("gid_offset", u64)]


class DigestSink(ctypes.Structure):
    _fields_ = [("xor_out", P64), ("sum_out", P64), ("iter_offset", u64), ("iters", u64), ("wsum_out", P64)]


SINK_FN = ctypes.CFUNCTYPE(ctypes.c_int, vp, u64, u32, u64, u64, P64)


class PrngError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_lib = None


def lib():
    """Load libprng_b200.so (building it with nvcc if the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    if os.environ.get("PRNG_B200_NO_BUILD") is None:
        _build_lib()  # no-op when libprng_b200.so is newer than its sources
    if not os.path.exists(LIB):
        raise PrngError(PRNG_ECUDA, f"{LIB} missing: the CUDA path is not built (no CPU fallback)")
    L = ctypes.CDLL(LIB)
    E = ctypes.POINTER(prng_err_t)
    sig = {
        "prng_strerror": ([i32], ctypes.c_char_p),
        "prng_create": ([u64, u64, E], vp),
        "prng_create_range": ([u64, u64, u64, u64, i32, E], vp),
        "prng_destroy": ([vp], None),
        "prng_get_range": ([vp, P64, P64, P64, E], i32),
        "prng_set_streams": ([vp, vp, vp, E], i32),
        "prng_init": ([vp, E], i32),
        "prng_seek": ([vp, u64, E], i32),
        "prng_generate": ([vp, u64, vp, vp, E], i32),
        "prng_generate_device": ([vp, u64, vp, u64, u64, vp, E], i32),
        "prng_device_ring": ([vp, ctypes.POINTER(vp), P64, P64, P64, P64, E], i32),
        "prng_generate_host": ([vp, u64, vp, u64, u64, E], i32),
        "prng_read_slot": ([vp, u64, vp, E], i32),
        "prng_read_state": ([vp, vp, E], i32),
        "prng_set_option": ([vp, i32, i64, E], i32),
        "prng_get_option": ([vp, i32, ctypes.POINTER(i64), E], i32),
        "prng_autotune": ([vp, u64, PD, E], i32),
        "prng_kernel_variants": ([], i32),
        "prng_kernel_variant_name": ([i32], ctypes.c_char_p),
        "prng_last_launch": ([vp, ctypes.POINTER(i32), P32, E], i32),
        "prng_last_grid": ([vp, P64, P32, P32, ctypes.POINTER(i32), E], i32),
        "prng_event_name": ([u32], ctypes.c_char_p),
        "prng_prof_events": ([vp, u64, vp, vp, vp, P64, PD, E], i32),
        "prng_prof_calc": ([u64, vp, vp, vp, u32, dbl, vp, vp, PD, PD, E], i32),
        "prng_prof_summary": ([u64, vp, vp, vp, u32, vp, dbl, i32, i32, vp, u64, P64, E], i32),
        "prng_prof_export": ([u64, vp, vp, vp, u32, vp, vp, ctypes.c_char_p, E], i32),
        "prng_sink_null": ([vp, u64, u32, u64, u64, P64], i32),
        "prng_sink_copy": ([vp, u64, u32, u64, u64, P64], i32),
        "prng_sink_digest": ([vp, u64, u32, u64, u64, P64], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes, f.restype = args, res
    _lib = L
    return L


_probes = None


def probes_lib():
    """Load libprng_probes.so: bench.py's same-box roofline probes (include/prng_probes.h),
    a library of its own, apart from the hot path's libprng_b200.so."""
    global _probes
    if _probes is not None:
        return _probes
    lib()  # builds both libraries when their sources are newer
    if not os.path.exists(PROBES_LIB):
        raise PrngError(PRNG_ECUDA, f"{PROBES_LIB} missing: the probes are not built")
    L = ctypes.CDLL(PROBES_LIB)
    sig = {
        "prng_probe_memset_gbs": ([u64, i32], dbl),
        "prng_probe_memset_sustained_gbs": ([u64, i32], dbl),
        "prng_probe_store_gbs": ([u64, i32], dbl),
        "prng_probe_fill_gbs": ([u64, i32], dbl),
        "prng_probe_d2h_gbs": ([u64, i32, i32, i32], dbl),
        "prng_probe_d2h_sustained_gbs": ([u64, i32], dbl),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes, f.restype = args, res
    _probes = L
    return L


def _sinkptr(name):
    return ctypes.cast(getattr(lib(), name), vp).value


def __getattr__(name):  # SINK_NULL / SINK_COPY / SINK_DIGEST resolve lazily to C function pointers
    m = {"SINK_NULL": "prng_sink_null", "SINK_COPY": "prng_sink_copy", "SINK_DIGEST": "prng_sink_digest"}
    if name in m:
        return _sinkptr(m[name])
    raise AttributeError(name)


def _check(rc, err):
    if rc != 0:
        raise PrngError(rc, err.msg.decode(errors="replace"))


def _ptr(a: np.ndarray):
    return a.ctypes.data


# ---------------------------------------------------------------- the C ABI, same names
def prng_strerror(code: int) -> str:
    return lib().prng_strerror(code).decode()


def prng_create(numrn: int, seed: int = 0):
    err = prng_err_t()
    h = lib().prng_create(numrn, seed & 0xFFFFFFFFFFFFFFFF, ctypes.byref(err))
    if not h:
        raise PrngError(err.code, err.msg.decode(errors="replace"))
    return h


def prng_create_range(numrn_total: int, seed: int, gid_begin: int, gid_count: int, cuda_device: int = -1):
    err = prng_err_t()
    h = lib().prng_create_range(numrn_total, seed & 0xFFFFFFFFFFFFFFFF, gid_begin, gid_count, cuda_device,
                                ctypes.byref(err))
    if not h:
        raise PrngError(err.code, err.msg.decode(errors="replace"))
    return h


def prng_destroy(h) -> None:
    lib().prng_destroy(h)


def prng_get_range(h):
    """-> (numrn_total, gid_begin, count) of the handle."""
    err = prng_err_t()
    n, b, c = u64(), u64(), u64()
    _check(lib().prng_get_range(h, ctypes.byref(n), ctypes.byref(b), ctypes.byref(c), ctypes.byref(err)), err)
    return n.value, b.value, c.value


def prng_set_streams(h, gen_stream: int, copy_stream: int) -> None:
    err = prng_err_t()
    _check(lib().prng_set_streams(h, gen_stream, copy_stream, ctypes.byref(err)), err)


def prng_init(h) -> None:
    err = prng_err_t()
    _check(lib().prng_init(h, ctypes.byref(err)), err)


def prng_seek(h, iteration: int) -> None:
    """Re-seed and jump so that the next iteration emitted is `iteration` (checkpoint/resume)."""
    err = prng_err_t()
    _check(lib().prng_seek(h, iteration, ctypes.byref(err)), err)


def prng_generate(h, numiter: int, sink=None, user=None) -> None:
    """sink: None (device only), a C function pointer (int, e.g. SINK_NULL), or a Python
    callable f(iter_begin, iters, gid_begin, count, ndarray[iters, count]) -> int."""
    err = prng_err_t()
    keep = None
    raised = []
    if sink is None:
        sp = None
    elif isinstance(sink, int):
        sp = sink
    else:
        def tramp(_u, k0, it, g0, cnt, data):
            try:
                arr = np.ctypeslib.as_array(data, shape=(it * cnt,)).reshape(it, cnt)
                return int(sink(k0, it, g0, cnt, arr) or 0)
            except BaseException as e:  # noqa: BLE001 -- abort generation, re-raise below
                raised.append(e)
                return 1
        keep = SINK_FN(tramp)
        sp = ctypes.cast(keep, vp).value
    up = ctypes.cast(ctypes.pointer(user), vp).value if isinstance(user, ctypes.Structure) else user
    rc = lib().prng_generate(h, numiter, sp, up, ctypes.byref(err))
    del keep
    if raised:
        raise raised[0]
    _check(rc, err)


def prng_generate_device(h, numiter: int, dst_ptr: int, dst_pitch: int, dst_slots: int, stream: int = 0) -> None:
    err = prng_err_t()
    _check(lib().prng_generate_device(h, numiter, dst_ptr, dst_pitch, dst_slots, stream or None,
                                      ctypes.byref(err)), err)


def prng_generate_host(h, numiter: int, dst: np.ndarray, dst_pitch: int, dst_rows: int, col_offset: int = 0) -> None:
    """D2H straight into a host array (shared-output multi-rank form): iteration k of the
    call -> dst.flat[(k % dst_rows) * dst_pitch + col_offset + j]."""
    if dst.dtype != np.uint64 or not dst.flags["C_CONTIGUOUS"] or not dst.flags["WRITEABLE"]:
        raise ValueError("dst must be a writeable C-contiguous uint64 array")
    count = prng_get_range(h)[2]
    if numiter >= 1 and dst_rows >= 1 and dst_pitch >= count:
        # the span the DMA writes: rows 0 .. min(rows, numiter)-1, columns col_offset .. +count
        need = (min(dst_rows, numiter) - 1) * dst_pitch + col_offset + count
        if col_offset < 0 or col_offset + count > dst_pitch or dst.size < need:
            raise ValueError(f"dst ({dst.size} u64) does not cover {need} u64 (rows {min(dst_rows, numiter)}, "
                             f"pitch {dst_pitch}, col_offset {col_offset}, count {count})")
    err = prng_err_t()
    _check(lib().prng_generate_host(h, numiter, dst.ctypes.data + 8 * col_offset, dst_pitch, dst_rows,
                                    ctypes.byref(err)), err)


def prng_device_ring(h):
    """-> (base, pitch, slots, iter0_slot, last_iter_end); iteration k sits in slot
    (iter0_slot + k) % slots."""
    err = prng_err_t()
    base, pitch, slots, first, end = vp(), u64(), u64(), u64(), u64()
    _check(lib().prng_device_ring(h, ctypes.byref(base), ctypes.byref(pitch), ctypes.byref(slots),
                                  ctypes.byref(first), ctypes.byref(end), ctypes.byref(err)), err)
    return base.value, pitch.value, slots.value, first.value, end.value


def prng_read_slot(h, slot: int, count: int | None = None) -> np.ndarray:
    n = prng_get_range(h)[2]
    if count is not None and count != n:
        raise ValueError(f"count {count} != the handle's count {n}")
    out = np.empty(n, dtype=np.uint64)
    err = prng_err_t()
    _check(lib().prng_read_slot(h, slot, _ptr(out), ctypes.byref(err)), err)
    return out


def prng_read_state(h, count: int | None = None) -> np.ndarray:
    n = prng_get_range(h)[2]
    if count is not None and count != n:
        raise ValueError(f"count {count} != the handle's count {n}")
    out = np.empty(n, dtype=np.uint64)
    err = prng_err_t()
    _check(lib().prng_read_state(h, _ptr(out), ctypes.byref(err)), err)
    return out


def prng_set_option(h, option: int, value: int) -> None:
    err = prng_err_t()
    _check(lib().prng_set_option(h, option, value, ctypes.byref(err)), err)


def prng_get_option(h, option: int) -> int:
    err = prng_err_t()
    v = i64()
    _check(lib().prng_get_option(h, option, ctypes.byref(v), ctypes.byref(err)), err)
    return v.value


def prng_autotune(h, probe_iters: int = 0) -> float:
    """Pick the fastest (kernel variant, warps per SM) for this handle's shape; returns the
    winner's probe GB/s.  The handle must be prng_init'ed again afterwards."""
    err = prng_err_t()
    best = dbl()
    _check(lib().prng_autotune(h, probe_iters, ctypes.byref(best), ctypes.byref(err)), err)
    return best.value


def prng_kernel_variants() -> int:
    return lib().prng_kernel_variants()


def prng_kernel_variant_name(i: int) -> str:
    r = lib().prng_kernel_variant_name(i)
    return r.decode() if r else None


def prng_last_launch(h):
    """(variant id, epoch iterations) of the handle's last batch launch."""
    err = prng_err_t()
    v, e = ctypes.c_int(-1), ctypes.c_uint32(0)
    _check(lib().prng_last_launch(h, ctypes.byref(v), ctypes.byref(e), ctypes.byref(err)), err)
    return v.value, e.value


def prng_last_grid(h):
    """(CTAs, threads per CTA, rounds of units per warp, one-shot?) of the handle's last
    batch launch (PRNG_OPT_ONE_SHOT)."""
    err = prng_err_t()
    b, t, r, o = u64(), ctypes.c_uint32(0), ctypes.c_uint32(0), ctypes.c_int(0)
    _check(lib().prng_last_grid(h, ctypes.byref(b), ctypes.byref(t), ctypes.byref(r), ctypes.byref(o),
                                ctypes.byref(err)), err)
    return b.value, t.value, r.value, bool(o.value)


def prng_event_name(i: int) -> str:
    return lib().prng_event_name(i).decode()


def prng_prof_events(h):
    """-> (name_id uint32[n], start_s float64[n], end_s float64[n], wall_s)."""
    err = prng_err_t()
    n, wall = u64(), dbl()
    _check(lib().prng_prof_events(h, 0, None, None, None, ctypes.byref(n), ctypes.byref(wall),
                                  ctypes.byref(err)), err)
    ids = np.zeros(n.value, np.uint32)
    s = np.zeros(n.value, np.float64)
    e = np.zeros(n.value, np.float64)
    _check(lib().prng_prof_events(h, n.value, _ptr(ids), _ptr(s), _ptr(e), ctypes.byref(n), ctypes.byref(wall),
                                  ctypes.byref(err)), err)
    return ids, s, e, wall.value


def prng_prof_calc(name_id, start_s, end_s, nnames: int = 4, elapsed: float = 0.0):
    """-> dict(agg=float64[nnames], overlap=float64[nnames, nnames] (upper triangle),
    effective=float, elapsed=float)."""
    ids = np.ascontiguousarray(name_id, dtype=np.uint32)
    s = np.ascontiguousarray(start_s, dtype=np.float64)
    e = np.ascontiguousarray(end_s, dtype=np.float64)
    agg = np.zeros(nnames, np.float64)
    ov = np.zeros((nnames, nnames), np.float64)
    eff, el = dbl(), dbl()
    err = prng_err_t()
    _check(lib().prng_prof_calc(len(ids), _ptr(ids), _ptr(s), _ptr(e), nnames, elapsed, _ptr(agg), _ptr(ov),
                                ctypes.byref(eff), ctypes.byref(el), ctypes.byref(err)), err)
    return {"agg": agg, "overlap": ov, "effective": eff.value, "elapsed": el.value}


PRNG_PROF_AGG_SORT_NAME, PRNG_PROF_AGG_SORT_TIME = 0x0, 0x1
PRNG_PROF_OVERLAP_SORT_NAME, PRNG_PROF_OVERLAP_SORT_DURATION = 0x0, 0x1
PRNG_PROF_SORT_ASC, PRNG_PROF_SORT_DESC = 0x0, 0x10


def _names_arg(names, nnames):
    if names is None:
        return None, None
    arr = (ctypes.c_char_p * nnames)(*[n.encode() if n is not None else None for n in names])
    return arr, arr


def prng_prof_summary(name_id, start_s, end_s, nnames: int = 4, names=None, elapsed: float = 0.0,
                      agg_sort: int = PRNG_PROF_AGG_SORT_TIME | PRNG_PROF_SORT_DESC,
                      overlap_sort: int = PRNG_PROF_OVERLAP_SORT_DURATION | PRNG_PROF_SORT_DESC) -> str:
    """Fig. 3-layout summary text."""
    ids = np.ascontiguousarray(name_id, dtype=np.uint32)
    s = np.ascontiguousarray(start_s, dtype=np.float64)
    e = np.ascontiguousarray(end_s, dtype=np.float64)
    arr, keep = _names_arg(names, nnames)
    n = u64()
    err = prng_err_t()
    lib().prng_prof_summary(len(ids), _ptr(ids), _ptr(s), _ptr(e), nnames, arr, elapsed, agg_sort, overlap_sort,
                            None, 0, ctypes.byref(n), ctypes.byref(err))
    buf = ctypes.create_string_buffer(n.value + 1)
    _check(lib().prng_prof_summary(len(ids), _ptr(ids), _ptr(s), _ptr(e), nnames, arr, elapsed, agg_sort,
                                   overlap_sort, buf, n.value + 1, ctypes.byref(n), ctypes.byref(err)), err)
    del keep
    return buf.value.decode()


def prng_prof_export(path: str, name_id, start_s, end_s, nnames: int = 4, names=None, queues=None) -> None:
    """Export table: queue, start ns, end ns, event name (tab-separated)."""
    ids = np.ascontiguousarray(name_id, dtype=np.uint32)
    s = np.ascontiguousarray(start_s, dtype=np.float64)
    e = np.ascontiguousarray(end_s, dtype=np.float64)
    narr, k1 = _names_arg(names, nnames)
    qarr, k2 = _names_arg(queues, nnames)
    err = prng_err_t()
    _check(lib().prng_prof_export(len(ids), _ptr(ids), _ptr(s), _ptr(e), nnames, narr, qarr, path.encode(),
                                  ctypes.byref(err)), err)
    del k1, k2


def prng_probe_memset_gbs(nbytes: int, reps: int = 5) -> float:
    return probes_lib().prng_probe_memset_gbs(nbytes, reps)


def prng_probe_memset_sustained_gbs(nbytes: int, reps: int = 100) -> float:
    return probes_lib().prng_probe_memset_sustained_gbs(nbytes, reps)


def prng_probe_store_gbs(nbytes: int, reps: int = 5) -> float:
    return probes_lib().prng_probe_store_gbs(nbytes, reps)


def prng_probe_fill_gbs(nbytes: int, reps: int = 5) -> float:
    return probes_lib().prng_probe_fill_gbs(nbytes, reps)


def prng_probe_d2h_gbs(nbytes: int, reps: int = 5, pinned: bool = True, nstreams: int = 1) -> float:
    return probes_lib().prng_probe_d2h_gbs(nbytes, reps, int(pinned), nstreams)


def prng_probe_d2h_sustained_gbs(nbytes: int, reps: int = 8) -> float:
    return probes_lib().prng_probe_d2h_sustained_gbs(nbytes, reps)
