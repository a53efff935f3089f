"""CPU-side checks of the C-ABI library (no GPU compute calls): it builds, loads, exports
every symbol include/*.h declares, validates arguments, fails loudly without a GPU, and its
host-side profiler arithmetic (row a6) matches oracle/prof.py."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1609_01257_b200 as P
from oracle import prof as oprof

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions(headers=("prng.h", "prng_sinks.h"), checked=False):
    """Functions include/ declares; declarations under #ifdef PRNG_CHECKED (the test-only
    checked build's) only with checked=True."""
    names = set()
    for h in headers:
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        if not checked:
            src = re.sub(r"#ifdef PRNG_CHECKED.*?#endif", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(prng_\w+)\s*\(", src, flags=re.M):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    P.lib()
    declared = _declared_functions()
    assert {"prng_create", "prng_init", "prng_generate", "prng_destroy", "prng_strerror",
            "prng_create_range", "prng_prof_calc", "prng_sink_null"} <= declared
    exported = _exported(P.LIB)
    missing = declared - exported
    assert not missing, f"declared in include/ but not exported: {missing}"


def _exported(path):
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    return {l.split()[-1] for l in out.splitlines() if l.strip()}


def test_probes_are_a_library_of_their_own():
    """bench.py's roofline probes (include/prng_probes.h) live in libprng_probes.so; the hot
    path's libprng_b200.so exports none of them, and the probes library none of the hot
    path's symbols."""
    P.probes_lib()
    probes = _declared_functions(("prng_probes.h",))
    assert {"prng_probe_memset_gbs", "prng_probe_fill_gbs", "prng_probe_d2h_sustained_gbs"} <= probes
    exported = _exported(P.PROBES_LIB)
    assert not probes - exported, probes - exported
    assert not {x for x in _exported(P.LIB) if x.startswith("prng_probe")}
    assert not {x for x in exported if x.startswith("prng_") and not x.startswith("prng_probe_")}


@pytest.mark.parametrize("which", ["LIB", "PROBES_LIB"])
def test_library_is_sm100a(which):
    P.probes_lib()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", getattr(P, which)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_strerror_total():
    assert P.prng_strerror(0) == "ok"
    assert P.prng_strerror(-5) == "sink aborted"
    assert P.prng_strerror(12345) == "unknown error 12345"


def test_create_validates_before_touching_the_device():
    for args in [(0, 0), ((1 << 32) + 1, 0)]:
        with pytest.raises(P.PrngError) as e:
            P.prng_create(*args)
        assert e.value.code == P.PRNG_EINVAL
    with pytest.raises(P.PrngError) as e:
        P.prng_create_range(100, 0, 90, 20)
    assert e.value.code == P.PRNG_EINVAL


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(P.PrngError) as e:
        P.prng_create(1024)
    assert e.value.code == P.PRNG_ECUDA


def test_null_handle_calls_fail_cleanly():
    err = P.prng_err_t()
    assert P.lib().prng_init(None, ctypes.byref(err)) == P.PRNG_EINVAL
    assert P.lib().prng_generate(None, 4, None, None, ctypes.byref(err)) == P.PRNG_EINVAL
    P.prng_destroy(None)  # NULL-safe


def test_variants_named():
    n = P.prng_kernel_variants()
    names = [P.prng_kernel_variant_name(i) for i in range(n)]
    assert names == ["auto", "v4n8s1a", "v4n4s1p", "v4n8s1", "v4n16s1", "v2n32s1", "v2n4s1", "v4n4s1", "v2n2s1"]
    assert n <= 12  # the product library carries no experiment variants
    assert P.prng_kernel_variant_name(n) is None
    assert [P.prng_event_name(i) for i in range(4)] == list(P.EV_NAMES)


# ---------------------------------------------------------------- a6: profiler arithmetic
def _compare(events, elapsed=None):
    names = sorted({n for n, _, _ in events}) or ["A"]
    idx = {n: i for i, n in enumerate(names)}
    ids = [idx[n] for n, _, _ in events]
    r = P.prng_prof_calc(ids, [s for _, s, _ in events], [e for _, _, e in events], len(names),
                         elapsed or 0.0)
    o = oprof.report(events, elapsed=elapsed)
    for n, (a, _) in o["aggregate"].items():
        assert r["agg"][idx[n]] == pytest.approx(a, abs=1e-9)
    for (a, b), v in o["overlaps"].items():
        i, j = sorted((idx[a], idx[b]))
        assert r["overlap"][i, j] == pytest.approx(v, abs=1e-9)
    tot_ov = sum(o["overlaps"].values())
    assert np.triu(r["overlap"]).sum() == pytest.approx(tot_ov, abs=1e-9)
    assert r["effective"] == pytest.approx(o["effective"], abs=1e-9)
    if events:
        assert r["elapsed"] == pytest.approx(o["elapsed"], abs=1e-12)


def test_prof_calc_matches_oracle_random():
    rng = np.random.default_rng(5)
    for _ in range(300):
        m = int(rng.integers(0, 12))
        ev = []
        for _ in range(m):
            s = int(rng.integers(0, 80))
            ev.append((str(rng.choice(["INIT_KERNEL", "RNG_KERNEL", "READ_BUFFER", "OUT"])), s,
                       s + int(rng.integers(0, 30))))
        _compare(ev)


def test_prof_calc_fig3(golden):
    """The Fig. 3 timeline through the C++ arithmetic."""
    g = golden("fig3_profile_summary.json")
    rng, read, init = (g["aggregate_abs_s"][k] for k in ("RNG_KERNEL", "READ_BUFFER", "INIT_KERNEL"))
    ov = g["overlap_total_s"]
    ids = [0, 2, 1]
    s = [0.0, 1.0, 1.0 + read - ov]
    e = [init, 1.0 + read, 1.0 + read - ov + rng]
    r = P.prng_prof_calc(ids, s, e, 4, g["elapsed_s"])
    assert r["overlap"][1, 2] == pytest.approx(ov, rel=1e-9)
    assert r["effective"] == pytest.approx(g["effective_s"], rel=5e-6)
    assert round(100 * r["effective"] / r["elapsed"], 2) == g["device_pct"]


def test_prof_calc_rejects_bad_input():
    with pytest.raises(P.PrngError):
        P.prng_prof_calc([5], [0.0], [1.0], 4)
    with pytest.raises(P.PrngError):
        P.prng_prof_calc([0], [2.0], [1.0], 4)


# ---------------------------------------------------------------- a6: properties (hypothesis)
from hypothesis import given, settings, strategies as st  # noqa: E402

_ev = st.lists(st.tuples(st.integers(0, 3), st.integers(0, 10_000), st.integers(0, 3_000)), max_size=25)


@settings(max_examples=200, deadline=None)
@given(_ev, st.integers(-50_000, 50_000))
def test_prof_calc_properties(evs, shift):
    """Union <= sum of durations; union >= longest event; union = sum - overlaps when no
    instant is covered three times; everything invariant under a time shift;
    per-name aggregates add up to the total."""
    ids = [i for i, _, _ in evs]
    s = [float(a) for _, a, _ in evs]
    e = [float(a + d) for _, a, d in evs]
    r = P.prng_prof_calc(ids, s, e, 4)
    total = sum(b - a for a, b in zip(s, e))
    assert r["agg"].sum() == pytest.approx(total)
    assert r["effective"] <= total + 1e-9
    if evs:
        assert r["effective"] >= max(b - a for a, b in zip(s, e)) - 1e-9
    rs = P.prng_prof_calc(ids, [x + shift for x in s], [x + shift for x in e], 4)
    assert rs["effective"] == pytest.approx(r["effective"]) and np.allclose(rs["overlap"], r["overlap"])
    cover = np.zeros(14_000, int)
    for a, b in zip(s, e):
        cover[int(a):int(b)] += 1
    if cover.max(initial=0) <= 2:
        assert r["effective"] == pytest.approx(total - np.triu(r["overlap"]).sum())


# ---------------------------------------------------------------- built-in sinks (plain host C)
def _sink_call(name, user, iter_begin, iters, gid_begin, count, data):
    f = getattr(P.lib(), name)
    return f(ctypes.cast(ctypes.pointer(user), ctypes.c_void_p), iter_begin, iters, gid_begin, count,
             data.ctypes.data_as(P.P64))


def test_sink_copy_checks_gid_and_iteration_range():
    """prng_sink_copy writes row k - iter_offset, columns gid - gid_offset; a batch whose gids
    or iterations fall outside the caller's array aborts (returns nonzero) untouched."""
    dst = np.zeros((2, 10), np.uint64)
    c = P.CopySink(dst.ctypes.data_as(P.P64), 10, 4, 2, 100)
    data = np.arange(1, 23, dtype=np.uint64)
    for it0, its, g0, cnt in [(4, 1, 95, 5), (4, 1, 100, 11), (4, 1, 106, 5), (3, 1, 100, 5), (5, 2, 100, 5)]:
        assert _sink_call("prng_sink_copy", c, it0, its, g0, cnt, data) != 0, (it0, its, g0, cnt)
    assert not dst.any()
    assert _sink_call("prng_sink_copy", c, 4, 2, 105, 5, data) == 0
    assert dst[0, 5:].tolist() == list(range(1, 6)) and dst[1, 5:].tolist() == list(range(6, 11))
    assert not dst[:, :5].any()


def test_sink_digest_folds():
    """prng_sink_digest: per-iteration XOR, wrapping sum and sum (2 g + 1) x with the global
    gid, accumulated over calls (shards combine); wsum_out may be NULL."""
    M = (1 << 64) - 1
    r = np.random.default_rng(8)
    data = r.integers(0, 1 << 63, size=2 * 6, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    x, s, w = (np.zeros(3, np.uint64) for _ in range(3))
    d = P.DigestSink(x.ctypes.data_as(P.P64), s.ctypes.data_as(P.P64), 10, 3, w.ctypes.data_as(P.P64))
    assert _sink_call("prng_sink_digest", d, 11, 2, 40, 6, data) == 0
    rows = data.reshape(2, 6).astype(object)
    for t in range(2):
        assert int(s[1 + t]) == sum(rows[t]) & M
        assert int(w[1 + t]) == sum((2 * (40 + j) + 1) * rows[t][j] for j in range(6)) & M
        xx = 0
        for v in rows[t]:
            xx ^= int(v)
        assert int(x[1 + t]) == xx
    assert x[0] == s[0] == w[0] == 0
    assert _sink_call("prng_sink_digest", d, 13, 1, 0, 6, data) != 0   # iteration 13 outside [10, 13)
    d2 = P.DigestSink(x.ctypes.data_as(P.P64), s.ctypes.data_as(P.P64), 10, 3, None)
    assert _sink_call("prng_sink_digest", d2, 10, 1, 0, 6, data) == 0   # no weighted output


def _sass_functions(path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    funcs, name = {}, None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            name = m.group(1)
            funcs[name] = []
        elif name:
            funcs[name].append(line)
    return funcs


def test_checked_build_traps_behind_every_kernel_store():
    """tools/gpu_checked.sh's library (the kernels' own bounds checks; compute-sanitizer is
    closed on the GPU pool): -DPRNG_CHECKED builds libprng_b200_checked.so, in which every
    seed / batch / epoch kernel carries a trap behind its ring-store and state-access checks;
    the default library has none."""
    import sys
    env = dict(os.environ, PRNG_B200_CHECKED="1")
    r = subprocess.run([sys.executable, "-c", "from paper_1609_01257_b200 import _build; print(_build.build())"],
                       env=env, capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    path = r.stdout.strip().splitlines()[-1]
    assert path.endswith("libprng_b200_checked.so") and path != P.LIB
    exported = _exported(path)
    assert _declared_functions(checked=True) <= exported
    assert "prng_checked_selftest" in exported and "prng_checked_selftest" not in _exported(P.LIB)
    checked = _sass_functions(path)
    plain = _sass_functions(P.LIB)
    assert set(checked) == set(plain)
    hot = [f for f in checked if re.search(r"seed_kernel|batch_kernel", f)]
    assert len(hot) >= 20, hot
    for f in hot:
        assert any("TRAP" in ln for ln in checked[f]), f"no trap in checked {f}"
    for f in plain:
        assert not any("TRAP" in ln for ln in plain[f]), f"trap in the default build's {f}"
