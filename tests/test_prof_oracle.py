"""Pins of the profiler-arithmetic oracle (oracle/prof.py, row a6) against Fig. 3
 and against brute-force / closed-form properties."""
import numpy as np
import pytest

from oracle import prof


def test_fig3_relative_times(golden):
    """Fig. 3 'Aggregate times by event': rel = abs / total, 4 decimals."""
    g = golden("fig3_profile_summary.json")
    # Build single events with the figure's aggregate durations (disjoint in time).
    t, ev = 0.0, []
    for name, a in g["aggregate_abs_s"].items():
        ev.append((name, t, t + a))
        t += a + 1.0
    agg = prof.aggregate(ev)
    for name, pct in g["aggregate_rel_pct"].items():
        assert round(100 * agg[name][1], 4) == pytest.approx(pct, abs=1.5e-4)
    assert sum(a for a, _ in agg.values()) == pytest.approx(g["total_s"], rel=5e-5)


def test_fig3_effective_and_device_share(golden):
    """Fig. 3: total - overlap = effective (concurrency <= 2), and
    device = effective / elapsed = 82.30 %, host 17.70 %."""
    g = golden("fig3_profile_summary.json")
    rng, read, init = (g["aggregate_abs_s"][k] for k in ("RNG_KERNEL", "READ_BUFFER", "INIT_KERNEL"))
    ov = g["overlap_total_s"]
    # One concrete timeline with exactly those durations and that single overlap.
    ev = [("INIT_KERNEL", 0.0, init),
          ("READ_BUFFER", 1.0, 1.0 + read),
          ("RNG_KERNEL", 1.0 + read - ov, 1.0 + read - ov + rng)]
    r = prof.report(ev, elapsed=g["elapsed_s"])
    assert r["overlaps"][("READ_BUFFER", "RNG_KERNEL")] == pytest.approx(ov, rel=1e-9)
    assert r["effective"] == pytest.approx(g["effective_s"], rel=5e-6)   # table rounding
    assert round(100 * r["device"], 2) == g["device_pct"]
    assert round(100 * r["host"], 2) == g["host_pct"]
    assert round(100 * g["effective_s"] / g["elapsed_s"], 2) == g["device_pct"]


def _timeline_measure(ev, res):
    """Independent brute force: integer timeline, mark every covered tick."""
    if not ev:
        return 0
    T = max(e for _, _, e in ev)
    cov = np.zeros(T + 1, dtype=bool)
    for _, s, e in ev:
        cov[s:e] = True
    return int(cov.sum())


def test_union_and_overlap_bruteforce():
    r = np.random.default_rng(0)
    for trial in range(200):
        m = int(r.integers(0, 9))
        ev = []
        for _ in range(m):
            s = int(r.integers(0, 60))
            ev.append((str(r.choice(["A", "B", "C"])), s, s + int(r.integers(0, 25))))
        assert prof.effective(ev) == _timeline_measure(ev, 1)
        # pairwise overlap bucket totals by tick counting
        ov = prof.overlaps(ev)
        for key, val in ov.items():
            tot = 0
            for i in range(len(ev)):
                for j in range(i + 1, len(ev)):
                    if tuple(sorted((ev[i][0], ev[j][0]))) == key:
                        a = np.zeros(100, bool); a[ev[i][1]:ev[i][2]] = True
                        b = np.zeros(100, bool); b[ev[j][1]:ev[j][2]] = True
                        tot += int((a & b).sum())
            assert val == tot
        # concurrency <= 2  =>  union = sum - sum(overlaps)
        T = 100
        cnt = np.zeros(T, int)
        for _, s, e in ev:
            cnt[s:e] += 1
        if cnt.max(initial=0) <= 2:
            assert prof.effective(ev) == sum(e - s for _, s, e in ev) - sum(ov.values())


def test_single_queue_has_no_overlap():
    """Events of one in-order queue are disjoint -> no overlaps, union = sum."""
    ev = [("K", 0, 5), ("K", 5, 9), ("R", 12, 20)]
    assert prof.overlaps(ev) == {}
    assert prof.effective(ev) == 17
