"""Profiler arithmetic oracle (row a6) -- TEST INFRASTRUCTURE, see oracle/__init__.py.

Plain definitions of what cf4ocl's ``ccl_prof_calc`` reports (§4.3,
Fig. 3), in the concrete reading of S:391 (profiler/prof_calc):

* aggregate  : group events by name; abs = sum(end - start); rel = abs / sum of all abs
               ("Absolute and relative durations of all events with same name").
* overlaps   : for every unordered pair of distinct events (i, j), from any queue,
               ov = max(0, min(end_i, end_j) - max(start_i, start_j)); add ov > 0 into the
               bucket of the unordered name pair ("event overlaps").
* effective  : measure of the union of all [start, end) intervals
               (Fig. 3 "Tot. of all events (eff.)").
* elapsed    : given wall time, else max end - min start (Fig. 3 "Total ellapsed time").
* device     : effective / elapsed; host = 1 - device (Fig. 3).

Deliberately brute force: O(E^2) pairs and an endpoint-discretised timeline for the
union, so a reader can check it against the definition by eye.
"""
from __future__ import annotations


def aggregate(events):
    """events: iterable of (name, start, end). Returns {name: (abs, rel)}."""
    tot = {}
    for name, s, e in events:
        tot[name] = tot.get(name, 0) + (e - s)
    total = sum(tot.values())
    return {n: (a, (a / total if total else 0.0)) for n, a in tot.items()}


def overlaps(events):
    """{frozenset-like sorted (name_a, name_b): total overlap} over all unordered pairs."""
    ev = list(events)
    out = {}
    for i in range(len(ev)):
        for j in range(i + 1, len(ev)):
            ni, si, ei = ev[i]
            nj, sj, ej = ev[j]
            ov = min(ei, ej) - max(si, sj)
            if ov > 0:
                key = tuple(sorted((ni, nj)))
                out[key] = out.get(key, 0) + ov
    return out


def effective(events):
    """Measure of the union of the intervals: discretise on all endpoints and add every
    elementary segment that at least one interval covers."""
    ev = [(s, e) for _, s, e in events if e > s]
    pts = sorted({p for s, e in ev for p in (s, e)})
    tot = 0
    for a, b in zip(pts, pts[1:]):
        if any(s <= a and b <= e for s, e in ev):
            tot += b - a
    return tot


def report(events, elapsed=None):
    ev = list(events)
    agg = aggregate(ev)
    ovl = overlaps(ev)
    eff = effective(ev)
    if elapsed is None:
        elapsed = (max(e for _, _, e in ev) - min(s for _, s, _ in ev)) if ev else 0
    dev = eff / elapsed if elapsed else 0.0
    return {
        "aggregate": agg,
        "total": sum(a for a, _ in agg.values()),
        "overlaps": ovl,
        "effective": eff,
        "elapsed": elapsed,
        "device": dev,
        "host": 1.0 - dev,
    }
