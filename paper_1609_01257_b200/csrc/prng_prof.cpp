// prng_prof.cpp -- row a6: cf4ocl's profiler arithmetic (ccl_prof_calc, §4.3,
// Fig. 3) over the gen / copy / sink intervals recorded by the engine.
//
// Definitions: per-name sum of durations; for every unordered pair of DISTINCT
// events, their intersection added to the (name_a, name_b) bucket; "effective" = measure
// of the union of all intervals; elapsed = max end - min start unless given.
//
// Implementation: one endpoint sweep.  Between consecutive endpoints the set of active
// events is constant; with c[a] active events of name a over a segment of length L,
// distinct pairs contribute c[a]*c[b]*L to bucket (a, b), a < b, and c[a]*(c[a]-1)/2*L
// to (a, a); the union gains L when any event is active.  O(E log E + S * nnames^2),
// versus the O(E^2) pair loop the paper calls "computationally expensive".
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <string>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/prng.h"

namespace {
int fail(prng_err_t *err, int code, const char *msg) {
    if (err) {
        err->code = code;
        std::snprintf(err->msg, sizeof(err->msg), "%s", msg);
    }
    return code;
}
}  // namespace

extern "C" int prng_prof_calc(uint64_t nevents, const uint32_t *name_id, const double *start_s,
                              const double *end_s, uint32_t nnames, double elapsed, double *agg_abs,
                              double *overlap, double *effective, double *elapsed_out, prng_err_t *err) {
    if (nnames == 0 || nnames > 4096 || !agg_abs || !overlap || !effective || !elapsed_out)
        return fail(err, PRNG_EINVAL, "prng_prof_calc: bad output arguments");
    if (nevents && (!name_id || !start_s || !end_s))
        return fail(err, PRNG_EINVAL, "prng_prof_calc: NULL event arrays");
    for (uint64_t i = 0; i < nevents; ++i) {
        if (name_id[i] >= nnames) return fail(err, PRNG_EINVAL, "prng_prof_calc: name id out of range");
        if (!(end_s[i] >= start_s[i])) return fail(err, PRNG_EINVAL, "prng_prof_calc: end < start");
    }
    std::fill(agg_abs, agg_abs + nnames, 0.0);
    std::fill(overlap, overlap + (size_t)nnames * nnames, 0.0);
    *effective = 0.0;

    struct Pt {
        double t;
        int delta;  // -1 end, +1 start (ends sort first at equal t: half-open intervals)
        uint32_t name;
    };
    std::vector<Pt> pts;
    pts.reserve(2 * nevents);
    double tmin = 0, tmax = 0;
    for (uint64_t i = 0; i < nevents; ++i) {
        agg_abs[name_id[i]] += end_s[i] - start_s[i];
        if (end_s[i] > start_s[i]) {
            pts.push_back({start_s[i], +1, name_id[i]});
            pts.push_back({end_s[i], -1, name_id[i]});
        }
        if (i == 0 || start_s[i] < tmin) tmin = start_s[i];
        if (i == 0 || end_s[i] > tmax) tmax = end_s[i];
    }
    std::sort(pts.begin(), pts.end(), [](const Pt &a, const Pt &b) {
        return a.t < b.t || (a.t == b.t && a.delta < b.delta);
    });
    std::vector<int64_t> c(nnames, 0);
    int64_t active = 0;
    for (size_t i = 0; i < pts.size(); ++i) {
        if (i > 0 && active > 0) {
            const double L = pts[i].t - pts[i - 1].t;
            if (L > 0) {
                *effective += L;
                if (active > 1) {
                    for (uint32_t a = 0; a < nnames; ++a) {
                        if (!c[a]) continue;
                        overlap[(size_t)a * nnames + a] += 0.5 * (double)(c[a] * (c[a] - 1)) * L;
                        for (uint32_t b = a + 1; b < nnames; ++b)
                            if (c[b]) overlap[(size_t)a * nnames + b] += (double)(c[a] * c[b]) * L;
                    }
                }
            }
        }
        c[pts[i].name] += pts[i].delta;
        active += pts[i].delta;
    }
    *elapsed_out = elapsed > 0 ? elapsed : (nevents ? tmax - tmin : 0.0);
    if (err) {
        err->code = PRNG_OK;
        err->msg[0] = 0;
    }
    return PRNG_OK;
}

// ---------------------------------------------------------------------------- summary (NEXT-2)
// ccl_prof_get_summary's layout, as printed in Fig. 3.  The figure's header
// line is cut at "Rel. time ("; it is read as "Rel. time (%)" / "Abs. time (s)"
// (A17).  "ellapsed" is spelled as printed.
namespace {
struct Appender {
    std::string s;
    void f(const char *fmt, ...) {
        char tmp[512];
        va_list ap;
        va_start(ap, fmt);
        std::vsnprintf(tmp, sizeof(tmp), fmt, ap);
        va_end(ap);
        s += tmp;
    }
};
const char *name_of(const char *const *names, uint32_t i) { return (names && names[i]) ? names[i] : prng_event_name(i); }
}  // namespace

extern "C" int prng_prof_summary(uint64_t nevents, const uint32_t *name_id, const double *start_s,
                                 const double *end_s, uint32_t nnames, const char *const *names, double elapsed,
                                 int agg_sort, int overlap_sort, char *buf, uint64_t cap, uint64_t *len,
                                 prng_err_t *err) {
    std::vector<double> agg(nnames ? nnames : 1), ov((size_t)(nnames ? nnames : 1) * (nnames ? nnames : 1));
    double eff = 0, el = 0;
    if (int rc = prng_prof_calc(nevents, name_id, start_s, end_s, nnames, elapsed, agg.data(), ov.data(), &eff, &el,
                                err))
        return rc;
    std::vector<char> seen(nnames, 0);
    for (uint64_t i = 0; i < nevents; ++i) seen[name_id[i]] = 1;
    double total = 0;
    std::vector<uint32_t> ids;
    for (uint32_t i = 0; i < nnames; ++i)
        if (seen[i]) {
            ids.push_back(i);
            total += agg[i];
        }
    const bool adesc = agg_sort & PRNG_PROF_SORT_DESC, aby_time = agg_sort & PRNG_PROF_AGG_SORT_TIME;
    std::stable_sort(ids.begin(), ids.end(), [&](uint32_t x, uint32_t y) {
        if (aby_time) return adesc ? agg[x] > agg[y] : agg[x] < agg[y];
        const int c = std::strcmp(name_of(names, x), name_of(names, y));
        return adesc ? c > 0 : c < 0;
    });
    Appender o;
    const char *rule = "   ------------------------------------------------------------------\n";
    o.f(" Aggregate times by event  :\n");
    o.s += rule;
    o.f("   | %-30s | %13s | %13s |\n", "Event name", "Rel. time (%)", "Abs. time (s)");
    o.s += rule;
    for (uint32_t i : ids)
        o.f("   | %-30s | %13.4f | %13.4e |\n", name_of(names, i), total > 0 ? 100.0 * agg[i] / total : 0.0, agg[i]);
    o.s += rule;
    o.f("                                    | %13s | %13.4e |\n", "Total", total);
    o.f("                                    ---------------------------------\n");
    struct Pair {
        uint32_t a, b;
        double v;
    };
    std::vector<Pair> pairs;
    double ovt = 0;
    for (uint32_t a = 0; a < nnames; ++a)
        for (uint32_t b = a; b < nnames; ++b)
            if (ov[(size_t)a * nnames + b] > 0) {
                pairs.push_back({a, b, ov[(size_t)a * nnames + b]});
                ovt += ov[(size_t)a * nnames + b];
            }
    const bool odesc = overlap_sort & PRNG_PROF_SORT_DESC, oby_dur = overlap_sort & PRNG_PROF_OVERLAP_SORT_DURATION;
    std::stable_sort(pairs.begin(), pairs.end(), [&](const Pair &x, const Pair &y) {
        if (oby_dur) return odesc ? x.v > y.v : x.v < y.v;
        int c = std::strcmp(name_of(names, x.a), name_of(names, y.a));
        if (!c) c = std::strcmp(name_of(names, x.b), name_of(names, y.b));
        return odesc ? c > 0 : c < 0;
    });
    if (!pairs.empty()) {
        o.f(" Event overlaps            :\n");
        o.s += rule;
        o.f("   | %-22s | %-22s | %-12s |\n", "Event 1", "Event2", "Overlap (s)");
        o.s += rule;
        for (const auto &p : pairs) o.f("   | %-22s | %-22s | %12.4e |\n", name_of(names, p.a), name_of(names, p.b), p.v);
        o.s += rule;
        o.f("                            | %22s | %12.4e |\n", "Total", ovt);
        o.f("                            -----------------------------------------\n");
    }
    o.f(" Tot. of all events (eff.) : %es\n", eff);
    o.f(" Total ellapsed time       : %es\n", el);
    const double dev = el > 0 ? eff / el : 0.0;
    o.f(" Time spent in device      : %.2f%%\n", 100.0 * dev);
    o.f(" Time spent in host        : %.2f%%\n", 100.0 * (1.0 - dev));
    if (len) *len = o.s.size();
    if (!buf || cap < o.s.size() + 1) {
        if (err) {
            err->code = PRNG_EINVAL;
            std::snprintf(err->msg, sizeof(err->msg), "summary needs %zu bytes", o.s.size() + 1);
        }
        return PRNG_EINVAL;
    }
    std::memcpy(buf, o.s.c_str(), o.s.size() + 1);
    if (err) {
        err->code = PRNG_OK;
        err->msg[0] = 0;
    }
    return PRNG_OK;
}

// ---------------------------------------------------------------------------- export (NEXT-2)
extern "C" int prng_prof_export(uint64_t nevents, const uint32_t *name_id, const double *start_s,
                                const double *end_s, uint32_t nnames, const char *const *names,
                                const char *const *queues, const char *path, prng_err_t *err) {
    if (!path || (nevents && (!name_id || !start_s || !end_s))) return fail(err, PRNG_EINVAL, "prng_prof_export: NULL");
    struct Row {
        long long a, b;
        std::string q, n;
    };
    std::vector<Row> rows;
    for (uint64_t i = 0; i < nevents; ++i) {
        const uint32_t id = name_id[i];
        if (id >= nnames) return fail(err, PRNG_EINVAL, "prng_prof_export: name id out of range");
        const char *q = (queues && queues[id]) ? queues[id]
                        : id == PRNG_EV_READ_BUFFER ? "Comms"
                        : id == PRNG_EV_OUT         ? "Host"
                                                    : "Main";
        rows.push_back({std::llround(start_s[i] * 1e9), std::llround(end_s[i] * 1e9), q, name_of(names, id)});
    }
    std::stable_sort(rows.begin(), rows.end(), [](const Row &x, const Row &y) {
        if (x.a != y.a) return x.a < y.a;
        if (x.b != y.b) return x.b < y.b;
        return x.q < y.q;
    });
    FILE *f = std::fopen(path, "w");
    if (!f) return fail(err, PRNG_EINVAL, "prng_prof_export: cannot open file");
    for (const auto &r : rows) std::fprintf(f, "%s\t%lld\t%lld\t%s\n", r.q.c_str(), r.a, r.b, r.n.c_str());
    const bool bad = std::fclose(f) != 0;
    if (bad) return fail(err, PRNG_EINVAL, "prng_prof_export: write failed");
    if (err) {
        err->code = PRNG_OK;
        err->msg[0] = 0;
    }
    return PRNG_OK;
}
