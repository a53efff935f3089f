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
