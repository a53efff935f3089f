// prng_engine.cu -- the C ABI of include/prng.h: handle lifecycle, options, kernel
// variants and their launch (a1, a2 + a3), the device-only ring, checkpoint/seek,
// autotune, interval capture (a6).  The end-to-end pipeline lives in prng_pipeline.cu,
// the roofline probes in prng_probes.cu, the built-in sinks in prng_sinks.cpp.
//
// Paper mapping (§5):
//   "main thread"  + Main queue  -> s_gen  (generation kernels)
//   "comms thread" + Comms queue -> s_copy (D2H) + the caller's thread (sink = `out`)
//   device-side double buffering -> two halves of a device ring of T-iteration batches
//   semaphores between the threads -> CUDA events (gen(j) -> copy(j); copy(j) -> gen(j+2))
//   limitation 2 (host-side dual buffer) -> two pinned host halves (mode O2)
//   limitation 3 (no vectorisation) -> NPT numbers per thread, vector stores
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "engine_internal.h"
#include "prng_kernels.cuh"

using namespace prng_detail;

namespace {

// ============================================================================ kernel variants
// Every variant: one warp owns a piece of 32 x NPT consecutive gids (VEC-wide vector stores,
// NPT numbers per thread), 4 warps per SM in one CTA, the CTA's warps meet at a barrier
// every iteration (so a CTA writes one contiguous chunk per iteration).  Each carries its
// scrambled-output (NEXT-3) and epoch-order (anti-absorption) instantiations.
// Round 1 measured ~40 more forms (free-running warps, cluster barriers, cache policies,
// barrier intervals, TMA bulk stores, interleaved vectors, a lean single-path loop); none
// was faster at the bench shape, and they were removed from the library in round 2
// (results: profiles/r1_sweeps.md, profiles/r1_l2_absorption.md; code: git history before
// the "strip experiment variants" commit).
using BatchFn = void (*)(prngk::BatchArgs);
struct Variant {
    const char *name;
    int vec, npt;                  // vector width (u64) and numbers per thread
    int warps_per_sm;              // default grid: resident warps per SM
    BatchFn fn, star;              // natural order: state output / xorshift64* output (NEXT-3)
    BatchFn epoch, epoch_star;     // epoch-major order (anti-absorption)
};
// AL: .aligned CTA barrier in uniform rounds; PP: ping-pong hot loop (prngk::run_piece)
#define VAR(name, vec, npt, al, pp)                                                             \
    {name, vec, npt, 4, prngk::batch_kernel<vec, npt, 0, al, pp>, prngk::batch_kernel<vec, npt, 1, al, pp>, \
     prngk::batch_kernel_epoch<vec, npt, 0, al>, prngk::batch_kernel_epoch<vec, npt, 1, al>}
// Measured on B200 at numrn = 2^24 x 1000 through a non-reused 64 GiB ring
// (profiles/r1_sweeps.md): 4 CTA-synchronised warps per SM writing 32-B vectors reach
// 6.6-6.9 TB/s with DRAM bytes = algorithmic bytes.
const Variant kVariants[] = {
    // id 0 "auto" (the default): resolved per launch by launch_batch -- v4n8s1a at >= 2^21
    // work-items per handle, v4n4s1p from 2^15, v2n2s1 below (measured), then
    // widened or run in epoch order by the anti-absorption rule.  Its own fields (= v4n4s1)
    // size the grid.
    VAR("auto", 4, 4, false, false),
    // the bench-shape default: one 32-B store per thread per vector, 8 numbers per thread
    // (2 KiB per warp-iteration), .aligned barrier in uniform rounds
    VAR("v4n8s1a", 4, 8, true, false),
    // the default below 2^21 work-items: 4 numbers per thread, ping-pong hot loop
    VAR("v4n4s1p", 4, 4, false, true),
    // the anti-absorption substitutes, 2 / 4 / 8 KiB per warp-iteration
    VAR("v4n8s1", 4, 8, false, false), VAR("v4n16s1", 4, 16, false, false), VAR("v2n32s1", 2, 32, false, false),
    // north_star's 16-byte form: two st.global.v2.u64 per thread per iteration (the round-1
    // default; bit-identical output, 1.5-3 % slower than the 32-B forms on B200)
    VAR("v2n4s1", 2, 4, false, false),
    // one 32-B store per thread, 4 numbers per thread (the round-1 default after v2n4s1)
    VAR("v4n4s1", 4, 4, false, false),
    // one 16-B store per thread, 2 numbers per thread: 64-gid pieces, so a small handle
    // spreads over more warps and each warp's iteration is shorter (latency-bound launches)
    VAR("v2n2s1", 2, 2, false, false),
};
#undef VAR
constexpr int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);
static_assert(kNumVariants <= kMaxVariants, "raise kMaxVariants");

}  // namespace


namespace prng_detail {


void free_host(int kind, void *p, size_t bytes) {
    if (!p) return;
    switch (kind) {
        case HK_PINNED:
        case HK_PINNED_WC:
        case HK_MAPPED: cudaFreeHost(p); break;
        case HK_HUGE_REGISTERED:
            cudaHostUnregister(p);
            munmap(p, bytes);
            break;
        default: std::free(p);
    }
}


void free_e2e(prng *h) {
    if (h->d_buf) cudaFree(h->d_buf);
    h->d_buf = nullptr;
    h->buf_T = 0;
    for (int i = 0; i < 2; ++i) {
        free_host(h->h_kind, h->h_buf[i], h->h_T * h->count * sizeof(uint64_t));
        h->h_buf[i] = h->h_dev[i] = nullptr;
    }
    h->h_T = 0;
    h->h_halves = 0;
}

void clear_prof(prng *h) {
    for (auto &iv : h->dev_iv) {
        cudaEventDestroy(iv.a);
        cudaEventDestroy(iv.b);
    }
    h->dev_iv.clear();
    h->host_iv.clear();
    if (h->ev_origin) cudaEventDestroy(h->ev_origin);
    h->ev_origin = nullptr;
    h->wall_s = 0;
}

int ensure_origin(prng *h, prng_err_t *err) {
    if (!h->profile || h->ev_origin) return PRNG_OK;
    CU(cudaEventCreate(&h->ev_origin));
    CU(cudaEventRecord(h->ev_origin, h->s_gen));
    CU(cudaEventSynchronize(h->ev_origin));
    h->host_origin = now_s();
    return PRNG_OK;
}

// Record-start helper for a profiled device interval on `s`.
int prof_begin(prng *h, cudaStream_t s, uint32_t name, prng_err_t *err) {
    if (!h->profile) return PRNG_OK;
    prng::DevIv iv{name, nullptr, nullptr};
    CU(cudaEventCreate(&iv.a));
    CU(cudaEventCreate(&iv.b));
    CU(cudaEventRecord(iv.a, s));
    h->dev_iv.push_back(iv);
    return PRNG_OK;
}
int prof_end(prng *h, cudaStream_t s, prng_err_t *err) {
    if (!h->profile) return PRNG_OK;
    CU(cudaEventRecord(h->dev_iv.back().b, s));
    return PRNG_OK;
}

// Persistent grid of a variant: at most one wave of resident warps.
// wps > 0: warps per SM chosen by the anti-absorption rule instead of the variant's.
static uint64_t max_grid_warps(const prng *h, int vid, int wps = 0) {
    const Variant &v = kVariants[vid];
    uint64_t w = (uint64_t)h->blocks_per_sm[vid] * h->num_sms * (kBlock / 32);
    if (h->grid_warps > 0)
        w = std::min<uint64_t>(w, (uint64_t)h->grid_warps);
    else if (wps > 0)
        w = std::min<uint64_t>(w, (uint64_t)wps * h->num_sms);
    else if (v.warps_per_sm > 0)
        w = std::min<uint64_t>(w, (uint64_t)v.warps_per_sm * h->num_sms);
    return std::max<uint64_t>(w, kBlock / 32);
}

// L2 absorption (profiles/r1_l2_absorption.md): in the natural order a warp
// runs one piece through all of a launch's iterations, so when the launch wraps a ring of
// R slots it rewrites the same R x (bytes per warp-iteration) every R iterations.  While
// the grid's live set -- R x warps x bytes per warp-iteration -- fits in L2, the rewrites
// hit dirty L2 lines and never reach DRAM (ncu: 12 % of the stores reach DRAM at
// numrn = 2^27 through 64 slots).  That is not sustained output bandwidth, so such launches
// are reorganised: a variant with more numbers per warp-iteration, or epoch order.
static uint64_t live_bytes(const prng *h, int vid, uint64_t nslots, int wps = 0) {
    const uint64_t piece = 32ull * kVariants[vid].npt;
    const uint64_t npieces = (h->count + piece - 1) / piece;
    return nslots * std::min<uint64_t>(max_grid_warps(h, vid, wps), npieces) * piece * sizeof(uint64_t);
}
static bool absorbs(const prng *h, int vid, uint64_t nslots, uint32_t iters, int wps = 0) {
    return iters > nslots && live_bytes(h, vid, nslots, wps) < 2 * (uint64_t)h->l2_bytes;
}
// Default-variant substitutes in order of numbers per warp-iteration (2, 4, 8 KiB):
// same CTA-synchronised 4-warps-per-SM structure as v4n4s1.
static const char *const kWideNames[] = {"v4n8s1", "v4n16s1", "v2n32s1"};
// "auto": one 32-B store per thread per iteration and a CTA barrier, 8 numbers per thread
// (2 KiB per warp-iteration, v4n8s1a: .aligned barrier in uniform rounds) from this many
// work-items per handle, 4 below (v4n4s1p: ping-pong hot loop, +2.5-3 % over v4n4s1 at the
// bench shape, exp35).  Measured on B200 (profiles/r1_sweeps.md,
// "Default"): v4n8s1 writes 7-9 % faster than v4n4s1 at 2^21..2^24 on some boxes and ties
// on others; v4n4s1 is ahead at 2^18 and 2^20.
constexpr uint64_t kAutoWideFrom = 1ull << 21;
// ... and v2n2s1 (64-gid pieces: more warps for a small handle, shorter iterations per
// warp) below this many: 5-25 % faster than v4n4s1p from 2^10 to 2^14 work-items at
// 10^2..10^4 iterations, slower from 2^15 at >= 10^3 (profiles/r2_fig4.md, raw_r2/m17).
constexpr uint64_t kAutoNarrowBelow = 1ull << 15;
// Shortest time-parallel chunk (iterations); see launch_batch.  48 measured at least as fast
// as 128 / 64 / 32 on the small-n cells and faster from 200 to 1000 iterations at <= 2^13
// work-items (profiles/r2_fig4.md "Round-2 session 3", raw_r2/m25).
constexpr uint64_t kTpMinChunk = 48;

// One-shot grids (PRNG_OPT_ONE_SHOT, profiles/r2_write_ceiling.md §7): a
// natural-order launch with many more pieces than one wave holds runs one piece per warp
// on a multi-wave grid of 4-warp CTAs, which the hardware dispatches in order as earlier
// CTAs retire.  Measured on B200 with 3 resident CTAs per SM (raw_r2/m38): from 2^20 to
// 2^24 work-items 2-7 % more DRAM write bandwidth than the persistent 4-warps-per-SM grid
// in a burst (2^21 x 1000: a tie) and 5.6 % more sustained under the power cap at the
// bench shape (7.09-7.10 vs 6.72 TB/s); at 2^19 (2.3 waves) 3-11 % slower.  Used from this
// many waves of resident one-shot warps on (2^20 with v4n4s1p / 2^21 with v4n8s1a: 4.6).
constexpr uint64_t kOneShotMinWaves = 4;

// Resident warps of a one-shot grid of variant vid (occupancy at kOneShotBlock threads of
// the instantiation this launch will run), queried once per handle.
// Resident one-shot CTAs per SM are capped at kOneShotCtasPerSm by giving each CTA an
// (unused) share of the SM's shared memory: more, shorter waves.  Measured (raw_r2/m37):
// at 2^22 work-items the uncapped grid (9 CTAs/SM, 3 waves) writes 6.41-6.43 TB/s, capped
// at 2 / 3 / 4 / 6 CTAs/SM 6.97-7.18 (persistent: 6.97-7.0); at 2^23-2^24 every cap is
// within 1 % of the uncapped grid (7.1-7.25 burst, 6.94-7.0 sustained).
constexpr int kOneShotCtasPerSm = 3;

static int oneshot_capacity(prng *h, int vid, BatchFn fn, uint64_t *warps, prng_err_t *err) {
    int &b = h->oneshot_blocks_per_sm[h->output == 1 ? 1 : 0][vid];
    if (b == 0) {
        int q = 0;
        CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->oneshot_smem));
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&q, fn, kOneShotBlock, h->oneshot_smem));
        b = std::max(q, 1);
    }
    *warps = (uint64_t)b * h->num_sms * (kOneShotBlock / 32);
    return PRNG_OK;
}

// Whether this launch of variant vid runs on a one-shot grid: the option allows it, the
// caller fixed neither the grid nor the work order, there are enough pieces (auto: at least
// kOneShotMinWaves waves), and the resident set does not let a wrapping launch rewrite
// L2-resident lines (the same live-set test as the persistent grid's, with the one-shot
// grid's resident warps).
static int oneshot_launch(prng *h, int vid, uint64_t nslots, uint32_t iters, bool *yes, prng_err_t *err) {
    *yes = false;
    if (h->one_shot == 0 || h->grid_warps > 0 || h->cta_warps > 0 || h->epoch_iters > 0 || h->chunk_iters > 0)
        return PRNG_OK;
    const Variant &v = kVariants[vid];
    const uint64_t piece = 32ull * v.npt;
    const uint64_t npieces = (h->count + piece - 1) / piece;
    uint64_t cap = 0;
    if (int rc = oneshot_capacity(h, vid, h->output == 1 ? v.star : v.fn, &cap, err)) return rc;
    if (h->one_shot == 1 && npieces < kOneShotMinWaves * cap) return PRNG_OK;
    if (iters > nslots && nslots * std::min(cap, npieces) * piece * sizeof(uint64_t) < 2 * (uint64_t)h->l2_bytes)
        return PRNG_OK;
    *yes = true;
    return PRNG_OK;
}

static int variant_id(const char *name) {
    for (int i = 0; i < kNumVariants; ++i)
        if (!std::strcmp(kVariants[i].name, name)) return i;
    return -1;
}

// Launch one batch of `iters` iterations (a2 + a3) into dst slots.
int launch_batch(prng *h, uint64_t *dst, uint64_t pitch, uint64_t nslots, uint64_t slot0, uint32_t iters,
                 bool first_is_state, cudaStream_t s, prng_err_t *err) {
    int vid = h->kernel;
    int wps = 0;  // warps per SM override (anti-absorption, second choice)
    bool oneshot = false;
    if (vid == 0) {  // "auto"
        vid = variant_id(h->count >= kAutoWideFrom ? "v4n8s1a" : h->count >= kAutoNarrowBelow ? "v4n4s1p" : "v2n2s1");
        // One-shot grid on the default variant, else on the narrowest wider one whose
        // one-shot resident set clears 2x L2 when the launch wraps a small ring (2^27 per
        // GPU through 64 slots: v4n16s1; 2^28 through 32: v2n32s1)
        if (int rc = oneshot_launch(h, vid, nslots, iters, &oneshot, err)) return rc;
        for (const char *nm : kWideNames) {
            if (oneshot) break;
            const int w = variant_id(nm);
            if (kVariants[w].npt * kVariants[w].vec <= kVariants[vid].npt * kVariants[vid].vec) continue;
            if (int rc = oneshot_launch(h, w, nslots, iters, &oneshot, err)) return rc;
            if (oneshot) vid = w;
        }
        // Anti-absorption, first choice: the narrowest wider variant whose live set exceeds
        // 2x L2 (output identical; measured honest and as fast).  Not with a user grid, and
        // not needed on a one-shot grid, whose resident set already clears it.
        if (!oneshot && h->epoch_iters == 0 && h->grid_warps == 0 && h->cta_warps == 0 &&
            absorbs(h, vid, nslots, iters)) {
            int widest = vid;
            bool found = false;
            for (const char *nm : kWideNames) {
                const int w = variant_id(nm);
                if (kVariants[w].npt * kVariants[w].vec <= kVariants[vid].npt * kVariants[vid].vec) continue;
                widest = w;
                if (!absorbs(h, w, nslots, iters)) {
                    vid = w;
                    found = true;
                    break;
                }
            }
            // second choice: the widest variant with twice the warps per SM (8), which
            // doubles the live set (numrn = 2^28 through 32 slots: 6.2 TB/s, ncu DRAM
            // bytes 99.6 % of the stores, vs 5.6 in epoch order; exp39)
            if (!found && !absorbs(h, widest, nslots, iters, 2 * kVariants[widest].warps_per_sm)) {
                vid = widest;
                wps = 2 * kVariants[widest].warps_per_sm;
                found = true;
            }
            // none clears 2x L2: epoch order below, on the widest variant (fewest units,
            // so the per-unit state round trip is amortised over the most stores) if it
            // still has a piece for every warp of the grid
            if (!found) {
                const uint64_t wp = 32ull * kVariants[widest].npt;
                if ((h->count + wp - 1) / wp >= max_grid_warps(h, widest)) vid = widest;
            }
        }
    } else if (int rc = oneshot_launch(h, vid, nslots, iters, &oneshot, err)) {
        return rc;
    }
    const Variant &v = kVariants[vid];
    BatchFn fn = h->output == 1 ? v.star : v.fn;
    prngk::BatchArgs a;
    a.dst = dst;
    a.pitch = pitch;
    a.nslots = (uint32_t)nslots;
    a.slot0 = (uint32_t)slot0;
    a.state = h->d_state;
    a.count = h->count;
    a.iters = iters;
    a.first_is_state = first_is_state ? 1u : 0u;
    a.nchunks = 1;
    a.chunk_len = iters;
    a.jump = nullptr;
    a.state_out = h->d_state;
    a.order = (uint32_t)h->piece_order;
    a.seeding = h->seed_pending ? 1u : 0u;  // a1 fused: this launch starts from the seeds
    a.seed = h->seed;
    a.gid_begin = h->gid_begin;

    const uint64_t piece = 32ull * v.npt;
    a.npieces = (h->count + piece - 1) / piece;
    // Persistent grid: at most one wave of resident warps; equalise pieces per warp.
    uint64_t max_warps = max_grid_warps(h, vid, wps);
    // Time-parallel mode (NEXT-4): when the pieces cannot fill the grid (small numrn), cut
    // the launch's iterations into chunks started by GF(2) jump-ahead, so that
    // pieces x chunks units fill it.
    uint64_t units = a.npieces;
    // (chunks >= kTpMinChunk = 48 iterations: the per-unit 64-step mat-vec costs about 27
    // iterations' worth of instructions, but such launches are latency-bound, not
    // issue-bound, so a shorter critical path wins)
    // Chunks of one piece run concurrently on different warps, so they are only used when
    // the launch does not wrap its slots (iters <= nslots): otherwise two chunks could
    // write the same slot and the earlier iteration could land last.
    // A time-parallel launch is latency-bound (each warp walks its chunk serially), so it
    // uses twice the warps per SM of the natural order unless the caller fixed the grid,
    // and at most one unit per warp: nch = floor(warps / pieces), used only from 3 chunks
    // (measured on the Fig. 4 cells, profiles/r2_fig4.md).
    uint64_t nch = 0;
    if (iters <= nslots && !oneshot) {
        if (h->chunk_iters > 0 && iters > (uint64_t)h->chunk_iters) {
            nch = (iters + h->chunk_iters - 1) / h->chunk_iters;  // PRNG_OPT_CHUNK_ITERS: forced
        } else if (h->time_parallel && iters >= 2 * kTpMinChunk) {
            const bool user_grid = h->grid_warps > 0 || h->cta_warps > 0;
            const uint64_t tp_warps = user_grid ? max_warps : max_grid_warps(h, vid, 2 * v.warps_per_sm);
            const uint64_t c = std::min<uint64_t>(tp_warps / a.npieces, iters / kTpMinChunk);
            if (c >= 3) {  // 2 chunks measured no faster than the natural order (2^16: -6 %)
                nch = c;
                if (!user_grid) {
                    wps = 2 * v.warps_per_sm;
                    max_warps = tp_warps;
                }
            }
        }
    }
    // Anti-absorption, fallback: epoch-major order (batch_kernel_epoch) with E = R, so an
    // address is rewritten only one whole epoch (the full ring) later.
    uint64_t E = 0;
    if (nch <= 1 && h->epoch_iters >= 0 && !oneshot) {
        if (h->epoch_iters > 0)
            E = (uint64_t)h->epoch_iters;  // PRNG_OPT_EPOCH_ITERS: forced
        else if (absorbs(h, vid, nslots, iters, wps))
            E = nslots;
        if (E >= iters) E = 0;
    }
    if (E > 0) {
        fn = h->output == 1 ? v.epoch_star : v.epoch;
        a.nchunks = (uint32_t)((iters + E - 1) / E);
        a.chunk_len = (uint32_t)E;
    } else if (nch > 1) {
        const uint64_t L = (iters + nch - 1) / nch;
        const uint64_t C = (iters + L - 1) / L;
        if (C > h->jump_cap) {
            if (h->d_jump) cudaFree(h->d_jump);
            h->d_jump = nullptr;
            h->jump_cap = 0;
            CU(cudaMalloc(&h->d_jump, C * 64 * sizeof(uint64_t)));
            h->jump_cap = C;
            h->jump_key[0] = 0;
        }
        const uint64_t e = first_is_state ? 0 : 1;
        if (h->jump_key[0] != C || h->jump_key[1] != L || h->jump_key[2] != e) {
            prngk::jump_columns_kernel<<<1, 64, 0, s>>>(h->d_jump, (uint32_t)C, (uint64_t)L, (uint32_t)e);
            CU(cudaGetLastError());
            h->jump_key[0] = C;
            h->jump_key[1] = L;
            h->jump_key[2] = e;
        }
        if (!h->d_state2)  // allocated on first use: small numrn only
            CU(cudaMalloc(&h->d_state2, pitch_for(h->count) * sizeof(uint64_t)));
        a.nchunks = (uint32_t)C;
        a.chunk_len = (uint32_t)L;
        a.jump = h->d_jump;
        a.state_out = h->d_state2;  // chunks read d_state; the last chunk writes the other half
        units = a.npieces * C;
    }
    uint64_t wpb, blocks;
    if (oneshot) {  // one unit per warp, 4-warp CTAs over as many waves as it takes
        wpb = kOneShotBlock / 32;
        blocks = (units + wpb - 1) / wpb;
    } else {
        const uint64_t rounds0 = (units + max_warps - 1) / max_warps;
        const uint64_t warps = (units + rounds0 - 1) / rounds0;
        // Spread the warps over all SMs: with <= 8 warps per SM use one CTA per SM of
        // ceil(warps / SMs) warps, else 256-thread CTAs.
        wpb = kBlock / 32;
        if (warps <= (uint64_t)h->num_sms * wpb) wpb = std::max<uint64_t>(1, (warps + h->num_sms - 1) / h->num_sms);
        if (h->cta_warps > 0) wpb = (uint64_t)h->cta_warps;  // PRNG_OPT_CTA_WARPS
        blocks = (warps + wpb - 1) / wpb;
    }
    if (blocks > 0x7FFFFFFFull) return set_err(err, PRNG_EINVAL, "grid of %llu CTAs", (unsigned long long)blocks);
    a.rounds = (uint32_t)((units + blocks * wpb - 1) / (blocks * wpb));
    h->last_kernel = vid;
    h->last_epoch = (uint32_t)E;
    h->last_blocks = blocks;
    h->last_threads = (uint32_t)(32 * wpb);
    h->last_rounds = a.rounds;
    h->last_one_shot = oneshot;
    if (int rc = prof_begin(h, s, PRNG_EV_RNG_KERNEL, err)) return rc;
    fn<<<(unsigned)blocks, (unsigned)(32 * wpb), oneshot ? h->oneshot_smem : 0, s>>>(a);
    if (a.jump) std::swap(h->d_state, h->d_state2);  // time-parallel: the final state is in the other half
    CU(cudaGetLastError());
    h->seed_pending = false;  // every launch writes the whole state array
    return prof_end(h, s, err);
}

// a1 as its own kernel (the paper's `init`) into d_state on s_gen.
static int seed_launch(prng *h, prng_err_t *err) {
    prngk::SeedArgs a{h->d_state, h->count, h->gid_begin, h->seed};
    const uint64_t pairs = (h->count + 1) / 2;
    const uint64_t max_blocks = (uint64_t)h->num_sms * 8;
    const uint64_t blocks = std::max<uint64_t>(1, std::min<uint64_t>((pairs + kBlock - 1) / kBlock, max_blocks));
    if (int rc = prof_begin(h, h->s_gen, PRNG_EV_INIT_KERNEL, err)) return rc;
    prngk::seed_kernel<<<(unsigned)blocks, kBlock, 0, h->s_gen>>>(a);
    CU(cudaGetLastError());
    return prof_end(h, h->s_gen, err);
}

int pipeline_events(prng *h, prng_err_t *err) {
    for (auto &e : h->pev)
        if (!e) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return PRNG_OK;
}

int materialize_seeds(prng *h, prng_err_t *err) {
    if (!h->seed_pending) return PRNG_OK;
    if (int rc = seed_launch(h, err)) return rc;
    h->seed_pending = false;
    return PRNG_OK;
}

int check_handle(prng *h, prng_err_t *err, bool need_init) {
    if (!h) return set_err(err, PRNG_EINVAL, "NULL handle");
    if (h->poisoned) return set_err(err, PRNG_ESTATE, "handle poisoned by an earlier error/abort; call prng_init");
    if (need_init && !h->inited) return set_err(err, PRNG_ESTATE, "prng_generate before prng_init");
    cudaError_t e = cudaSetDevice(h->device);
    if (e != cudaSuccess) return set_err(err, PRNG_ECUDA, "cudaSetDevice(%d): %s", h->device, cudaGetErrorString(e));
    return PRNG_OK;
}

}  // namespace prng_detail

// ============================================================================ C ABI
extern "C" {

const char *prng_strerror(int code) {
    switch (code) {
        case PRNG_OK: return "ok";
        case PRNG_EINVAL: return "invalid argument";
        case PRNG_ESTATE: return "bad state";
        case PRNG_ENOMEM: return "out of memory";
        case PRNG_ECUDA: return "CUDA error";
        case PRNG_ESINK: return "sink aborted";
        default: {
            static thread_local char buf[48];
            std::snprintf(buf, sizeof(buf), "unknown error %d", code);
            return buf;
        }
    }
}

const char *prng_event_name(uint32_t id) {
    static const char *names[PRNG_EV_NAMES] = {"INIT_KERNEL", "RNG_KERNEL", "READ_BUFFER", "OUT"};
    return id < PRNG_EV_NAMES ? names[id] : "UNKNOWN";
}

int prng_kernel_variants(void) { return kNumVariants; }
int prng_last_launch(const prng_t *h, int *variant, uint32_t *epoch_iters, prng_err_t *err) {
    if (!h) return set_err(err, PRNG_EINVAL, "NULL handle");
    if (variant) *variant = h->last_kernel;
    if (epoch_iters) *epoch_iters = h->last_epoch;
    return ok(err);
}
int prng_last_grid(const prng_t *h, uint64_t *blocks, uint32_t *threads, uint32_t *rounds, int *one_shot,
                   prng_err_t *err) {
    if (!h) return set_err(err, PRNG_EINVAL, "NULL handle");
    if (blocks) *blocks = h->last_blocks;
    if (threads) *threads = h->last_threads;
    if (rounds) *rounds = h->last_rounds;
    if (one_shot) *one_shot = h->last_one_shot ? 1 : 0;
    return ok(err);
}
const char *prng_kernel_variant_name(int id) { return (id >= 0 && id < kNumVariants) ? kVariants[id].name : nullptr; }

prng_t *prng_create_range(uint64_t numrn_total, uint64_t seed, uint64_t gid_begin, uint64_t gid_count,
                          int cuda_device, prng_err_t *err) {
    // A12: numrn is a cl_uint in the paper: 1 <= numrn <= 2^32.
    if (numrn_total < 1 || numrn_total > (1ull << 32)) {
        set_err(err, PRNG_EINVAL, "numrn %llu outside [1, 2^32]", (unsigned long long)numrn_total);
        return nullptr;
    }
    if (gid_count < 1 || gid_begin >= numrn_total || gid_count > numrn_total - gid_begin) {
        set_err(err, PRNG_EINVAL, "gid range [%llu, +%llu) outside [0, %llu)", (unsigned long long)gid_begin,
                (unsigned long long)gid_count, (unsigned long long)numrn_total);
        return nullptr;
    }
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        set_err(err, PRNG_ECUDA, "no CUDA device: %s", e != cudaSuccess ? cudaGetErrorString(e) : "count 0");
        return nullptr;
    }
    int dev = cuda_device;
    if (dev < 0) cudaGetDevice(&dev);
    if (dev >= ndev) {
        set_err(err, PRNG_EINVAL, "cuda device %d of %d", dev, ndev);
        return nullptr;
    }
    prng *h = new (std::nothrow) prng();
    if (!h) {
        set_err(err, PRNG_ENOMEM, "host allocation");
        return nullptr;
    }
    h->device = dev;
    if (const char *f = std::getenv("PRNG_B200_FAULT_AFTER")) h->fault_after = std::atoll(f);
    h->numrn_total = numrn_total;
    h->seed = seed;
    h->gid_begin = gid_begin;
    h->count = gid_count;
    auto bail = [&](const char *what, cudaError_t ce) -> prng_t * {
        set_err(err, ce == cudaErrorMemoryAllocation ? PRNG_ENOMEM : PRNG_ECUDA, "%s: %s", what, cudaGetErrorString(ce));
        prng_destroy(h);
        return nullptr;
    };
    if ((e = cudaSetDevice(dev)) != cudaSuccess) return bail("cudaSetDevice", e);
    if ((e = cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
        return bail("cudaDeviceGetAttribute(SMs)", e);
    cudaDeviceGetAttribute(&h->l2_bytes, cudaDevAttrL2CacheSize, dev);
    {   // dynamic shared memory per one-shot CTA that leaves room for kOneShotCtasPerSm
        int sm_smem = 0, reserved = 0, cta_max = 0;
        cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev);
        cudaDeviceGetAttribute(&cta_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        const int per = sm_smem / kOneShotCtasPerSm - reserved;
        h->oneshot_smem = (size_t)std::max(0, std::min(per, cta_max));
    }
    for (int i = 0; i < kNumVariants; ++i) {
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&h->blocks_per_sm[i], kVariants[i].fn, kBlock, 0)) !=
            cudaSuccess)
            return bail("cudaOccupancyMaxActiveBlocksPerMultiprocessor", e);
        if (h->blocks_per_sm[i] < 1) h->blocks_per_sm[i] = 1;
    }
    if ((e = cudaMalloc(&h->d_state, pitch_for(gid_count) * sizeof(uint64_t))) != cudaSuccess)
        return bail("cudaMalloc(state)", e);
    if ((e = cudaStreamCreateWithFlags(&h->s_gen, cudaStreamNonBlocking)) != cudaSuccess)
        return bail("cudaStreamCreate", e);
    if ((e = cudaStreamCreateWithFlags(&h->s_copy, cudaStreamNonBlocking)) != cudaSuccess)
        return bail("cudaStreamCreate", e);
    ok(err);
    return h;
}

int prng_get_range(const prng_t *h, uint64_t *numrn_total, uint64_t *gid_begin, uint64_t *count, prng_err_t *err) {
    if (!h) return set_err(err, PRNG_EINVAL, "NULL handle");
    if (numrn_total) *numrn_total = h->numrn_total;
    if (gid_begin) *gid_begin = h->gid_begin;
    if (count) *count = h->count;
    return ok(err);
}

prng_t *prng_create(uint64_t numrn, uint64_t seed, prng_err_t *err) {
    return prng_create_range(numrn, seed, 0, numrn, -1, err);
}

void prng_destroy(prng_t *h) {
    if (!h) return;
    cudaSetDevice(h->device);
    if (h->s_gen) cudaStreamSynchronize(h->s_gen);
    if (h->s_copy) cudaStreamSynchronize(h->s_copy);
    clear_prof(h);
    free_e2e(h);
    for (auto &e : h->pev)
        if (e) cudaEventDestroy(e);
    if (h->d_ring) cudaFree(h->d_ring);
    if (h->d_state) cudaFree(h->d_state);
    if (h->d_state2) cudaFree(h->d_state2);
    if (h->d_jump) cudaFree(h->d_jump);
    if (h->own_streams) {
        if (h->s_gen) cudaStreamDestroy(h->s_gen);
        if (h->s_copy) cudaStreamDestroy(h->s_copy);
    }
    delete h;
}

int prng_set_streams(prng_t *h, void *gen_stream, void *copy_stream, prng_err_t *err) {
    if (!h) return set_err(err, PRNG_EINVAL, "NULL handle");
    // validate before touching the handle: a rejected call leaves its streams as they were
    if (!gen_stream || !copy_stream || gen_stream == copy_stream)
        return set_err(err, PRNG_EINVAL, "need two distinct non-NULL streams");
    CU(cudaSetDevice(h->device));
    CU(cudaStreamSynchronize(h->s_gen));
    CU(cudaStreamSynchronize(h->s_copy));
    if (h->own_streams) {
        cudaStreamDestroy(h->s_gen);
        cudaStreamDestroy(h->s_copy);
    }
    h->s_gen = (cudaStream_t)gen_stream;
    h->s_copy = (cudaStream_t)copy_stream;
    h->own_streams = false;
    return ok(err);
}

int prng_set_option(prng_t *h, int option, int64_t value, prng_err_t *err) {
    if (!h) return set_err(err, PRNG_EINVAL, "NULL handle");
    switch (option) {
        case PRNG_OPT_MODE:
            if (value < PRNG_MODE_SERIAL || value > PRNG_MODE_ZEROCOPY) return set_err(err, PRNG_EINVAL, "bad mode");
            if (value != h->mode) free_e2e(h);
            h->mode = (int)value;
            break;
        case PRNG_OPT_BATCH_ITERS:
            if (value < 0 || value > (1 << 30)) return set_err(err, PRNG_EINVAL, "bad batch iters");
            if (value != h->batch_iters) free_e2e(h);
            h->batch_iters = value;
            break;
        case PRNG_OPT_RING_SLOTS:
            if (value < 0 || value > (1 << 30)) return set_err(err, PRNG_EINVAL, "bad ring slots");
            if (value != h->ring_slots_opt && h->d_ring) {
                cudaSetDevice(h->device);
                cudaStreamSynchronize(h->s_gen);
                cudaFree(h->d_ring);
                h->d_ring = nullptr;
                h->ring_slots = 0;
            }
            h->ring_slots_opt = value;
            break;
        case PRNG_OPT_PROFILE:
            if (value < 0 || value > 2) return set_err(err, PRNG_EINVAL, "bad profile mode");
            if (value != h->profile) {
                cudaSetDevice(h->device);
                cudaStreamSynchronize(h->s_gen);
                cudaStreamSynchronize(h->s_copy);
                clear_prof(h);
            }
            h->profile = (int)value;
            break;
        case PRNG_OPT_BLOCKING:
            h->blocking = value ? 1 : 0;
            break;
        case PRNG_OPT_KERNEL:
            if (value < 0 || value >= kNumVariants) return set_err(err, PRNG_EINVAL, "bad kernel variant");
            h->kernel = (int)value;
            break;
        case PRNG_OPT_TIME_PARALLEL:
            h->time_parallel = value ? 1 : 0;
            break;
        case PRNG_OPT_CTA_WARPS:
            if (value < 0 || value > kBlock / 32) return set_err(err, PRNG_EINVAL, "bad CTA warps");
            h->cta_warps = value;
            break;
        case PRNG_OPT_OUTPUT:
            if (value < 0 || value > 1) return set_err(err, PRNG_EINVAL, "bad output transform");
            h->output = (int)value;
            break;
        case PRNG_OPT_GRID_WARPS:
            if (value < 0) return set_err(err, PRNG_EINVAL, "bad grid warps");
            h->grid_warps = value;
            break;
        case PRNG_OPT_RING_PAD:
            if (value < 0 || (value & 3) || value > (1 << 24)) return set_err(err, PRNG_EINVAL, "bad ring pad");
            h->ring_pad = value;
            break;
        case PRNG_OPT_HOST_MEM:
            if (value < HK_PINNED || value > HK_HUGE_REGISTERED) return set_err(err, PRNG_EINVAL, "bad host mem kind");
            h->host_mem = (int)value;
            break;
        case PRNG_OPT_CHUNK_ITERS:
            if (value < 0 || value > 0xFFFFFFFFll) return set_err(err, PRNG_EINVAL, "bad chunk iterations");
            h->chunk_iters = value;
            break;
        case PRNG_OPT_PIECE_ORDER:
            if (value < 0 || value > 1) return set_err(err, PRNG_EINVAL, "bad piece order");
            h->piece_order = (int)value;
            break;
        case PRNG_OPT_EPOCH_ITERS:
            if (value < -1 || value > 0xFFFFFFFFll) return set_err(err, PRNG_EINVAL, "bad epoch iterations");
            h->epoch_iters = value;
            break;
        case PRNG_OPT_FUSED_SEED:
            if (value < 0 || value > 1) return set_err(err, PRNG_EINVAL, "bad fused-seed flag");
            h->fused_seed = (int)value;
            break;
        case PRNG_OPT_ONE_SHOT:
            if (value < 0 || value > 2) return set_err(err, PRNG_EINVAL, "bad one-shot mode");
            h->one_shot = (int)value;
            break;


        default:
            return set_err(err, PRNG_EINVAL, "unknown option %d", option);
    }
    return ok(err);
}

int prng_get_option(const prng_t *h, int option, int64_t *value, prng_err_t *err) {
    if (!h || !value) return set_err(err, PRNG_EINVAL, "NULL argument");
    switch (option) {
        case PRNG_OPT_MODE: *value = h->mode; break;
        case PRNG_OPT_BATCH_ITERS: *value = h->batch_iters; break;
        case PRNG_OPT_RING_SLOTS: *value = h->ring_slots_opt; break;
        case PRNG_OPT_PROFILE: *value = h->profile; break;
        case PRNG_OPT_BLOCKING: *value = h->blocking; break;
        case PRNG_OPT_KERNEL: *value = h->kernel; break;
        case PRNG_OPT_OUTPUT: *value = h->output; break;
        case PRNG_OPT_TIME_PARALLEL: *value = h->time_parallel; break;
        case PRNG_OPT_CTA_WARPS: *value = h->cta_warps; break;
        case PRNG_OPT_GRID_WARPS: *value = h->grid_warps; break;
        case PRNG_OPT_RING_PAD: *value = h->ring_pad; break;
        case PRNG_OPT_HOST_MEM: *value = h->host_mem; break;
        case PRNG_OPT_CHUNK_ITERS: *value = h->chunk_iters; break;
        case PRNG_OPT_PIECE_ORDER: *value = h->piece_order; break;
        case PRNG_OPT_EPOCH_ITERS: *value = h->epoch_iters; break;
        case PRNG_OPT_FUSED_SEED: *value = h->fused_seed; break;
        case PRNG_OPT_ONE_SHOT: *value = h->one_shot; break;


        default: return set_err(err, PRNG_EINVAL, "unknown option %d", option);
    }
    return ok(err);
}

// ---------------------------------------------------------------------------- a1
int prng_init(prng_t *h, prng_err_t *err) {
    if (!h) return set_err(err, PRNG_EINVAL, "NULL handle");
    CU(cudaSetDevice(h->device));
    h->poisoned = false;
    if (h->profile != 2) clear_prof(h);  // 2: intervals accumulate across runs
    if (int rc = ensure_origin(h, err)) return rc;
    const double t0 = now_s();
    h->pos = 0;
    h->ring_iter0 = h->ring_cursor;
    h->inited = true;
    if (h->fused_seed) {  // a1 runs inside the next batch launch
        h->seed_pending = true;
        return ok(err);
    }
    h->seed_pending = false;
    if (int rc = seed_launch(h, err)) return rc;
    if (h->profile == 1) {
        CU(cudaStreamSynchronize(h->s_gen));
        h->wall_s += now_s() - t0;
    }
    return ok(err);
}

// ---------------------------------------------------------------------------- seek
// Checkpoint / resume ("the state after iteration k is output k"): position
// the stream so that the next iteration emitted is `iteration`, without generating the
// ones before it -- the seeds (a1) jumped (iteration - 1) xorshift steps ahead by one
// GF(2) mat-vec per work-item with T^(iteration-1) built by binary exponentiation
// (xs is linear, P8).  seek(0) == prng_init.
int prng_seek(prng_t *h, uint64_t iteration, prng_err_t *err) {
    if (int rc = prng_init(h, err)) return rc;
    if (iteration == 0) return ok(err);
    if (int rc = materialize_seeds(h, err)) return rc;  // the jump reads the seeds from d_state
    if (h->jump_cap < 2) {
        if (h->d_jump) cudaFree(h->d_jump);
        h->d_jump = nullptr;
        h->jump_cap = 0;
        CU(cudaMalloc(&h->d_jump, 2 * 64 * sizeof(uint64_t)));
        h->jump_cap = 2;
    }
    h->jump_key[0] = 0;  // the chunk cache no longer matches
    // J_1 = T^L * T^0 with L = iteration - 1
    prngk::jump_columns_kernel<<<1, 64, 0, h->s_gen>>>(h->d_jump, 2u, iteration - 1, 0u);
    CU(cudaGetLastError());
    const uint64_t blocks = std::max<uint64_t>(1, std::min<uint64_t>((h->count + kBlock - 1) / kBlock,
                                                                     (uint64_t)h->num_sms * 8));
    prngk::jump_states_kernel<<<(unsigned)blocks, kBlock, 0, h->s_gen>>>(h->d_state, h->count, h->d_jump + 64);
    CU(cudaGetLastError());
    h->pos = iteration;  // state == out[iteration - 1]: the next launch steps, then emits
    if (h->blocking) CU(cudaStreamSynchronize(h->s_gen));
    return ok(err);
}

// ---------------------------------------------------------------------------- device only
int prng_generate_device(prng_t *h, uint64_t numiter, uint64_t *dst, uint64_t dst_pitch, uint64_t dst_slots,
                         void *stream, prng_err_t *err) {
    if (int rc = check_handle(h, err, true)) return rc;
    if (numiter < 1) return set_err(err, PRNG_EINVAL, "numiter must be >= 1");
    if (!dst || ((uintptr_t)dst & 31) || (dst_pitch & 3) || dst_pitch < h->count || dst_slots < 1 ||
        dst_slots > 0xFFFFFFFFull)
        return set_err(err, PRNG_EINVAL, "dst must be 32-B aligned, pitch %% 4 == 0, pitch >= count, slots >= 1");
    cudaStream_t s = stream ? (cudaStream_t)stream : h->s_gen;
    if (int rc = ensure_origin(h, err)) return rc;
    uint64_t slot = 0, done = 0;
    while (done < numiter) {
        const uint32_t it = (uint32_t)std::min<uint64_t>(numiter - done, 0x7FFFFFFFull);
        if (int rc = launch_batch(h, dst, dst_pitch, dst_slots, slot, it, h->pos == 0, s, err)) return rc;
        h->pos += it;
        done += it;
        slot = (slot + it) % dst_slots;
    }
    return ok(err);
}

// Device-only ring.  B200 measurement (profiles/r1_ring_absorption.md): when the same
// addresses are rewritten within a few GiB, ncu's dram__bytes_write drops far below the
// bytes stored (2.3 GB DRAM writes for 134 GB stored through a 2 GiB ring; 11 GB through
// 4 GiB; 84 GB through 8 GiB; 128 GB through 16 GiB; all 134 GB at >= 32 GiB) and the
// kernel runs ~25 % faster -- a benchmark artefact, not sustainable output bandwidth.  So
// the default ring is large (kRingBytes, capped at 40 % of free HBM) and ROTATES: the
// write cursor persists across prng_init, so the reuse distance of any address is the
// whole ring, also across repeated runs.
constexpr uint64_t kRingBytes = 64ull << 30;

static int ensure_ring(prng *h, uint64_t numiter, prng_err_t *err) {
    const uint64_t pitch = pitch_for(h->count) + (uint64_t)h->ring_pad;
    const uint64_t slot_bytes = pitch * sizeof(uint64_t);
    uint64_t slots = (uint64_t)h->ring_slots_opt;
    // fast path: the ring exists and still matches the options (no cudaMemGetInfo, which
    // costs milliseconds, on every generate call)
    if (h->d_ring && h->ring_pitch == pitch && (slots == 0 ? h->ring_auto : slots == h->ring_slots))
        return PRNG_OK;
    if (slots == 0) {
        uint64_t target = kRingBytes;
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
            uint64_t have = (uint64_t)free_b + (h->d_ring ? h->ring_slots * h->ring_pitch * 8 : 0);
            target = std::min<uint64_t>(target, have * 2 / 5);
        }
        slots = std::max<uint64_t>(2, target / slot_bytes);
        slots = std::min<uint64_t>(slots, 0x7FFFFFFFull);
    }
    if (h->d_ring && h->ring_slots == slots && h->ring_pitch == pitch) {
        h->ring_auto = h->ring_slots_opt == 0;
        return PRNG_OK;
    }
    if (h->d_ring) {
        CU(cudaStreamSynchronize(h->s_gen));
        cudaFree(h->d_ring);
        h->d_ring = nullptr;
    }
    CU(cudaMalloc(&h->d_ring, slots * slot_bytes));
    h->ring_slots = slots;
    h->ring_pitch = pitch;
    h->ring_auto = h->ring_slots_opt == 0;
    h->ring_cursor = 0;
    h->ring_iter0 = (slots - (h->pos % slots)) % slots;  // keep "iteration k -> (iter0 + k) mod R"
    (void)numiter;
    return PRNG_OK;
}

static int generate_device_only(prng *h, uint64_t numiter, prng_err_t *err) {
    if (int rc = ensure_ring(h, numiter, err)) return rc;
    const double t0 = now_s();
    // Slot of an iteration = iteration mod R, across calls (prng_device_ring documents it).
    uint64_t done = 0;
    while (done < numiter) {
        const uint32_t it = (uint32_t)std::min<uint64_t>(numiter - done, 0x7FFFFFFFull);
        if (int rc = launch_batch(h, h->d_ring, h->ring_pitch, h->ring_slots, (h->ring_iter0 + h->pos) % h->ring_slots, it,
                                  h->pos == 0, h->s_gen, err))
            return rc;
        h->pos += it;
        done += it;
    }
    h->ring_cursor = (h->ring_iter0 + h->pos) % h->ring_slots;
    if (h->blocking) {
        CU(cudaStreamSynchronize(h->s_gen));
        h->wall_s += now_s() - t0;
    }
    return PRNG_OK;
}

// ---------------------------------------------------------------------------- autotune
// Which (variant, warps per SM) writes fastest depends on the shape (count, ring pitch,
// slots) through the DRAM page / channel mapping, so measure instead of
// guessing: each candidate generates `probe_iters` iterations into the handle's own ring
// (best of 2 after a warm-up), the fastest becomes the handle's kernel + grid.  The
// state array is consumed, so the handle needs prng_init afterwards.
static const struct {
    const char *variant;
    int warps_per_sm;  // persistent grid of this many warps per SM; 0: one-shot grid
} kTuneCandidates[] = {{"v4n8s1a", 4}, {"v4n4s1p", 4}, {"v4n4s1", 4},  {"v2n4s1", 4}, {"v2n4s1", 8},
                       {"v4n8s1", 4},  {"v4n16s1", 4}, {"v2n32s1", 8}, {"v2n2s1", 4}, {"v4n8s1a", 0},
                       {"v4n16s1", 0}};

extern "C" int prng_autotune(prng_t *h, uint64_t probe_iters, double *best_gbs, prng_err_t *err) {
    if (int rc = check_handle(h, err, false)) return rc;
    if (int rc = ensure_ring(h, 0, err)) return rc;
    if (probe_iters == 0)  // ~16 GiB of output per probe, within [8, 1000] iterations
        probe_iters = std::min<uint64_t>(1000, std::max<uint64_t>(8, (16ull << 30) / (h->count * 8)));
    // a probe never wraps the ring inside its launch: no rewrite can be absorbed in L2
    // (DESIGN.md §5), so every candidate is timed on DRAM-bound stores
    probe_iters = std::min<uint64_t>(probe_iters, h->ring_slots);
    const int saved_profile = h->profile;
    h->profile = 0;
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    double best = -1;
    int best_k = h->kernel;
    int64_t best_w = h->grid_warps;
    const int saved_one_shot = h->one_shot;
    int best_os = h->one_shot;
    int rc = PRNG_OK;
    for (const auto &c : kTuneCandidates) {
        const int k = variant_id(c.variant);
        if (k < 0) continue;
        h->kernel = k;
        h->grid_warps = (int64_t)c.warps_per_sm * h->num_sms;  // 0: no user grid ...
        h->one_shot = c.warps_per_sm ? saved_one_shot : 2;     // ... and a one-shot grid
        double cand = 0;
        for (int rep = 0; rep < 3 && !rc; ++rep) {
            cudaEventRecord(e0, h->s_gen);
            rc = launch_batch(h, h->d_ring, h->ring_pitch, h->ring_slots, h->ring_cursor, (uint32_t)probe_iters, false, h->s_gen,
                              err);
            cudaEventRecord(e1, h->s_gen);
            h->ring_cursor = (h->ring_cursor + probe_iters) % h->ring_slots;
            if (rc) break;
            cudaError_t e = cudaEventSynchronize(e1);
            if (e != cudaSuccess) {
                rc = set_err(err, PRNG_ECUDA, "autotune: %s", cudaGetErrorString(e));
                break;
            }
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0) cand = std::max(cand, 8.0 * h->count * probe_iters / (ms * 1e-3) / 1e9);
        }
        if (rc) break;
        if (cand > best) {
            best = cand;
            best_k = k;
            best_w = h->grid_warps;
            best_os = h->one_shot;
        }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    h->profile = saved_profile;
    h->kernel = best_k;
    h->grid_warps = best_w;
    h->one_shot = rc ? saved_one_shot : best_os;
    h->inited = false;  // the probes consumed the state: prng_init before generating
    h->pos = 0;
    if (rc) return rc;
    if (best_gbs) *best_gbs = best;
    return ok(err);
}

int prng_generate(prng_t *h, uint64_t numiter, prng_sink_fn sink, void *user, prng_err_t *err) {
    if (int rc = check_handle(h, err, true)) return rc;
    if (numiter < 1) return set_err(err, PRNG_EINVAL, "numiter must be >= 1");
    if (int rc = ensure_origin(h, err)) return rc;
    int rc = sink ? generate_e2e(h, numiter, sink, user, err) : generate_device_only(h, numiter, err);
    if (rc) return rc;
    return ok(err);
}

int prng_device_ring(const prng_t *h, uint64_t **base, uint64_t *pitch, uint64_t *slots, uint64_t *iter0_slot,
                     uint64_t *last_iter_end, prng_err_t *err) {
    if (!h || !base || !pitch || !slots || !iter0_slot || !last_iter_end)
        return set_err(err, PRNG_EINVAL, "NULL argument");
    *iter0_slot = h->ring_iter0;
    *base = h->d_ring;
    *pitch = h->ring_pitch;
    *slots = h->ring_slots;
    *last_iter_end = h->pos;
    return ok(err);
}

int prng_read_slot(prng_t *h, uint64_t slot, uint64_t *host_dst, prng_err_t *err) {
    if (int rc = check_handle(h, err, false)) return rc;
    if (!h->d_ring || slot >= h->ring_slots || !host_dst) return set_err(err, PRNG_EINVAL, "no such ring slot");
    CU(cudaStreamSynchronize(h->s_gen));
    CU(cudaMemcpy(host_dst, h->d_ring + slot * h->ring_pitch, h->count * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return ok(err);
}

int prng_read_state(prng_t *h, uint64_t *host_dst, prng_err_t *err) {
    if (int rc = check_handle(h, err, false)) return rc;
    if (!host_dst) return set_err(err, PRNG_EINVAL, "NULL destination");
    if (int rc = materialize_seeds(h, err)) return rc;
    CU(cudaStreamSynchronize(h->s_gen));
    CU(cudaMemcpy(host_dst, h->d_state, h->count * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return ok(err);
}

#ifdef PRNG_CHECKED
// Checked build only (tools/gpu_checked.sh, tests/test_gpu_parity.py): the negative control
// of the kernels' bounds checks.  One natural-order launch into a one-slot ring whose pitch
// (= its allocation) is 4 u64 short of the handle's count, so the last vector of the piece
// holding the last gids falls outside it: the check must trap, and the call returns
// PRNG_ECUDA (the context is then unusable: run it in a process of its own).
int prng_checked_selftest(prng_t *h, prng_err_t *err) {
    if (int rc = check_handle(h, err, false)) return rc;
    if (h->count < 8 || h->count % 4) return set_err(err, PRNG_EINVAL, "selftest needs count %% 4 == 0, >= 8");
    const uint64_t pitch = h->count - 4;
    uint64_t *buf = nullptr;
    CU(cudaMalloc(&buf, pitch * sizeof(uint64_t)));
    h->kernel = variant_id("v4n4s1");
    int rc = launch_batch(h, buf, pitch, 1, 0, 2, true, h->s_gen, err);
    const cudaError_t e = cudaStreamSynchronize(h->s_gen);
    cudaFree(buf);
    if (rc) return rc;
    if (e != cudaSuccess) return set_err(err, PRNG_ECUDA, "selftest launch: %s", cudaGetErrorString(e));
    return ok(err);  // not reached when the checks work
}
#endif

// ---------------------------------------------------------------------------- a6 capture
int prng_prof_events(const prng_t *hc, uint64_t cap, uint32_t *name_id, double *start_s, double *end_s,
                     uint64_t *n_out, double *wall_s, prng_err_t *err) {
    prng *h = const_cast<prng *>(hc);
    if (!h || !n_out) return set_err(err, PRNG_EINVAL, "NULL argument");
    const uint64_t n = h->dev_iv.size() + h->host_iv.size();
    *n_out = n;
    if (wall_s) *wall_s = h->wall_s;
    if (cap && (!name_id || !start_s || !end_s)) return set_err(err, PRNG_EINVAL, "NULL output arrays");
    CU(cudaSetDevice(h->device));
    uint64_t i = 0;
    for (const auto &iv : h->dev_iv) {
        if (i >= cap) break;
        float a = 0, b = 0;
        CU(cudaEventSynchronize(iv.b));
        CU(cudaEventElapsedTime(&a, h->ev_origin, iv.a));
        CU(cudaEventElapsedTime(&b, h->ev_origin, iv.b));
        name_id[i] = iv.name;
        start_s[i] = a * 1e-3;
        end_s[i] = b * 1e-3;
        ++i;
    }
    for (const auto &iv : h->host_iv) {
        if (i >= cap) break;
        name_id[i] = iv.name;
        start_s[i] = iv.a;
        end_s[i] = iv.b;
        ++i;
    }
    return ok(err);
}

}  // extern "C"
