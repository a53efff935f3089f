// engine_internal.h -- shared internals of libprng_b200.so's translation units:
// prng_engine.cu (handle, options, kernels dispatch, device-only, seek, autotune),
// prng_pipeline.cu (end-to-end modes a4-a5, host array), prng_probes.cu (roofline
// probes), prng_sinks.cpp (built-in sinks).  Not part of the C ABI.
#pragma once
#include <cuda_runtime.h>

#include <chrono>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "../../include/prng.h"

namespace prng_detail {

inline int set_err(prng_err_t *err, int code, const char *fmt, ...) {
    if (err) {
        err->code = code;
        va_list ap;
        va_start(ap, fmt);
        std::vsnprintf(err->msg, sizeof(err->msg), fmt, ap);
        va_end(ap);
    }
    return code;
}
inline int ok(prng_err_t *err) {
    if (err) {
        err->code = PRNG_OK;
        err->msg[0] = 0;
    }
    return PRNG_OK;
}

#define CU(call)                                                                                    \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess) {                                                                    \
            if (h) h->poisoned = true;                                                              \
            return set_err(err, e_ == cudaErrorMemoryAllocation ? PRNG_ENOMEM : PRNG_ECUDA,        \
                           "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__);   \
        }                                                                                           \
    } while (0)

constexpr int kBlock = 256;     // threads per CTA of the batch kernels (max)
constexpr int kOneShotBlock = 128;  // threads per CTA of a one-shot grid (4 warps, measured best)
constexpr int kMaxVariants = 16;

inline double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Host buffer kinds (PRNG_OPT_HOST_MEM selects among the pinned ones).
enum HostKind { HK_PINNED = 0, HK_PINNED_WC = 1, HK_HUGE_REGISTERED = 2, HK_MAPPED = 3, HK_PAGEABLE = 4 };

inline uint64_t pitch_for(uint64_t count) { return (count + 3) & ~3ull; }  // 32-byte aligned slots

}  // namespace prng_detail

// ============================================================================ the handle
struct prng {
    int device = 0;
    int num_sms = 0;
    int l2_bytes = 0;
    uint64_t numrn_total = 0, seed = 0, gid_begin = 0, count = 0;
    uint64_t pos = 0;  // iterations emitted since prng_init
    bool inited = false, poisoned = false;
    // a1 fused (PRNG_OPT_FUSED_SEED): prng_init only marks the seeds pending; the next batch
    // launch computes them in registers (or materialize_seeds runs seed_kernel first when
    // something reads d_state directly)
    bool seed_pending = false;
    int fused_seed = 1;

    uint64_t *d_state = nullptr;   // [round_up(count, 4)]
    uint64_t *d_state2 = nullptr;  // the other half of the state double buffer (time-parallel launches)
    uint64_t *d_jump = nullptr;    // jump-ahead columns [chunks][64] (time-parallel launches)
    uint64_t jump_cap = 0, jump_key[3] = {0, 0, 0};  // capacity (chunks), cached (C, L, e)
    int time_parallel = 1;         // PRNG_OPT_TIME_PARALLEL

    // device-only ring
    uint64_t *d_ring = nullptr;
    uint64_t ring_pitch = 0, ring_slots = 0;
    uint64_t ring_cursor = 0;  // next slot to write; persists across prng_init (rotating ring)
    bool ring_auto = false;    // the ring was sized automatically (PRNG_OPT_RING_SLOTS 0)
    uint64_t ring_iter0 = 0;   // slot holding iteration 0 of the current init

    // end-to-end buffers
    uint64_t *d_buf = nullptr;  // 2 halves x T slots, pitch buf_pitch
    uint64_t buf_pitch = 0, buf_T = 0;
    uint64_t *h_buf[2] = {nullptr, nullptr};
    uint64_t *h_dev[2] = {nullptr, nullptr};  // device aliases of mapped host halves (zero-copy)
    int h_kind = -1;                          // enum HostKind of the allocated halves
    int host_mem = 0;                         // PRNG_OPT_HOST_MEM
    uint64_t h_T = 0;
    int h_halves = 0;

    cudaStream_t s_gen = nullptr, s_copy = nullptr;
    bool own_streams = true;
    // ordering events of the end-to-end pipelines (gen -> copy, copy -> gen), created on
    // first use and reused by every later call (creating 8-16 events per call cost tens of
    // microseconds at small n); calls on one handle never overlap, so one pool suffices
    static constexpr int kPipeEvents = 16;
    cudaEvent_t pev[kPipeEvents] = {};

    // options
    int mode = PRNG_MODE_OVERLAP2;
    int64_t batch_iters = 0, ring_slots_opt = 0, grid_warps = 0, ring_pad = 0, cta_warps = 0;
    int64_t chunk_iters = 0;  // PRNG_OPT_CHUNK_ITERS
    int piece_order = 0;      // PRNG_OPT_PIECE_ORDER
    int64_t epoch_iters = 0;  // PRNG_OPT_EPOCH_ITERS
    int last_kernel = -1;     // variant id of the last batch launch (after the anti-absorption rule)
    uint32_t last_epoch = 0;  // its epoch length (0: natural order)

    int profile = 0, kernel = 0, output = 0, blocking = 1;
    // Test-only fault injection (env PRNG_B200_FAULT_AFTER=N, read at create): the N-th
    // checked CUDA call of prng_generate_host reports failure, so tests can prove that a
    // failed record / wait / copy poisons the handle instead of returning silent output.
    int64_t fault_after = 0;
    int blocks_per_sm[prng_detail::kMaxVariants] = {0};
    // resident CTAs per SM of each variant at prng_detail::kOneShotBlock threads (one-shot
    // grids, PRNG_OPT_ONE_SHOT); 0 = not queried yet
    int oneshot_blocks_per_sm[2][prng_detail::kMaxVariants] = {};  // [output transform][variant]
    int one_shot = 1;               // PRNG_OPT_ONE_SHOT: 0 off, 1 auto, 2 always (when allowed)
    size_t oneshot_smem = 0;        // dynamic shared memory per one-shot CTA (residency cap)
    uint64_t last_blocks = 0;       // grid of the last batch launch (prng_last_grid)
    uint32_t last_threads = 0, last_rounds = 0;
    bool last_one_shot = false;

    // profiling (a6)
    cudaEvent_t ev_origin = nullptr;
    double host_origin = 0;
    struct DevIv {
        uint32_t name;
        cudaEvent_t a, b;
    };
    std::vector<DevIv> dev_iv;
    struct HostIv {
        uint32_t name;
        double a, b;
    };
    std::vector<HostIv> host_iv;
    double wall_s = 0;
};

namespace prng_detail {

inline cudaError_t fault_point(prng *h, cudaError_t e) {
    if (e == cudaSuccess && h->fault_after > 0 && --h->fault_after == 0) return cudaErrorUnknown;
    return e;
}

void free_host(int kind, void *p, size_t bytes);
void free_e2e(prng *h);
void clear_prof(prng *h);
int ensure_origin(prng *h, prng_err_t *err);
int prof_begin(prng *h, cudaStream_t s, uint32_t name, prng_err_t *err);
int prof_end(prng *h, cudaStream_t s, prng_err_t *err);
// Launch one batch of `iters` iterations (a2 + a3) into ring slots of `dst`.
int launch_batch(prng *h, uint64_t *dst, uint64_t pitch, uint64_t nslots, uint64_t slot0, uint32_t iters,
                 bool first_is_state, cudaStream_t s, prng_err_t *err);
int check_handle(prng *h, prng_err_t *err, bool need_init);
// Run the pending a1 (seed_kernel into d_state on s_gen) if prng_init deferred it.
int materialize_seeds(prng *h, prng_err_t *err);
// The handle's pipeline events (prng::pev), created on the first call that needs them.
int pipeline_events(prng *h, prng_err_t *err);
// prng_pipeline.cu: the end-to-end modes (S0, S1, O1, O2, O3) of prng_generate with a sink.
int generate_e2e(prng *h, uint64_t numiter, prng_sink_fn sink, void *user, prng_err_t *err);

}  // namespace prng_detail
