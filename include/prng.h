/*
 * prng.h -- C ABI of the B200-native massive-PRNG hot path.
 *
 * What it computes (the paper's §5 example application, arXiv 1609.01257):
 *   "each work-item generates a 64-bit random value per invocation. The init kernel
 *    creates the initial random values by applying a hash function [wang1997inthash]
 *    to the global ID of the associated work-items. The generated values not only
 *    constitute the first batch of random numbers, but also serve as seeds for the
 *    next batch."                                                   (§5)
 *   "... a simple Xorshift PRNG [marsaglia2003xorshift]"           (§5)
 *   n numbers per iteration, i iterations, N = 8*n*i bytes          (Eq. 1)
 * The exact arithmetic (readings A1-A8 of DESIGN.md §3) is:
 *   out[0][g] = seed64(g, seed)           (Wang hash of the global id, 0 -> 1)
 *   out[k][g] = xorshift64(out[k-1][g])   (x^=x<<13; x^=x>>7; x^=x<<17), k = 1..numiter-1
 * Output layout: iteration-major, gid ascending, little-endian u64 (A8): exactly the
 * paper's binary stdout stream.
 *
 * Conventions follow cf4ocl's (§4.1): an opaque object with a create/destroy
 * pair; functions take the object first; every fallible call returns a status (0 ok,
 * < 0 error) AND fills an optional detail object passed last (may be NULL); an errors
 * module maps codes to strings.
 *
 * Ownership: the handle owns all device memory (state array, device ring), pinned host
 * buffers, CUDA streams and events it creates.  Pointers passed to a sink are BORROWED:
 * valid only for the duration of the callback ("automatically released and should not
 * be destroyed by client code").
 *
 * Thread-safety: one handle must not be used from two threads at once.  Distinct
 * handles (e.g. one per GPU / rank) are independent.
 *
 * There is no CPU fallback: every generation step runs in the sm_100a kernels of
 * libprng_b200.so; without a CUDA device prng_create fails with PRNG_ECUDA.
 */
#ifndef PRNG_B200_H
#define PRNG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ errors */
#define PRNG_OK 0
#define PRNG_EINVAL -1  /* bad argument (numrn = 0 or > 2^32, numiter = 0, bad range/option) */
#define PRNG_ESTATE -2  /* bad state: generate before init, or handle poisoned by an abort   */
#define PRNG_ENOMEM -3  /* device or pinned host allocation failed                          */
#define PRNG_ECUDA -4   /* CUDA runtime error; detail holds cudaGetErrorString()           */
#define PRNG_ESINK -5   /* the sink returned nonzero: generation aborted                    */

/* Optional detail object, last argument of every fallible call. */
typedef struct prng_err {
    int code;
    char msg[256];
} prng_err_t;

/* Total function: unknown codes map to "unknown error <code>". */
const char *prng_strerror(int code);

/* ------------------------------------------------------------------ handle */
typedef struct prng prng_t;

/* Sink ("out"): receives `iters` consecutive iterations starting at
 * iteration `iter_begin`, each `count` u64 for gids [gid_begin, gid_begin + count),
 * as data[t * count + j] (dense, iteration-major).  `data` is borrowed (pinned host
 * memory owned by the library).  Called on the caller's thread, strictly in iteration
 * order.  Return 0 to continue; nonzero aborts prng_generate with PRNG_ESINK. */
typedef int (*prng_sink_fn)(void *user, uint64_t iter_begin, uint32_t iters,
                            uint64_t gid_begin, uint64_t count, const uint64_t *data);

/* One generator over all numrn work-items, on the current CUDA device.
 * numrn in [1, 2^32] (the paper's numrn is a cl_uint).  seed: 0 reproduces the
 * paper (which has no seed); other values premix into the hash keys (A4).
 * Returns NULL on error (err filled). */
prng_t *prng_create(uint64_t numrn, uint64_t seed, prng_err_t *err);

/* A rank's share: the gids [gid_begin, gid_begin + gid_count) of a numrn_total stream,
 * on CUDA device `cuda_device` (-1 = current).  Values depend only on the GLOBAL gid,
 * so shards reassemble bit-exactly into the single-device stream (A11). */
prng_t *prng_create_range(uint64_t numrn_total, uint64_t seed, uint64_t gid_begin,
                          uint64_t gid_count, int cuda_device, prng_err_t *err);

/* The handle's share of the stream: numrn_total, its first gid and its gid count (any
 * pointer may be NULL).  PRNG_EINVAL for a NULL handle. */
int prng_get_range(const prng_t *h, uint64_t *numrn_total, uint64_t *gid_begin, uint64_t *count,
                   prng_err_t *err);

/* NULL-safe.  Synchronises the handle's streams, frees device + pinned memory. */
void prng_destroy(prng_t *h);

/* Use caller-owned CUDA streams (cudaStream_t, e.g. torch.cuda.Stream().cuda_stream) for
 * generation and D2H instead of the handle's own; the caller keeps ownership and must
 * keep them alive until prng_destroy.  The two must differ. */
int prng_set_streams(prng_t *h, void *gen_stream, void *copy_stream, prng_err_t *err);

/* a1 -- the init kernel: state[g] = seed64(g, seed) on the device; the stream
 * position is reset to iteration 0 (the next iteration emitted is the seeds themselves).
 * With PRNG_OPT_FUSED_SEED 1 (the default) no kernel runs here: the next batch launch
 * computes the seeds in registers (same output). */
int prng_init(prng_t *h, prng_err_t *err);

/* Checkpoint / resume: re-seed (as prng_init) and position the stream so that the next
 * iteration emitted is `iteration` -- the same values a run from prng_init would emit
 * from there on -- in O(log iteration) work: xorshift is GF(2)-linear, so
 * iteration - 1 steps are one 64x64 bit-matrix product per work-item (readings A5, P8). */
int prng_seek(prng_t *h, uint64_t iteration, prng_err_t *err);

/* a2-a5 -- emit the next `numiter` iterations (numiter >= 1).
 *  sink != NULL (end to end): batches of T iterations are generated into a device ring,
 *    copied D2H on a side stream into a pinned host double buffer and handed to `sink`
 *    while the next batches are generated and copied (P:164-173, P:177 limitation 2).
 *  sink == NULL (device only): iterations are generated into the handle's device ring of
 *    R slots with no host transfer; see prng_device_ring().  The ring is large (64 GiB,
 *    capped at 40 % of free HBM) and rotating, so no address is rewritten within 64 GiB of
 *    output -- see DESIGN.md §5 for why that matters on B200.
 * Repeated calls continue the stream: generate(a); generate(b) == generate(a + b) (A10).
 * Blocks until all work of the call is complete. */
int prng_generate(prng_t *h, uint64_t numiter, prng_sink_fn sink, void *user, prng_err_t *err);

/* Device-only generation into a caller-owned device buffer (e.g. a torch tensor):
 * iteration t of this call goes to dst + (t mod dst_slots) * dst_pitch (u64 elements).
 * dst must be 32-byte aligned and dst_pitch a multiple of 4 with dst_pitch >= count.
 * Enqueued on `stream` (a cudaStream_t, NULL = the handle's generation stream);
 * asynchronous: returns after enqueueing.  prng_init and the other generate calls run on
 * the handle's generation stream: with a different `stream` the caller orders them against
 * this call (e.g. an event); calls on one handle must not overlap in time.  (With
 * PRNG_OPT_FUSED_SEED 1, prng_init enqueues nothing: the seeds are computed by this call's
 * own kernel on `stream`.) */
int prng_generate_device(prng_t *h, uint64_t numiter, uint64_t *dst, uint64_t dst_pitch,
                         uint64_t dst_slots, void *stream, prng_err_t *err);

/* a4 + a5, multi-rank form: "each rank generates its own gid range and writes its slice of
 * the host output directly" (BASELINE north_star).  Generates the next `numiter` iterations
 * and copies them D2H straight into the caller's host array (no staging buffer, no sink):
 * iteration k of this call goes to dst[(k mod dst_rows) * dst_pitch + j], j < count.  For
 * one array shared by all ranks of a node, pass dst = array + gid_begin and dst_pitch =
 * numrn_total.  dst need not be pinned (it is cudaHostRegister'ed for the call if it is
 * not).  Blocks until the copies are done; the array is the caller's.  Every CUDA call is
 * checked: on a failure the call returns PRNG_ECUDA and the handle is poisoned until
 * prng_init (tests inject one with the environment variable PRNG_B200_FAULT_AFTER=N, read at
 * create time: the N-th checked call fails; not for production use). */
int prng_generate_host(prng_t *h, uint64_t numiter, uint64_t *dst, uint64_t dst_pitch,
                       uint64_t dst_rows, prng_err_t *err);

/* The handle's device ring (device-only mode): base pointer, pitch (u64 elements), number
 * of slots R, and the slot holding iteration 0 of the current prng_init: iteration k
 * (k < last_iter_end, the stream position) was written to slot (iter0_slot + k) mod R and
 * is still there if k >= last_iter_end - R.  The write cursor rotates across prng_init
 * calls (iter0_slot changes). */
int prng_device_ring(const prng_t *h, uint64_t **base, uint64_t *pitch, uint64_t *slots,
                     uint64_t *iter0_slot, uint64_t *last_iter_end, prng_err_t *err);

/* Copy the handle's `count` outputs (prng_get_range) of device-ring slot `slot` to host
 * memory, which must hold count u64 (test/inspection aid). */
int prng_read_slot(prng_t *h, uint64_t slot, uint64_t *host_dst, prng_err_t *err);

/* Copy the current per-gid state (== the last emitted iteration; count u64) to host memory. */
int prng_read_state(prng_t *h, uint64_t *host_dst, prng_err_t *err);

/* ------------------------------------------------------------------ options */
enum prng_option {
    PRNG_OPT_MODE = 1,         /* enum prng_mode, default PRNG_MODE_OVERLAP2            */
    PRNG_OPT_BATCH_ITERS = 2,  /* T for end-to-end batches; 0 = auto (~256 MiB per batch) */
    PRNG_OPT_RING_SLOTS = 3,   /* R of the device-only ring; 0 = auto (64 GiB, <= 40 % free) */
    PRNG_OPT_PROFILE = 4,      /* 1 = record per-batch intervals (CUDA events), reset by
                                  prng_init; 2 = same, accumulated across prng_init calls
                                  and without the host syncs mode 1 adds for wall time    */
    PRNG_OPT_KERNEL = 5,       /* kernel variant id (see prng_kernel_variants); 0 = "auto"
                                  (default): v4n8s1a from 2^21 work-items per handle,
                                  v4n4s1p from 2^15, v2n2s1 below, widened / epoch-ordered by the
                                  anti-absorption rule (see PRNG_OPT_EPOCH_ITERS,
                                  prng_last_launch)                                       */
    PRNG_OPT_GRID_WARPS = 6,   /* cap on resident warps of the persistent grid; 0 = auto  */
    PRNG_OPT_RING_PAD = 7,     /* extra u64 elements between device-only ring slots (multiple
                                  of 4; breaks power-of-two slot strides); default 0       */
    PRNG_OPT_HOST_MEM = 8,     /* pinned host halves of modes O1/O2/S0: 0 cudaHostAlloc,
                                  1 write-combined, 2 THP-backed mmap + cudaHostRegister  */
                               /* 9: reserved (a round-1 diagnostic option, removed)        */
    PRNG_OPT_OUTPUT = 10,      /* NEXT-3 output transform: 0 = the state (the paper, A7);
                                  1 = state * 0x2545F4914F6CDD1D mod 2^64 (xorshift64*-style
                                  scrambler, A19).  Every kernel variant supports both.    */
    PRNG_OPT_TIME_PARALLEL = 11, /* 1 (default): when numrn is too small to fill the GPU, cut
                                  a launch's iterations into chunks started by GF(2)
                                  jump-ahead (xs^k is linear: a 64x64 bit matrix), at 8
                                  warps per SM, one chunk per warp, >= 3 chunks of >= 48 
                                  iterations, in launches that do not wrap their slots;
                                  0: off.  Output unchanged.                              */
    PRNG_OPT_BLOCKING = 12,    /* 1 (default): device-only prng_generate returns when the work
                                  is done; 0: returns after enqueueing on the generation
                                  stream (synchronise the stream before reading results)   */
    PRNG_OPT_CTA_WARPS = 13,   /* warps per CTA of the batch kernels (1..8); 0 = auto: one
                                  CTA per SM when <= 8 warps per SM are used               */
    PRNG_OPT_CHUNK_ITERS = 14, /* L > 0: cut every launch of more than L iterations into
                                  chunks of L started by GF(2) jump-ahead, at any numrn
                                  (the work order of time-parallel mode); 0 (default): only
                                  as PRNG_OPT_TIME_PARALLEL decides.  Output unchanged.     */
    PRNG_OPT_PIECE_ORDER = 15, /* how work units are dealt to warps (output unchanged):
                                  0 (default) round-robin, adjacent CTAs hold adjacent
                                  pieces; 1 CTA-blocked, CTA b holds a contiguous run of
                                  units, so concurrently written 4 KiB chunks are spread
                                  over the whole slot.                                      */
    PRNG_OPT_EPOCH_ITERS = 16, /* epoch-major order for CTA-synchronised variants (output
                                  unchanged): every warp runs each of its pieces through E
                                  iterations, then the next piece; the state goes through
                                  HBM between epochs (+16 B per number per epoch).
                                  0 (default) auto: E = R when a device-only launch wraps
                                  a ring of R slots whose live lines (R x grid warps x
                                  bytes per warp-iteration) are < 2x L2, so no address is
                                  rewritten while its line may still be in L2 (DESIGN.md
                                  §5); E > 0 forced; -1 off.                                */
    PRNG_OPT_FUSED_SEED = 17,  /* 1 (default): prng_init only records that the stream restarts;
                                  the next batch launch computes the seeds (a1) in registers
                                  before its first iteration -- one launch and 16 B per
                                  work-item of state traffic less, output unchanged.  Calls
                                  that read the state array directly (prng_read_state,
                                  prng_seek) run the seed kernel first.  0: prng_init
                                  launches the seed kernel itself (the paper's separate
                                  `init` kernel; its interval is INIT_KERNEL in the
                                  profile, as in Fig. 5).                                   */
    PRNG_OPT_ONE_SHOT = 18     /* grid of natural-order launches with many more pieces than
                                  one wave of resident warps: 1 (default) auto -- from 4
                                  waves of the one-shot grid's resident warps on (3 CTAs
                                  per SM; 2^20 work-items with v4n4s1p, 2^21 with v4n8s1a),
                                  one piece per warp on a multi-wave grid of 4-warp CTAs
                                  that the hardware dispatches in order (measured 2-7 %
                                  more write bandwidth than the persistent grid from 2^20
                                  work-items, 5.6 % more under the power cap; DESIGN.md
                                  §5); 0: always the
                                  persistent one-wave grid; 2: one-shot whenever the launch
                                  form allows it (natural order, no PRNG_OPT_GRID_WARPS /
                                  CTA_WARPS / EPOCH_ITERS / CHUNK_ITERS, no L2-absorbing
                                  ring wrap), for tests and measurements.  Output
                                  unchanged.  prng_last_grid reports the grid used.        */
};

/* End-to-end pipelines: two serialised reproductions of the paper's finding, and the two
 * overlapped fixes. */
enum prng_mode {
    PRNG_MODE_SERIAL = 0,    /* S0: generate, copy and sink back to back on one stream          */
    PRNG_MODE_PAGEABLE = 1,  /* S1: side stream, but pageable (malloc) host buffers             */
    PRNG_MODE_OVERLAP1 = 2,  /* O1: side copy stream + device double buffer, ONE pinned host
                                buffer: read and out serialised as in the paper */
    PRNG_MODE_OVERLAP2 = 3,  /* O2: O1 + host-side dual buffer, sink(j) || D2H(j+1) || gen(j+2) */
    PRNG_MODE_ZEROCOPY = 4   /* O3: the kernel stores each batch straight into mapped pinned host
                                memory (two halves): generation and transfer fused, no device ring
                                and no copy engine; sink(j) || gen(j+1).  Needs count % 4 == 0. */
};

int prng_set_option(prng_t *h, int option, int64_t value, prng_err_t *err);
int prng_get_option(const prng_t *h, int option, int64_t *value, prng_err_t *err);

/* Measure a short list of (kernel variant, grid) candidates -- persistent grids of 4 or 8
 * warps per SM and one-shot grids -- on this handle's device-only ring (probe_iters
 * iterations each, 0 = auto: ~16 GiB of output) and keep the fastest as PRNG_OPT_KERNEL +
 * PRNG_OPT_GRID_WARPS (a persistent winner) or PRNG_OPT_KERNEL + PRNG_OPT_ONE_SHOT 2 with
 * PRNG_OPT_GRID_WARPS 0 (a one-shot winner).  The probes consume the device
 * state, so the handle must be prng_init'ed again afterwards (generate returns
 * PRNG_ESTATE otherwise).  best_gbs (may be NULL) gets the winner's probe GB/s. */
int prng_autotune(prng_t *h, uint64_t probe_iters, double *best_gbs, prng_err_t *err);

/* Number of kernel variants compiled in (9), and the name of one: id 0 "auto" (the
 * default, resolved per launch -- see PRNG_OPT_KERNEL); "v<V>n<N>s1" = V-wide u64 vector
 * stores (V = 4: 32 bytes, V = 2: 16 bytes), N numbers per thread, CTA barrier every
 * iteration, 4 warps per SM; suffix "a" = .aligned barrier in uniform rounds, "p" =
 * ping-pong hot loop.  "v2n4s1" is north_star's 16-byte form.  NULL for an id out of
 * range. */
int prng_kernel_variants(void);
const char *prng_kernel_variant_name(int id);

/* The batch kernel the handle's last launch actually ran: *variant = its variant id (the
 * PRNG_OPT_KERNEL choice, or the wider variant the anti-absorption rule substituted for the
 * default), *epoch_iters = its epoch length (0 = natural order).  -1 / 0
 * before any launch.  Either pointer may be NULL.  PRNG_EINVAL for a NULL handle. */
int prng_last_launch(const prng_t *h, int *variant, uint32_t *epoch_iters, prng_err_t *err);

/* The grid of the last batch launch: CTAs, threads per CTA, the rounds of units each warp
 * walks, and whether it was a one-shot grid (PRNG_OPT_ONE_SHOT; rounds is then 1).  Zeros
 * before any launch.  Any pointer may be NULL.  PRNG_EINVAL for a NULL handle. */
int prng_last_grid(const prng_t *h, uint64_t *blocks, uint32_t *threads, uint32_t *rounds, int *one_shot,
                   prng_err_t *err);

/* ------------------------------------------------------------------ profiling (a6) */
/* Event name ids, as cf4ocl names them in Fig. 3 plus the host sink. */
#define PRNG_EV_INIT_KERNEL 0
#define PRNG_EV_RNG_KERNEL 1
#define PRNG_EV_READ_BUFFER 2
#define PRNG_EV_OUT 3
#define PRNG_EV_NAMES 4
const char *prng_event_name(uint32_t id);

/* Intervals recorded by the last prng_init + prng_generate with PRNG_OPT_PROFILE on:
 * name id, start and end in seconds from a common origin (device intervals from CUDA
 * events; OUT intervals from the host clock aligned to the same origin).  `n_out` gets
 * the number available; at most `cap` are written.  `wall_s` (may be NULL) gets the host
 * wall time of the profiled calls.  An INIT_KERNEL interval exists only when the seed
 * kernel ran on its own (PRNG_OPT_FUSED_SEED 0, or a materialising call); with a1 fused
 * the seeding is inside the first RNG_KERNEL interval. */
int prng_prof_events(const prng_t *h, uint64_t cap, uint32_t *name_id, double *start_s,
                     double *end_s, uint64_t *n_out, double *wall_s, prng_err_t *err);

/* cf4ocl's ccl_prof_calc arithmetic over arbitrary intervals:
 *  agg_abs[nnames]          sum of durations per name                       (CCLProfAgg)
 *  overlap[nnames*nnames]   overlap[a*nnames+b] (a <= b): total pairwise intersection
 *                           of distinct events named a and b                 (CCLProfOverlap)
 *  effective                measure of the union of all intervals ("eff.", Fig. 3)
 *  elapsed_out              = elapsed if elapsed > 0 else max end - min start
 * Plain host arithmetic (endpoint sweep, O(E log E + S * nnames^2)); no GPU needed. */
int prng_prof_calc(uint64_t nevents, const uint32_t *name_id, const double *start_s,
                   const double *end_s, uint32_t nnames, double elapsed, double *agg_abs,
                   double *overlap, double *effective, double *elapsed_out, prng_err_t *err);

/* Sort flags of the summary, after cf4ocl's (CCL_PROF_AGG_SORT_TIME |
 * CCL_PROF_SORT_DESC, CCL_PROF_OVERLAP_SORT_DURATION | CCL_PROF_SORT_DESC). */
#define PRNG_PROF_AGG_SORT_NAME 0x0
#define PRNG_PROF_AGG_SORT_TIME 0x1
#define PRNG_PROF_OVERLAP_SORT_NAME 0x0
#define PRNG_PROF_OVERLAP_SORT_DURATION 0x1
#define PRNG_PROF_SORT_ASC 0x0
#define PRNG_PROF_SORT_DESC 0x10

/* NEXT-2: the text summary of cf4ocl's ccl_prof_get_summary in the layout of Fig. 3
 * (P:297-321): aggregate table (name, relative %, absolute s), event-overlap table,
 * "Tot. of all events (eff.)", "Total ellapsed time" (sic, as printed), device and host
 * shares.  names[nnames] are the event names (NULL = prng_event_name(id)); only names
 * that occur are listed; zero overlaps are omitted.  Writes a NUL-terminated string into
 * buf (cap bytes); *len (may be NULL) gets the full length, PRNG_EINVAL if cap is short. */
int prng_prof_summary(uint64_t nevents, const uint32_t *name_id, const double *start_s,
                      const double *end_s, uint32_t nnames, const char *const *names, double elapsed,
                      int agg_sort, int overlap_sort, char *buf, uint64_t cap, uint64_t *len,
                      prng_err_t *err);

/* NEXT-2: the profiler's export table: one line per event,
 * "queue<TAB>start_ns<TAB>end_ns<TAB>event name", sorted by (start, end, queue), LF line
 * endings, written to `path`.  queues[nnames] name the queue of each event name (NULL =
 * "Main" for kernels, "Comms" for READ_BUFFER, "Host" for OUT).  For ccl_plot_events-style
 * charts (tools/plot_events.py, Fig. 5). */
int prng_prof_export(uint64_t nevents, const uint32_t *name_id, const double *start_s,
                     const double *end_s, uint32_t nnames, const char *const *names,
                     const char *const *queues, const char *path, prng_err_t *err);

/* The same-box roofline probes bench.py divides by (memset, SM fill / store kernels, D2H
 * host link) are measurement tools, not part of the hot path: they live in their own
 * library, libprng_probes.so (include/prng_probes.h). */

#ifdef PRNG_CHECKED
/* Test-only, and exported only by the bounds-checked build libprng_b200_checked.so
 * (-DPRNG_CHECKED; PRNG_B200_CHECKED=1 makes the Python package load it).  In that build every
 * ring store and state access of the seed / batch / epoch kernels is checked against its
 * launch's arguments and traps on a violation.  This is the negative control: one launch into
 * a one-slot ring 4 u64 short of the handle's count (count % 4 == 0, >= 8) must trap, so the
 * call returns PRNG_ECUDA.  The CUDA context is then unusable: call it in a process of its
 * own (tests/test_checked_build.py). */
int prng_checked_selftest(prng_t *h, prng_err_t *err);
#endif

#ifdef __cplusplus
}
#endif
#endif /* PRNG_B200_H */
