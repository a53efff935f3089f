// prng_kernels.cuh -- sm_100a kernels of the massive-PRNG hot path (arXiv 1609.01257 §5).
//
//   a1  seed_kernel   : state[g] = seed64(gid_begin + g, seed)          (readings A1-A4)
//   a2+a3 batch_kernel: T iterations of xorshift64 per launch, state held in registers,
//                       every iteration stored with 16-byte (or 32-byte) coalesced vector
//                       stores into a ring of iteration slots            (A5-A8)
//   NEXT-4 jump_columns_kernel: GF(2) jump-ahead matrices for time-parallel launches
//
// The paper's OpenCL `prng` kernel re-reads its state from one buffer and writes the
// successor to another every iteration (16 B/number of global traffic).
// Here a persistent grid-strided warp owns a "piece" of 32*NPT consecutive gids, keeps
// its NPT states in registers for all T iterations of the launch and only writes
// (8 B/number); the state array is read once and written once per launch.
//
// Work decomposition:
//   piece p covers gids [p*32*NPT, (p+1)*32*NPT) of the handle's range;
//   lane l holds, for v in 0..NPT/VEC-1, the VEC consecutive gids at
//   p*32*NPT + v*32*VEC + l*VEC  -> one warp-wide store instruction writes 32*VEC*8
//   contiguous bytes (512 B for VEC = 2, 1 KiB for VEC = 4).
//   warp w of W processes units w, w+W, w+2W, ... (`rounds` of them); a unit is a piece
//   over all of the launch's iterations, or (time-parallel mode, small numrn) a piece
//   over one chunk of them.  The host sizes W so that every warp gets the same number of
//   units +- 1 and the grid is <= one wave.
//
// No code here is shared with oracle/ (the CPU definition); see DESIGN.md §2.
#pragma once
#include <cstdint>
#ifdef PRNG_CHECKED
#include <cstdio>
#endif

namespace prngk {

// ---------------------------------------------------------------- checked build
// -DPRNG_CHECKED (libprng_b200_checked.so, PRNG_B200_CHECKED=1; tests only): every global
// store and state load of the seed / batch kernels is checked against its launch's
// arguments -- inside the ring of nslots x pitch, column + width <= count, aligned to its
// vector width; state index + width <= count -- and traps on a violation.  compute-sanitizer
// is closed on the GPU pool, so the kernels carry their own bounds checks.
// The default build compiles them out.
#ifdef PRNG_CHECKED
__device__ __noinline__ void check_fail(const char *what, const void *p, uint64_t v, uint64_t n) {
    printf("prng bounds violation: %s at %p (index %llu, width %llu), block %u thread %u\n", what, p,
           (unsigned long long)v, (unsigned long long)n, blockIdx.x, threadIdx.x);
    __trap();
}
#define PRNG_CHK(cond, what, p, v, n) \
    do {                               \
        if (!(cond)) ::prngk::check_fail(what, p, v, n); \
    } while (0)
#else
#define PRNG_CHK(cond, what, p, v, n) \
    do {                               \
    } while (0)
#endif

// ---------------------------------------------------------------- the method's arithmetic
// A1: Wang's 32-bit multiplicative hash ("hash32shiftmult"), P:173 [wang1997inthash].
__device__ __forceinline__ uint32_t wang32(uint32_t x) {
    x = (x ^ 61u) ^ (x >> 16);
    x = x * 9u;
    x = x ^ (x >> 4);
    x = x * 0x27d4eb2du;
    x = x ^ (x >> 15);
    return x;
}

// A4: seed premix (the paper has no seed; fmix64(0) == 0 keeps seed 0 == the paper).
__device__ __forceinline__ uint64_t premix64(uint64_t z) {
    z ^= z >> 33;
    z *= 0xff51afd7ed558ccdull;
    z ^= z >> 33;
    z *= 0xc4ceb9fe1a85ec53ull;
    z ^= z >> 33;
    return z;
}

// A2/A3: two 32-bit hashes of the 32-bit gid composed into the 64-bit state; 0 -> 1.
__device__ __forceinline__ uint64_t seed64(uint32_t g, uint32_t key_hi, uint32_t key_lo) {
    const uint64_t st = ((uint64_t)wang32(g ^ key_hi) << 32) | (uint64_t)wang32(g ^ 0x9E3779B9u ^ key_lo);
    return st ? st : 1ull;
}

// A5: Marsaglia's xor64 triple (13, 7, 17), P:177 [marsaglia2003xorshift].
__device__ __forceinline__ uint64_t xorshift64(uint64_t x) {
    x ^= x << 13;
    x ^= x >> 7;
    x ^= x << 17;
    return x;
}

// NEXT-3 (P:177 limitation 1, "a more complex PRNG could probably be used"):
// optional xorshift64*-style output scrambling -- the emitted value is the state times
// Vigna's xorshift64* multiplier (mod 2^64); the state recurrence is unchanged (DESIGN.md
// A19).  One 64-bit multiply per number on the otherwise idle FMA pipe.
constexpr uint64_t kStarMul = 0x2545F4914F6CDD1Dull;
template <int OUT>
__device__ __forceinline__ uint64_t emit(uint64_t x) {
    if constexpr (OUT == 1)
        return x * kStarMul;
    else
        return x;
}

// ---------------------------------------------------------------- vector memory helpers
// Plain write-back stores: the measured alternatives (.cs, L2::evict_first, L1::no_allocate,
// TMA bulk stores from shared memory) were not faster on B200.
__device__ __forceinline__ void st_v4(uint64_t *p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
__device__ __forceinline__ void st_v2(uint64_t *p, uint64_t a, uint64_t b) {
    asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_v4(const uint64_t *p, uint64_t &a, uint64_t &b, uint64_t &c, uint64_t &d) {
    asm volatile("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}
__device__ __forceinline__ void ld_v2(const uint64_t *p, uint64_t &a, uint64_t &b) {
    asm volatile("ld.global.nc.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
}

template <int VEC>
__device__ __forceinline__ void store_vec(uint64_t *p, const uint64_t *x) {
    if constexpr (VEC == 4)
        st_v4(p, x[0], x[1], x[2], x[3]);
    else
        st_v2(p, x[0], x[1]);
}
template <int VEC>
__device__ __forceinline__ void load_vec(const uint64_t *p, uint64_t *x) {
    if constexpr (VEC == 4)
        ld_v4(p, x[0], x[1], x[2], x[3]);
    else
        ld_v2(p, x[0], x[1]);
}

// Weak (non-.nc) loads: the epoch kernel re-reads states that the same thread wrote at the
// end of its previous unit (see batch_kernel_epoch).
__device__ __forceinline__ void ld_v4_wk(const uint64_t *p, uint64_t &a, uint64_t &b, uint64_t &c, uint64_t &d) {
    asm volatile("ld.global.v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}
__device__ __forceinline__ void ld_v2_wk(const uint64_t *p, uint64_t &a, uint64_t &b) {
    asm volatile("ld.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
}
template <int VEC>
__device__ __forceinline__ void load_vec_wk(const uint64_t *p, uint64_t *x) {
    if constexpr (VEC == 4)
        ld_v4_wk(p, x[0], x[1], x[2], x[3]);
    else
        ld_v2_wk(p, x[0], x[1]);
}

// ---------------------------------------------------------------- a1: seed kernel
struct SeedArgs {
    uint64_t *state;     // [count] out, 16-byte aligned
    uint64_t count;      // gids in this handle's range
    uint64_t gid_begin;  // first global gid (< 2^32)
    uint64_t seed;
};

// Each thread seeds 2 consecutive gids per grid-stride step and writes them with one
// 16-byte store.
__global__ void __launch_bounds__(256) seed_kernel(SeedArgs a) {
    const uint64_t m = premix64(a.seed);
    const uint32_t key_hi = (uint32_t)m, key_lo = (uint32_t)(m >> 32);
    const uint64_t stride = 2ull * gridDim.x * blockDim.x;
    for (uint64_t i = 2ull * (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x); i < a.count; i += stride) {
        const uint32_t g = (uint32_t)(a.gid_begin + i);
        const uint64_t s0 = seed64(g, key_hi, key_lo);
        if (i + 1 < a.count) {
            const uint64_t s1 = seed64(g + 1u, key_hi, key_lo);
            PRNG_CHK(((uintptr_t)(a.state + i) & 15) == 0, "seed store", a.state + i, i, 2);
            st_v2(a.state + i, s0, s1);
        } else {
            PRNG_CHK(i < a.count, "seed store", a.state + i, i, 1);
            a.state[i] = s0;
        }
    }
}

// ---------------------------------------------------------------- a2+a3: batch kernel
struct BatchArgs {
    uint64_t *dst;            // slot s starts at dst + s * pitch (32-byte aligned)
    uint64_t pitch;           // u64 elements between slots (multiple of 4, >= count)
    uint32_t nslots;          // ring slots R (iteration t of the launch -> slot (slot0 + t) mod R)
    uint32_t slot0;           // slot of the launch's first iteration
    uint64_t *state;          // [count] in/out: state before / after the launch
    uint64_t count;           // gids in the handle's range
    uint32_t iters;           // T iterations in this launch
    uint32_t first_is_state;  // 1: the launch's first iteration is iteration 0 (= the seeds):
                              //    emit the state unchanged, then step (A6)
    uint64_t npieces;         // ceil(count / (32 * NPT))
    uint32_t rounds;          // ceil(npieces * nchunks / warps in grid)
    // Time-parallel mode (NEXT-4, small numrn): the launch's iterations are cut into nchunks
    // chunks of chunk_len; chunk c starts from J_c * state where J_c = T^(c*chunk_len + e)
    // is the GF(2) matrix of xs^(c*chunk_len + e) (e = 0 if first_is_state else 1), stored
    // as 64 columns J_c e_i at jump[c*64 + i].  nchunks == 1: the plain sequential mode.
    // The epoch kernel reuses nchunks / chunk_len as its epoch count / length.
    uint32_t nchunks;
    uint32_t chunk_len;
    const uint64_t *jump;     // [nchunks][64] (nchunks > 1)
    uint64_t *state_out;      // nchunks > 1: the last chunk writes the final state here
    uint32_t order;           // 0: unit r*W + w to warp w in round r (adjacent CTAs, adjacent
                              //    pieces); 1: CTA b takes units [b*rounds*wpb, (b+1)*rounds*wpb)
    // a1 fused into the launch (PRNG_OPT_FUSED_SEED): seeding != 0 -> a unit computes its
    // start states as seed64(gid_begin + gid, premix64(seed)) in registers instead of
    // loading them from `state` (which it still writes at the end); the launch then
    // behaves exactly as if seed_kernel had written `state` before it.
    uint32_t seeding;
    uint64_t seed;
    uint64_t gid_begin;
};

// Checked build: a store of n u64 at p into the launch's ring (or zero-copy host half).
__device__ __forceinline__ void chk_ring(const BatchArgs &a, const uint64_t *p, int n) {
#ifdef PRNG_CHECKED
    const uint64_t off = (uint64_t)(p - a.dst);  // wraps to a huge value below dst
    const bool ok = p >= a.dst && off + n <= (uint64_t)a.nslots * a.pitch && off % a.pitch + n <= a.count &&
                    ((uintptr_t)p % (8u * n)) == 0;
    PRNG_CHK(ok, "ring store", p, off, n);
#endif
}
// ... and an access of n u64 at state index idx (state, state_out).
__device__ __forceinline__ void chk_state(const BatchArgs &a, const uint64_t *base, uint64_t idx, int n) {
#ifdef PRNG_CHECKED
    PRNG_CHK(idx + n <= a.count && ((uintptr_t)(base + idx) % (8u * n)) == 0, "state access", base + idx, idx, n);
#endif
}

// The start states of a lane's NPT gids (handle-relative base, VEC-wide groups vs apart):
// seeds computed in registers (a1 fused) or loaded from the state array.  Gids at or past
// `count` (the ragged last piece, PARTIAL only) get 0 and are never stored.
template <int VEC, int NPT, bool FULLP, bool NC = true>
__device__ __forceinline__ void start_states(const BatchArgs &a, uint64_t base, uint64_t vs, uint64_t *x,
                                             bool seed_now) {
    constexpr int NV = NPT / VEC;
    if (seed_now) {
        const uint64_t m = premix64(a.seed);
        const uint32_t key_hi = (uint32_t)m, key_lo = (uint32_t)(m >> 32);
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
                const uint64_t idx = base + (uint64_t)v * vs + e;
                const uint64_t s = seed64((uint32_t)(a.gid_begin + idx), key_hi, key_lo);
                x[v * VEC + e] = (FULLP || idx < a.count) ? s : 0ull;
            }
    } else if constexpr (FULLP) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            chk_state(a, a.state, base + (uint64_t)v * vs, VEC);
            if constexpr (NC)
                load_vec<VEC>(a.state + base + (uint64_t)v * vs, x + v * VEC);
            else
                load_vec_wk<VEC>(a.state + base + (uint64_t)v * vs, x + v * VEC);
        }
    } else {
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
                const uint64_t idx = base + (uint64_t)v * vs + e;
                x[v * VEC + e] = idx < a.count ? a.state[idx] : 0ull;
            }
    }
}

// y = J x over GF(2): XOR of the columns J e_i selected by the bits of x (xs^k is linear).
__device__ __forceinline__ uint64_t gf2_matvec(const uint64_t *__restrict__ J, uint64_t x) {
    uint64_t y = 0;
#pragma unroll 16
    for (int i = 0; i < 64; ++i) y ^= __ldg(J + i) & (0ull - ((x >> i) & 1ull));
    return y;
}

// Columns of J_c = T^(c*L + e), c = 0..C-1, by one CTA of 64 threads (thread i owns column
// i; xs is GF(2)-linear, so the column T^k e_i is xs^k(e_i)).  P = T^L by binary
// exponentiation (log2 L matrix products, each column a 64-step mat-vec against the other
// matrix's columns in shared memory), J_0 = T^e, J_c = P * J_{c-1}.
__device__ __forceinline__ uint64_t gf2_matvec_smem(const uint64_t *M, uint64_t x) {
    uint64_t y = 0;
#pragma unroll 16
    for (int b = 0; b < 64; ++b) y ^= M[b] & (0ull - ((x >> b) & 1ull));
    return y;
}

__global__ void __launch_bounds__(64) jump_columns_kernel(uint64_t *jump, uint32_t C, uint64_t L, uint32_t e) {
    __shared__ uint64_t B[64], R[64];
    const uint32_t i = threadIdx.x;
    const uint64_t t_col = xorshift64(1ull << i);  // T e_i
    B[i] = t_col;
    R[i] = 1ull << i;  // identity
    __syncthreads();
    for (uint64_t k = L; k; k >>= 1) {
        if (k & 1) {
            const uint64_t r = gf2_matvec_smem(B, R[i]);  // R = B R
            __syncthreads();
            R[i] = r;
            __syncthreads();
        }
        const uint64_t b = gf2_matvec_smem(B, B[i]);  // B = B B
        __syncthreads();
        B[i] = b;
        __syncthreads();
    }
    // R = P = T^L (column i in R[i])
    uint64_t col = e ? t_col : (1ull << i);
    jump[i] = col;
    for (uint32_t c = 1; c < C; ++c) {
        col = gf2_matvec_smem(R, col);
        jump[(uint64_t)c * 64 + i] = col;
    }
}

// Checkpoint / resume: state[g] = J * state[g] for every gid (J = T^k from
// jump_columns_kernel), i.e. k xorshift steps in one GF(2) mat-vec per state.
__global__ void __launch_bounds__(256) jump_states_kernel(uint64_t *state, uint64_t count, const uint64_t *J) {
    __shared__ uint64_t Js[64];
    if (threadIdx.x < 64) Js[threadIdx.x] = J[threadIdx.x];
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < count; g += stride)
        state[g] = gf2_matvec_smem(Js, state[g]);
}

// One work unit of a warp: the gids of one piece over iterations [t_begin, t_begin + t_count).
struct Unit {
    uint64_t base;         // this lane's first gid (handle-relative) of the piece
    uint32_t t_begin;      // first iteration of the launch this unit emits
    uint32_t t_count;      // iterations it emits
    const uint64_t *jump;  // nullptr: start from the state; else from J * state
    uint64_t *state_out;   // nullptr: do not write the state back
    bool emit_first;       // true: the unit's first iteration emits its start value unchanged
};

enum PieceMode { FULL = 0, PARTIAL = 1 };

// The per-iteration CTA barrier: the warps of a CTA (adjacent pieces) meet at named barrier
// 1 after every iteration's stores, so a CTA writes one contiguous chunk per iteration
// (measured: -6 % without it; free-running warps at full occupancy ~6.2 TB/s against
// 6.7-6.9).  The non-.aligned form by default: the warps of one CTA reach it
// from different instructions (full and partial pieces, the peeled first trip, idle trips),
// which `bar.sync` (= barrier.sync.aligned) does not allow -- compute-sanitizer synccheck
// flags it.  AL = true: the CTA's warps are known to run identical instruction sequences
// this round (all full pieces, same trip count), which the .aligned form needs.
template <bool AL = false>
__device__ __forceinline__ void cta_barrier(uint32_t threads) {
    if constexpr (AL)
        asm volatile("bar.sync 1, %0;" ::"r"(threads) : "memory");
    else
        asm volatile("barrier.sync 1, %0;" ::"r"(threads) : "memory");
}

// PP: the hot loop is unrolled by two with the state ping-ponging between two register
// arrays, so each step's results land directly in the registers the next 32-B store
// reads (without it ptxas copies 8 registers into a staging octet before every STG.256:
// 16 extra IMAD.MOV per iteration at NPT = 8, 13 % of the loop's instructions).
template <int VEC, int NPT, int MODE, int OUT = 0, bool AL = false, bool PP = false>
__device__ __forceinline__ void run_piece(const BatchArgs &a, const Unit &u, uint32_t bar_threads) {
    constexpr int NV = NPT / VEC;
    constexpr uint64_t vs = 32ull * VEC;  // elements between a lane's vectors
    const uint64_t base = u.base;
    uint64_t x[NPT];
    // ---- the NPT start states of this lane (read once per unit, or seeded: a1 fused)
    start_states<VEC, NPT, MODE == FULL>(a, base, vs, x, a.seeding != 0);
    if (u.jump) {  // time-parallel chunk: jump ahead (c*L + e) steps in one GF(2) mat-vec
#pragma unroll
        for (int j = 0; j < NPT; ++j) x[j] = gf2_matvec(u.jump, x[j]);
    }
    uint32_t slot = (uint32_t)(((uint64_t)a.slot0 + u.t_begin) % a.nslots);
    uint64_t *p = a.dst + (uint64_t)slot * a.pitch + base;
    const uint64_t wrap = (uint64_t)(a.nslots - 1) * a.pitch;
    // One loop trip: store this iteration (if the unit is active), meet the CTA barrier,
    // advance to the next ring slot.  Every unit of a launch makes the same number of trips
    // (the barriers must match): a shorter last chunk idles through its surplus trips.  The
    // first trip is peeled so the hot loop has no conditions.
    auto trip = [&](bool active, const uint64_t *src) {
        if (active) {
            if constexpr (MODE == FULL) {
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    chk_ring(a, p + v * vs, VEC);
                    if constexpr (OUT == 0) {
                        store_vec<VEC>(p + v * vs, src + v * VEC);
                    } else {
                        uint64_t y[VEC];
#pragma unroll
                        for (int e = 0; e < VEC; ++e) y[e] = emit<OUT>(src[v * VEC + e]);
                        store_vec<VEC>(p + v * vs, y);
                    }
                }
            } else {
#pragma unroll
                for (int v = 0; v < NV; ++v)
#pragma unroll
                    for (int e = 0; e < VEC; ++e)
                        if (base + (uint64_t)v * vs + e < a.count) {
                            chk_ring(a, p + v * vs + e, 1);
                            p[v * vs + e] = emit<OUT>(src[v * VEC + e]);
                        }
            }
        }
        cta_barrier<AL>(bar_threads);
        if (++slot == a.nslots) {  // warp-uniform
            slot = 0;
            p -= wrap;
        } else {
            p += a.pitch;
        }
    };
    auto step = [&]() {
#pragma unroll
        for (int j = 0; j < NPT; ++j) x[j] = xorshift64(x[j]);
    };
    const uint32_t t_loop = a.nchunks > 1 ? a.chunk_len : a.iters;
    const uint32_t t_act = u.t_count;
    uint32_t t = 0;
    if (t_act > 0) {
        if (!u.emit_first) step();
        trip(true, x);
        t = 1;
    }
    if constexpr (PP && MODE == FULL) {
        uint64_t y[NPT];
        for (; t + 1 < t_act; t += 2) {  // the hot loop, two iterations per trip
#pragma unroll
            for (int j = 0; j < NPT; ++j) y[j] = xorshift64(x[j]);
            trip(true, y);
#pragma unroll
            for (int j = 0; j < NPT; ++j) x[j] = xorshift64(y[j]);
            trip(true, x);
        }
    }
    for (; t < t_act; ++t) {  // the hot loop (PP: the odd last iteration)
        step();
        trip(true, x);
    }
    for (; t < t_loop; ++t) trip(false, x);  // idle trips (short last chunk)
    // ---- write the state back (== the unit's last iteration) if this unit ends the launch
    if (u.state_out) {
        if constexpr (MODE == FULL) {
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                chk_state(a, u.state_out, base + (uint64_t)v * vs, VEC);
                store_vec<VEC>(u.state_out + base + (uint64_t)v * vs, x + v * VEC);
            }
        } else {
#pragma unroll
            for (int v = 0; v < NV; ++v)
#pragma unroll
                for (int e = 0; e < VEC; ++e) {
                    const uint64_t idx = base + (uint64_t)v * vs + e;
                    if (idx < a.count) u.state_out[idx] = x[v * VEC + e];
                }
        }
    }
}

// The work unit dealt to a warp: unit index w -> (piece = w mod npieces, chunk = w div
// npieces), so adjacent warps hold adjacent pieces of the same chunk.
template <int NPT, int VEC>
__device__ __forceinline__ Unit make_unit(const BatchArgs &a, uint64_t unit, uint32_t lane) {
    Unit u;
    const uint64_t piece = unit % a.npieces, chunk = unit / a.npieces;
    u.base = piece * 32ull * NPT + (uint64_t)lane * VEC;
    if (a.nchunks <= 1) {
        u.t_begin = 0;
        u.t_count = a.iters;
        u.jump = nullptr;
        u.state_out = a.state;  // in place: each lane reads then writes its own states
        u.emit_first = a.first_is_state != 0;
    } else {
        u.t_begin = (uint32_t)chunk * a.chunk_len;
        const uint32_t left = a.iters - u.t_begin;
        u.t_count = left < a.chunk_len ? left : a.chunk_len;
        u.jump = a.jump + chunk * 64;
        u.state_out = (chunk + 1 == a.nchunks) ? a.state_out : nullptr;
        u.emit_first = true;
    }
    return u;
}

// AL: use the .aligned CTA barrier in rounds where the CTA is uniform (see cta_barrier).
template <int VEC, int NPT, int OUT = 0, bool AL = false, bool PP = false>
__global__ void __launch_bounds__(256) batch_kernel(BatchArgs a) {
    static_assert(NPT % VEC == 0, "NPT must be a multiple of VEC");
    constexpr uint64_t PIECE = 32ull * NPT;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t wpb = blockDim.x >> 5;
    const uint64_t cta_warp0 = (uint64_t)blockIdx.x * wpb;
    const uint64_t nunits = a.npieces * (a.nchunks ? a.nchunks : 1);
    for (uint32_t r = 0; r < a.rounds; ++r) {
        // unit index of this CTA's warp 0 in round r; the CTA's warps hold consecutive units
        const uint64_t first = a.order ? ((uint64_t)blockIdx.x * a.rounds + r) * wpb : (uint64_t)r * nwarps + cta_warp0;
        const uint64_t unit = first + (warp - cta_warp0);
        if (unit >= nunits) break;  // warp-uniform: a suffix of the CTA's warps
        const Unit u = make_unit<NPT, VEC>(a, unit, lane);
        // warps of this CTA holding a unit in round r: a prefix of the CTA's warps
        const uint32_t bar_threads = 32u * (uint32_t)(nunits - first < wpb ? nunits - first : wpb);
        const uint64_t piece = unit % a.npieces;
        if ((piece + 1) * PIECE <= a.count) {
            if constexpr (AL) {
                // uniform round: every active warp of the CTA has a full piece and the same
                // trip count (only the last piece can be partial, only the last chunk short)
                const uint64_t last = first + bar_threads / 32 - 1;
                const uint64_t pf = first % a.npieces;
                const bool has_partial = a.count % PIECE != 0 && pf + (last - first) >= a.npieces - 1;
                const bool same_trips = a.nchunks <= 1 || first / a.npieces == last / a.npieces ||
                                        last / a.npieces + 1 < a.nchunks;
                if (!has_partial && same_trips)
                    run_piece<VEC, NPT, FULL, OUT, true, PP>(a, u, bar_threads);
                else
                    run_piece<VEC, NPT, FULL, OUT, false, PP>(a, u, bar_threads);
            } else {
                run_piece<VEC, NPT, FULL, OUT, false, PP>(a, u, bar_threads);
            }
        } else {
            run_piece<VEC, NPT, PARTIAL, OUT, false>(a, u, bar_threads);
        }
    }
}

// ---------------------------------------------------------------- a2+a3, epoch-major order
// L2 absorption: batch_kernel runs each piece through all T iterations of a
// launch, so when a launch wraps a ring of R slots a warp rewrites its piece's R slots
// every R iterations; if the grid's live set (R x warps x bytes per warp-iteration) fits
// in L2 the rewrites merge in L2 and never reach DRAM.  Here the launch is cut into epochs
// of E <= R iterations: in epoch e every warp runs each of its pieces (piece r*W + w,
// r = 0, 1, ...) through iterations [eE, eE + E), keeping the state in registers inside a
// unit and in d_state between epochs, so an address is rewritten only a whole epoch (all
// pieces x E iterations) later.  Extra traffic: 16 B per number per epoch (2/E of the
// output).
//
// Every piece of a warp is always run by the same lanes, so a state written at the end of
// one unit is read back by the thread that wrote it: a weak load is enough (same-thread
// program order, PTX memory model) -- and measured faster than a .cg (LDG.STRONG.GPU)
// load or prefetching the next unit's state during the current one (exp21).  CTA barrier
// every iteration as in batch_kernel.
// One unit of the epoch kernel: a piece through iterations [t_begin, t_begin + t_count).
template <int VEC, int NPT, int OUT, bool FULL, bool AL = false>
__device__ __forceinline__ void epoch_unit(const BatchArgs &a, uint64_t *x, uint64_t base, uint32_t slot,
                                           uint32_t t_count, bool emit_first, uint32_t bar_threads) {
    constexpr int NV = NPT / VEC;
    const uint64_t wrap = (uint64_t)(a.nslots - 1) * a.pitch;
    uint64_t *p = a.dst + (uint64_t)slot * a.pitch + base;
    auto trip = [&]() {
        if constexpr (FULL) {
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                uint64_t y[VEC];
#pragma unroll
                for (int q = 0; q < VEC; ++q) y[q] = emit<OUT>(x[v * VEC + q]);
                chk_ring(a, p + v * 32 * VEC, VEC);
                store_vec<VEC>(p + v * 32 * VEC, y);
            }
        } else {
#pragma unroll
            for (int v = 0; v < NV; ++v)
#pragma unroll
                for (int q = 0; q < VEC; ++q)
                    if (base + (uint64_t)v * 32 * VEC + q < a.count) {
                        chk_ring(a, p + v * 32 * VEC + q, 1);
                        p[v * 32 * VEC + q] = emit<OUT>(x[v * VEC + q]);
                    }
        }
        cta_barrier<AL>(bar_threads);
        if (++slot == a.nslots) {  // warp-uniform
            slot = 0;
            p -= wrap;
        } else {
            p += a.pitch;
        }
    };
    auto step = [&]() {
#pragma unroll
        for (int j = 0; j < NPT; ++j) x[j] = xorshift64(x[j]);
    };
    if (!emit_first) step();
    trip();
    for (uint32_t t = 1; t < t_count; ++t) {  // the hot loop
        step();
        trip();
    }
}

template <int VEC, int NPT, int OUT = 0, bool AL = false>
__global__ void __launch_bounds__(256) batch_kernel_epoch(BatchArgs a) {
    static_assert(NPT % VEC == 0, "NPT must be a multiple of VEC");
    constexpr int NV = NPT / VEC;
    constexpr uint64_t PIECE = 32ull * NPT;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t wpb = blockDim.x >> 5;
    const uint64_t cta_warp0 = (uint64_t)blockIdx.x * wpb;
    const uint64_t warp = cta_warp0 + (threadIdx.x >> 5);
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    if (warp >= a.npieces) return;  // warp-uniform; such warps are never counted in bar_threads
    const uint64_t kw = (a.npieces - warp + nwarps - 1) / nwarps;  // pieces of this warp
    // Every warp of the CTA that has pieces takes part in every barrier of every round up to
    // the CTA's last (its warp 0 has the most pieces): a warp without a piece in a round
    // idles through that round's barriers, so the CTA's warps never run into different
    // rounds (or epochs) on the same named barrier.
    const uint64_t kw_cta = (a.npieces - cta_warp0 + nwarps - 1) / nwarps;
    const uint32_t bar_threads = 32u * (uint32_t)(a.npieces - cta_warp0 < wpb ? a.npieces - cta_warp0 : wpb);
    const uint32_t E = a.chunk_len;
    for (uint32_t e = 0; e < a.nchunks; ++e) {
        const uint32_t t_begin = e * E;
        const uint32_t t_count = a.iters - t_begin < E ? a.iters - t_begin : E;
        const bool emit_first = e == 0 && a.first_is_state;
        const uint32_t slot_begin = (uint32_t)(((uint64_t)a.slot0 + t_begin) % a.nslots);
        for (uint64_t r = 0; r < kw_cta; ++r) {
            if (r >= kw) {  // no piece for this warp in round r: idle through its barriers
                for (uint32_t t = 0; t < t_count; ++t) cta_barrier(bar_threads);
                continue;
            }
            const uint64_t piece = r * nwarps + warp;
            const uint64_t base = piece * PIECE + (uint64_t)lane * VEC;
            uint64_t x[NPT];
            const bool seed_now = e == 0 && a.seeding != 0;  // a1 fused: epoch 0 starts from the seeds
            if ((piece + 1) * PIECE <= a.count) {
                start_states<VEC, NPT, true, false>(a, base, 32ull * VEC, x, seed_now);
                // uniform round: all of the CTA's active warps hold a full piece in round r
                const uint64_t last = r * nwarps + cta_warp0 + bar_threads / 32 - 1;
                if (AL && last < a.npieces && (last + 1) * PIECE <= a.count)
                    epoch_unit<VEC, NPT, OUT, true, AL>(a, x, base, slot_begin, t_count, emit_first, bar_threads);
                else
                    epoch_unit<VEC, NPT, OUT, true, false>(a, x, base, slot_begin, t_count, emit_first, bar_threads);
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    chk_state(a, a.state, base + (uint64_t)v * 32 * VEC, VEC);
                    store_vec<VEC>(a.state + base + (uint64_t)v * 32 * VEC, x + v * VEC);
                }
            } else {  // the ragged last piece
                start_states<VEC, NPT, false>(a, base, 32ull * VEC, x, seed_now);
                epoch_unit<VEC, NPT, OUT, false>(a, x, base, slot_begin, t_count, emit_first, bar_threads);
#pragma unroll
                for (int v = 0; v < NV; ++v)
#pragma unroll
                    for (int q = 0; q < VEC; ++q) {
                        const uint64_t idx = base + (uint64_t)v * 32 * VEC + q;
                        if (idx < a.count) a.state[idx] = x[v * VEC + q];
                    }
            }
        }
    }
}

}  // namespace prngk
