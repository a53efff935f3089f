// Round-2 research probe (not product code): does bounding the drift between CTAs bring the
// iteration-major generator's DRAM write stream closer to the one-shot fill?
//
// profiles/r2_write_ceiling.md §2-3: a one-shot fill (write front moving through memory in
// order) keeps DRAM 91 % active; the persistent generator (each warp holds its piece for all
// T iterations, CTAs free-running, ~180 iterations of drift between them) 84 %.  With zero
// drift the grid would write one contiguous window of slot k at a time; a hard grid barrier
// per iteration costs ~1.5 us and was far slower.  Here CTAs are kept within a slack instead:
// every K iterations a CTA adds 1 to the counter of its group of iterations, and before it
// starts group j it waits until every CTA has finished group j - D (one polling thread, the
// CTA barrier that follows releases the rest).  Drift is then bounded by ~D*K iterations and
// a CTA only stalls when it runs ahead by more than that.
//
//   G1  the round-1/2 generator structure (one CTA of W warps per SM, NPT = 8 numbers per
//       thread in registers, 2 x 32-B stores per thread per iteration, CTA barrier every
//       iteration), no drift control
//   G4  G1 + the slack-bounded grid sync (K, D)
//   out[k][g] with pitch n, T iterations per piece, rounds of pieces as in the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -o drift drift.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>

__device__ __forceinline__ uint64_t xs(uint64_t x) {
    x ^= x << 13;
    x ^= x >> 7;
    x ^= x << 17;
    return x;
}
__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}
__device__ __forceinline__ void st4(uint64_t *p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
__device__ __forceinline__ void ld4(const uint64_t *p, uint64_t &a, uint64_t &b, uint64_t &c, uint64_t &d) {
    asm volatile("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}
__device__ __forceinline__ void bar(uint32_t n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }
// Pacing only, no memory ordering: relaxed operations (a release would drain the CTA's
// outstanding stores every K iterations -- measured 0.9-2.7 TB/s with red.release).
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void red_release(uint32_t *p, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v));
}

// K = 0: no drift control.  cnt: one counter per group of K global iterations (zeroed).
// ts != nullptr: CTA b records globaltimer at the start of every group into ts[b*ngroups + j].
template <int NPT>
__global__ void __launch_bounds__(256) g4(uint64_t *out, uint64_t *state, uint64_t n, uint32_t T, uint32_t K,
                                          uint32_t D, uint32_t *cnt, uint64_t *ts, uint32_t ngroups) {
    constexpr int NV = NPT / 4;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t wpb = blockDim.x >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * wpb;
    const uint64_t npieces = n / (32 * NPT);
    const uint64_t rounds = (npieces + nwarps - 1) / nwarps;
    uint64_t j = 0;        // group of K iterations this CTA is in
    uint32_t kk = 0;       // iterations left in the current group (0: a group starts)
    uint32_t pending = 0;  // thread 0: cnt[j - D], loaded one group ahead (latency hidden)
        for (uint64_t r = 0; r < rounds; ++r) {
        const uint64_t piece = r * nwarps + blockIdx.x * wpb + (threadIdx.x >> 5);
        const bool live = piece < npieces;
        const uint64_t base = piece * 32 * NPT + lane * 4;
        uint64_t x[NPT];
        if (live) {
#pragma unroll
            for (int v = 0; v < NV; ++v) ld4(state + base + v * 128, x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
        }
        uint64_t *p = out + base;
        for (uint32_t t = 0; t < T; ++t) {
            if (K && kk == 0) {
                if (threadIdx.x == 0) {
                    if (j >= D) {
                        const uint32_t *c = cnt + (j - D);
                        uint32_t v = j > D ? pending : ld_acquire(c);
                        while (v < gridDim.x) {
                            __nanosleep(32);
                            v = ld_acquire(c);
                        }
                    }
                    if (j + 1 >= D) pending = ld_acquire(cnt + (j + 1 - D));  // checked next group
                    if (ts && j < ngroups) {
                        uint64_t g;
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
                        ts[(uint64_t)blockIdx.x * ngroups + j] = g;
                    }
                }
                kk = K;
            }
            if (live) {
#pragma unroll
                for (int q = 0; q < NPT; ++q) x[q] = xs(x[q]);
#pragma unroll
                for (int v = 0; v < NV; ++v) st4(p + v * 128, x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
            }
            bar(blockDim.x);
            if (K && --kk == 0) {
                if (threadIdx.x == 0) red_release(cnt + j, 1);
                ++j;
            }
            p += n;
        }
        if (live) {
#pragma unroll
            for (int v = 0; v < NV; ++v) st4(state + base + v * 128, x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
        }
    }
}

__global__ void init_state(uint64_t *s, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        s[i] = mix(i + 1) | 1;
}

int main(int argc, char **argv) {
    const uint64_t n = argc > 1 ? strtoull(argv[1], 0, 10) : (1ull << 24);
    const uint32_t T = argc > 2 ? atoi(argv[2]) : 1000;
    const char *mode = argc > 3 ? argv[3] : "sweep";
    const uint64_t out_elems = n * T;
    uint64_t *out, *state;
    if (cudaMalloc(&out, out_elems * 8) != cudaSuccess || cudaMalloc(&state, n * 8) != cudaSuccess) return 1;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    init_state<<<sms * 4, 256>>>(state, n);
    const uint32_t maxgroups = 1u << 22;
    uint32_t *cnt;
    cudaMalloc(&cnt, maxgroups * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](int W, int cps, uint32_t K, uint32_t D) {
        const unsigned grid = sms * cps;
        auto launch = [&] {
            cudaMemsetAsync(cnt, 0, maxgroups * 4);
            g4<8><<<grid, 32 * W>>>(out, state, n, T, K, D, cnt, nullptr, 0);
        };
        launch();
        cudaDeviceSynchronize();
        float best = 1e30f, sum = 0;
        const int reps = 3;
        for (int r = 0; r < reps; ++r) {
            cudaMemsetAsync(cnt, 0, maxgroups * 4);
            cudaEventRecord(a);
            g4<8><<<grid, 32 * W>>>(out, state, n, T, K, D, cnt, nullptr, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
            sum += ms;
        }
        cudaError_t e = cudaGetLastError();
        printf("{\"warps_per_cta\": %d, \"ctas_per_sm\": %d, \"K\": %u, \"D\": %u, \"n\": %llu, \"T\": %u, "
               "\"gbs_best\": %.1f, \"gbs_mean\": %.1f, \"err\": \"%s\"}\n",
               W, cps, K, D, (unsigned long long)n, T, out_elems * 8.0 / (best * 1e-3) / 1e9,
               out_elems * 8.0 / (sum / reps * 1e-3) / 1e9, cudaGetErrorString(e));
        fflush(stdout);
    };
    if (!strcmp(mode, "drift")) {
        // drift of the free-running structure: per-CTA timestamps at every 16th iteration
        const uint32_t K = 16, ngroups = 4096;
        uint64_t *ts;
        cudaMalloc(&ts, (uint64_t)sms * ngroups * 8);
        cudaMemset(ts, 0, (uint64_t)sms * ngroups * 8);
        cudaMemset(cnt, 0, maxgroups * 4);
        // D huge: never waits (counter only), timestamps only
        g4<8><<<sms, 128>>>(out, state, n, T, K, 1u << 30, cnt, ts, ngroups);
        cudaDeviceSynchronize();
        uint64_t *h = (uint64_t *)malloc((uint64_t)sms * ngroups * 8);
        cudaMemcpy(h, ts, (uint64_t)sms * ngroups * 8, cudaMemcpyDeviceToHost);
        // for each group j: spread (max - min) of the CTA start times, in us and in iterations
        for (uint32_t j = 0; j < ngroups; j += 256) {
            uint64_t lo = ~0ull, hi = 0;
            for (int c = 0; c < sms; ++c) {
                const uint64_t v = h[(uint64_t)c * ngroups + j];
                if (v < lo) lo = v;
                if (v > hi) hi = v;
            }
            const double per_group_ns = (double)(h[ngroups - 1] - h[0]) / (ngroups - 1);
            printf("{\"group\": %u, \"iteration\": %u, \"spread_us\": %.2f, \"spread_iterations\": %.1f}\n", j, j * K,
                   (hi - lo) / 1e3, (hi - lo) / per_group_ns * K);
        }
        return 0;
    }
    run(4, 1, 0, 0);
    for (uint32_t K : {1u, 2u, 4u, 8u, 16u, 32u})
        for (uint32_t D : {1u, 2u, 4u, 8u, 16u, 64u}) {
            if (K * D > 512) continue;
            run(4, 1, K, D);
        }
    run(4, 1, 0, 0);
    run(8, 1, 0, 0);
    for (uint32_t K : {2u, 4u, 8u})
        for (uint32_t D : {2u, 4u, 8u}) run(8, 1, K, D);
    run(4, 2, 0, 0);
    for (uint32_t K : {2u, 4u, 8u})
        for (uint32_t D : {2u, 4u, 8u}) run(4, 2, K, D);
    return 0;
}
