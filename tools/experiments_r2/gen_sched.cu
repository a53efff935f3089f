// Round-2 research probe (not product code): which write schedule lets SM stores reach the
// 91 % DRAM-active of a one-shot fill kernel (wprobe.cu) with the generator's output?
//
//   fill patterns (random data, 32-B stores): a one-shot grid of CTAs, CTA b writes one
//   contiguous chunk; chunk position = b (sequential) or a scrambled permutation of b.
//   generator schedules (real xorshift64 streams, out[k][g], pitch n, no ring wrap):
//     G1 persistent: one CTA of 4 warps per SM, a warp owns 256 gids (NPT 8, VEC 4) for all
//        T iterations, CTA barrier every iteration (the round-1 bench kernel's structure);
//     G2 L-tiled one-shot: one launch per block of L iterations; a CTA of W warps owns
//        W*256 gids for those L iterations (state read + written once per launch).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -o gen_sched gen_sched.cu
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

// ---- fill: CTA b writes chunk perm(b) of `chunk` u64 (chunk multiple of 4 * blockDim)
__global__ void fill_chunks(uint64_t *p, uint64_t chunk, uint64_t nchunks, int perm) {
    uint64_t c = blockIdx.x;
    if (perm == 1) c = (c * 2654435761ull) % nchunks;  // scattered (nchunks odd-prime-coprime)
    uint64_t *q = p + c * chunk;
    for (uint64_t i = 4 * threadIdx.x; i < chunk; i += 4 * blockDim.x) {
        const uint64_t x = mix(c * chunk + i + 1);
        st4(q + i, x, x ^ 1, x ^ 2, x ^ 3);
    }
}

// ---- F3: persistent fill: the grid loops over the chunks (grid-stride over chunk index)
__global__ void fill_persistent(uint64_t *p, uint64_t chunk, uint64_t nchunks, int perm) {
    for (uint64_t b = blockIdx.x; b < nchunks; b += gridDim.x) {
        uint64_t c = b;
        if (perm == 1) c = (c * 2654435761ull) % nchunks;
        uint64_t *q = p + c * chunk;
        for (uint64_t i = 4 * threadIdx.x; i < chunk; i += 4 * blockDim.x) {
            const uint64_t x = mix(c * chunk + i + 1);
            st4(q + i, x, x ^ 1, x ^ 2, x ^ 3);
        }
    }
}

// ---- F4: fill where each CTA writes `per` consecutive-in-b chunks (chunk index b*per + i,
// scattered by perm), with `sync` after each chunk: 0 none, 1 __syncthreads, 2 __threadfence
// (membar.gl: the warp waits until its stores are performed), 3 fence + __syncthreads.
__global__ void fill_multi(uint64_t *p, uint64_t chunk, uint64_t nchunks, int perm, int per, int sync) {
    for (int i = 0; i < per; ++i) {
        uint64_t c = (uint64_t)blockIdx.x * per + i;
        if (c >= nchunks) return;
        if (perm == 1) c = (c * 2654435761ull) % nchunks;
        uint64_t *q = p + c * chunk;
        for (uint64_t j = 4 * threadIdx.x; j < chunk; j += 4 * blockDim.x) {
            const uint64_t x = mix(c * chunk + j + 1);
            st4(q + j, x, x ^ 1, x ^ 2, x ^ 3);
        }
        if (sync & 2) __threadfence();
        if (sync & 1) __syncthreads();
    }
}
__global__ void fill_persistent_sync(uint64_t *p, uint64_t chunk, uint64_t nchunks, int sync) {
    for (uint64_t b = blockIdx.x; b < nchunks; b += gridDim.x) {
        uint64_t *q = p + b * chunk;
        for (uint64_t i = 4 * threadIdx.x; i < chunk; i += 4 * blockDim.x) {
            const uint64_t x = mix(b * chunk + i + 1);
            st4(q + i, x, x ^ 1, x ^ 2, x ^ 3);
        }
        if (sync & 2) __threadfence();
        if (sync & 1) __syncthreads();
    }
}

// ---- G1: persistent, one CTA per SM of W warps, barrier each iteration
template <int NPT>
__global__ void __launch_bounds__(256) g1_persistent(uint64_t *out, uint64_t *state, uint64_t n, uint32_t T, int pace = 0) {
    uint64_t dummy = threadIdx.x + 1;
    constexpr int NV = NPT / 4;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t wpb = blockDim.x >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * wpb;
    const uint64_t npieces = n / (32 * NPT);
    for (uint64_t piece = blockIdx.x * wpb + (threadIdx.x >> 5); piece < npieces; piece += nwarps) {
        const uint64_t base = piece * 32 * NPT + lane * 4;
        uint64_t x[NPT];
#pragma unroll
        for (int v = 0; v < NV; ++v) ld4(state + base + v * 128, x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
        uint64_t *p = out + base;
        for (uint32_t t = 0; t < T; ++t) {
#pragma unroll
            for (int j = 0; j < NPT; ++j) x[j] = xs(x[j]);
#pragma unroll
            for (int v = 0; v < NV; ++v) st4(p + v * 128, x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
            for (int q = 0; q < pace; ++q) dummy = xs(dummy);
            bar(blockDim.x);
            p += n;
        }
#pragma unroll
        for (int v = 0; v < NV; ++v) st4(state + base + v * 128, x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
    }
    if (dummy == 42) state[0] = dummy;
}

// ---- G2: one-shot tile launch: CTA b owns gids [b*W*32*NPT, ...) for iterations [k0, k0+L)
template <int NPT, bool BAR>
__global__ void __launch_bounds__(256) g2_tile(uint64_t *out, uint64_t *state, uint64_t n, uint32_t k0, uint32_t L, int pace = 0) {
    uint64_t dummy = threadIdx.x + 1;
    constexpr int NV = NPT / 4;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t piece = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint64_t base = piece * 32 * NPT + lane * 4;
    uint64_t x[NPT];
#pragma unroll
    for (int v = 0; v < NV; ++v) ld4(state + base + v * 128, x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
    uint64_t *p = out + (uint64_t)k0 * n + base;
    for (uint32_t t = 0; t < L; ++t) {
#pragma unroll
        for (int j = 0; j < NPT; ++j) x[j] = xs(x[j]);
#pragma unroll
        for (int v = 0; v < NV; ++v) st4(p + v * 128, x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
        for (int q = 0; q < pace; ++q) dummy = xs(dummy);
        if (BAR) bar(blockDim.x);
        p += n;
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) st4(state + base + v * 128, x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
    if (dummy == 42) state[0] = dummy;
}

// ---- G3: gid-blocked layout: CTA block b (W warps x 32 x NPT gids = `chunk` u64) writes
// iteration t of its gids at out + b*T*chunk + t*chunk (each CTA one sequential stream).
// Grid-stride over blocks (persistent if gridDim < nblocks, one-shot otherwise).
template <int NPT>
__global__ void __launch_bounds__(256) g3_blocked(uint64_t *out, uint64_t *state, uint64_t n, uint32_t T) {
    constexpr int NV = NPT / 4;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t chunk = (uint64_t)blockDim.x * NPT;
    const uint64_t nblk = n / chunk;
    for (uint64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const uint64_t wbase = (threadIdx.x >> 5) * 32 * NPT + lane * 4;  // within the block
        uint64_t x[NPT];
#pragma unroll
        for (int v = 0; v < NV; ++v)
            ld4(state + blk * chunk + wbase + v * 128, x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
        uint64_t *p = out + blk * T * chunk + wbase;
        for (uint32_t t = 0; t < T; ++t) {
#pragma unroll
            for (int j = 0; j < NPT; ++j) x[j] = xs(x[j]);
#pragma unroll
            for (int v = 0; v < NV; ++v) st4(p + v * 128, x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
            p += chunk;
        }
#pragma unroll
        for (int v = 0; v < NV; ++v)
            st4(state + blk * chunk + wbase + v * 128, x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
    }
}

__global__ void init_state(uint64_t *s, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        s[i] = mix(i + 1) | 1;
}

int main(int argc, char **argv) {
    const uint64_t n = argc > 1 ? strtoull(argv[1], 0, 10) : (1ull << 24);
    const uint32_t T = argc > 2 ? atoi(argv[2]) : 256;
    const char *only = argc > 3 ? argv[3] : "";
    const uint64_t out_elems = n * T;
    uint64_t *out, *state;
    if (cudaMalloc(&out, out_elems * 8) != cudaSuccess || cudaMalloc(&state, n * 8) != cudaSuccess) return 1;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    init_state<<<sms * 4, 256>>>(state, n);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char *name, const char *params, auto launch) {
        if (*only && !strstr(name, only)) return;
        launch();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        cudaError_t e = cudaGetLastError();
        printf("{\"sched\": \"%s\", %s, \"n\": %llu, \"T\": %u, \"gbs\": %.1f, \"err\": \"%s\"}\n", name, params,
               (unsigned long long)n, T, out_elems * 8.0 / (best * 1e-3) / 1e9, cudaGetErrorString(e));
        fflush(stdout);
    };
    char prm[256];
    // G3 blocked layout
    for (int W : {1, 4, 8}) {
        const uint64_t nblk = n / (W * 32 * 8);
        for (int cps : {1, 2, 4, 16, 0}) {  // 0: one-shot (grid = nblk)
            const unsigned grid = cps ? sms * cps : (unsigned)nblk;
            snprintf(prm, sizeof prm, "\"npt\": 8, \"warps_per_cta\": %d, \"ctas_per_sm\": %d", W, cps);
            run("g3_blocked", prm, [&] { g3_blocked<8><<<grid, 32 * W>>>(out, state, n, T); });
        }
    }
    // G1 persistent reference
    snprintf(prm, sizeof prm, "\"npt\": 8, \"warps_per_cta\": 4, \"ctas_per_sm\": 1, \"pace\": 0");
    run("g1_persistent", prm, [&] { g1_persistent<8><<<sms, 128>>>(out, state, n, T, 0); });
    return 0;
}
