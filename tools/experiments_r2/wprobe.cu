// Round-2 research probe (not product code): HBM write ceilings on B200 for
// compressible vs incompressible data, in the access pattern of torch's fill kernel
// (one-shot grid, 128-thread CTAs, each CTA one contiguous 16 KiB chunk) and of a
// persistent grid-stride sweep.  Question: is the 7.4 TB/s memset / fill "ceiling" a
// property of the write path, or of data compression?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o wprobe wprobe.cu
//   ./wprobe <GiB> <reps>
#include <cuda_runtime.h>
#include <cuda_profiler_api.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}
__device__ __forceinline__ uint64_t val(int pattern, uint64_t i) {
    switch (pattern) {
        case 0: return 0;                 // constant zero
        case 1: return 7;                 // constant
        case 2: return i;                 // index
        default: return mix(i + 1);       // pseudo-random (incompressible)
    }
}
__device__ __forceinline__ void st4(uint64_t *p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
__device__ __forceinline__ void st2(uint64_t *p, uint64_t a, uint64_t b) {
    asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

// torch-fill-like: one-shot grid, CTA b writes elements [b*E, (b+1)*E) (E = 2048 u64 =
// 16 KiB), thread t writes 16-B vectors at t*2 + k*256 for k = 0..7.
__global__ void __launch_bounds__(128) oneshot16(uint64_t *p, int pattern) {
    const uint64_t base = (uint64_t)blockIdx.x * 2048;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint64_t i = base + k * 256 + threadIdx.x * 2;
        st2(p + i, val(pattern, i), val(pattern, i + 1));
    }
}
// the same with 32-B vectors (4 per thread)
__global__ void __launch_bounds__(128) oneshot32(uint64_t *p, int pattern) {
    const uint64_t base = (uint64_t)blockIdx.x * 2048;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint64_t i = base + k * 512 + threadIdx.x * 4;
        st4(p + i, val(pattern, i), val(pattern, i + 1), val(pattern, i + 2), val(pattern, i + 3));
    }
}
// persistent grid-stride 32-B sweep
__global__ void __launch_bounds__(256) sweep32(uint64_t *p, uint64_t n4, int pattern) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n4; j += stride) {
        const uint64_t i = 4 * j;
        st4(p + i, val(pattern, i), val(pattern, i + 1), val(pattern, i + 2), val(pattern, i + 3));
    }
}

int main(int argc, char **argv) {
    const uint64_t gib = argc > 1 ? strtoull(argv[1], 0, 10) : 32;
    const int reps = argc > 2 ? atoi(argv[2]) : 3;
    const uint64_t bytes = gib << 30, n = bytes / 8;
    uint64_t *p;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return 1;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char *pn[] = {"zero", "seven", "index", "random"};
    auto run = [&](const char *name, int pattern, auto launch) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < reps; ++r) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("{\"kernel\": \"%s\", \"pattern\": \"%s\", \"gib\": %llu, \"gbs\": %.1f}\n", name, pn[pattern],
               (unsigned long long)gib, bytes / (best * 1e-3) / 1e9);
        fflush(stdout);
    };
    for (int pat = 0; pat < 4; ++pat) {
        if (pat < 2) run("memset", pat, [&] { cudaMemsetAsync(p, pat == 1 ? 7 : 0, bytes); });
        run("oneshot16", pat, [&] { oneshot16<<<(unsigned)(n / 2048), 128>>>(p, pat); });
        run("oneshot32", pat, [&] { oneshot32<<<(unsigned)(n / 2048), 128>>>(p, pat); });
        run("sweep32", pat, [&] { sweep32<<<sms * 8, 256>>>(p, n / 4, pat); });
    }
    // one profiled range per memset pattern (ncu --replay-mode app-range)
    if (argc > 3) {
        for (int pat = 0; pat < 2; ++pat) {
            cudaProfilerStart();
            cudaMemsetAsync(p, pat == 1 ? 7 : 0, bytes);
            cudaDeviceSynchronize();
            cudaProfilerStop();
        }
    }
    cudaFree(p);
    return 0;
}
