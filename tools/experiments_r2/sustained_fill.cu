// Round-2 research probe: sustained (seconds-long, power-capped) write rates of the
// copy-engine memset and the one-shot SM fill kernel, timed as one interval each, with the
// SM clock read by NVML-free means (clock64 / globaltimer ratio in a tiny kernel after).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o sustained_fill sustained_fill.cu
#include <cuda_runtime.h>

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
__device__ __forceinline__ void st4(uint64_t *p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
__global__ void __launch_bounds__(128) oneshot32(uint64_t *p, uint64_t salt) {
    const uint64_t base = (uint64_t)blockIdx.x * 2048;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint64_t i = base + k * 512 + threadIdx.x * 4;
        st4(p + i, mix(i + salt), mix(i + 1 + salt), mix(i + 2 + salt), mix(i + 3 + salt));
    }
}

int main(int argc, char **argv) {
    const uint64_t gib = argc > 1 ? strtoull(argv[1], 0, 10) : 32;
    const int reps = argc > 2 ? atoi(argv[2]) : 100;
    const uint64_t bytes = gib << 30, n = bytes / 8;
    uint64_t *p;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return 1;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int round = 0; round < 2; ++round) {
        for (int which = 0; which < 2; ++which) {
            cudaDeviceSynchronize();
            cudaEventRecord(a);
            for (int r = 0; r < reps; ++r) {
                if (which == 0)
                    cudaMemsetAsync(p, r & 0xff, bytes);
                else
                    oneshot32<<<(unsigned)(n / 2048), 128>>>(p, (uint64_t)r << 40);
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("{\"round\": %d, \"what\": \"%s\", \"seconds\": %.2f, \"gbs\": %.1f}\n", round,
                   which ? "oneshot_fill_kernel" : "memset", ms * 1e-3, bytes * (double)reps / (ms * 1e-3) / 1e9);
            fflush(stdout);
        }
    }
    return 0;
}
