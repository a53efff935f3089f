// Round-2 research probe (not product code): the generator's 2-D write pattern without the
// arithmetic.  The output is R rows (iterations) of `pitch` bytes; CTA b owns a column
// block of `wc` bytes (grid-strided over blocks) and writes it row after row (iteration
// after iteration), like a warp group holding its states for all iterations.  Questions:
// does the contiguous width per CTA-row (8 KiB .. 512 KiB) matter?  does inter-CTA drift
// (removed by a grid barrier every row) matter?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -rdc=true -o colblock colblock.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <initializer_list>
namespace cg = cooperative_groups;

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

// wc, pitch in u64; rows R; sync: 0 none, 1 __syncthreads per row, 2 grid sync per row
__global__ void colblock(uint64_t *p, uint64_t pitch, uint32_t R, uint64_t wc, int sync) {
    const uint64_t nblk = pitch / wc;
    uint64_t x = mix(blockIdx.x * 1024 + threadIdx.x + 1);
    for (uint64_t b = blockIdx.x; b < nblk + (sync == 2 ? (gridDim.x - nblk % gridDim.x) % gridDim.x : 0);
         b += gridDim.x) {
        for (uint32_t r = 0; r < R; ++r) {
            if (b < nblk) {
                uint64_t *q = p + r * pitch + b * wc;
                for (uint64_t j = 4 * threadIdx.x; j < wc; j += 4 * blockDim.x) {
                    x = x * 0x9E3779B97F4A7C15ull + 1;
                    st4(q + j, x, x ^ 1, x ^ 2, x ^ 3);
                }
            }
            if (sync == 1) __syncthreads();
            if (sync == 2) cg::this_grid().sync();
        }
    }
}

int main(int argc, char **argv) {
    const uint64_t pitch = (argc > 1 ? strtoull(argv[1], 0, 10) : (1ull << 24));  // u64 per row
    const uint32_t R = argc > 2 ? atoi(argv[2]) : 256;
    const uint64_t elems = pitch * R;
    uint64_t *p;
    if (cudaMalloc(&p, elems * 8) != cudaSuccess) return 1;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (uint64_t wcb : {8192ull, 32768ull, 131072ull, 524288ull}) {
        for (int thr : {128, 256}) {
            for (int cps : {1, 2}) {
                for (int sync : {0, 1, 2}) {
                    const uint64_t wc = wcb / 8;
                    const unsigned grid = sms * cps;
                    auto launch = [&] {
                        if (sync == 2) {
                            uint64_t pp = pitch, ww = wc;
                            uint32_t rr = R;
                            int ss = sync;
                            void *args[] = {&p, &pp, &rr, &ww, &ss};
                            cudaLaunchCooperativeKernel((void *)colblock, grid, thr, args);
                        } else {
                            colblock<<<grid, thr>>>(p, pitch, R, wc, sync);
                        }
                    };
                    launch();
                    cudaDeviceSynchronize();
                    float best = 1e30f;
                    for (int r = 0; r < 2; ++r) {
                        cudaEventRecord(a);
                        launch();
                        cudaEventRecord(b);
                        cudaEventSynchronize(b);
                        float ms;
                        cudaEventElapsedTime(&ms, a, b);
                        if (ms < best) best = ms;
                    }
                    printf("{\"wc_bytes\": %llu, \"threads\": %d, \"ctas_per_sm\": %d, \"sync\": %d, \"gbs\": %.1f, \"err\": \"%s\"}\n",
                           (unsigned long long)wcb, thr, cps, sync, elems * 8.0 / (best * 1e-3) / 1e9,
                           cudaGetErrorString(cudaGetLastError()));
                    fflush(stdout);
                }
            }
        }
    }
    return 0;
}
