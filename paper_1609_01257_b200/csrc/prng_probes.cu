// prng_probes.cu -- libprng_probes.so (include/prng_probes.h), same-box roofline
// denominators, built apart from libprng_b200.so: the copy-engine
// memset fill, two SM store kernels over pseudo-random (incompressible) data, and the
// pinned / pageable D2H host link (alone, or sustained while other ranks copy too).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <chrono>

#include "../../include/prng_probes.h"

namespace probek {

constexpr int kBlock = 256;  // threads per CTA of the store sweep

inline double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Self-contained helpers: the probes measure the hardware, not the method.
__device__ __forceinline__ void st4(uint64_t *p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
__device__ __forceinline__ uint64_t mix(uint64_t x) {  // splitmix64 finaliser: incompressible data
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

// Persistent grid-stride 32-byte store sweep (every resident thread, full occupancy).
__global__ void __launch_bounds__(256) store_probe_kernel(uint64_t *p, uint64_t n4) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
        const uint64_t x = mix(4 * i + 1);
        st4(p + 4 * i, x, x ^ 1, x ^ 2, x ^ 3);
    }
}

// One-shot fill: CTA b (128 threads) writes the contiguous 16 KiB chunk b with four 32-byte
// stores per thread and exits (the structure of a framework fill kernel).  The hardware
// dispatches the CTAs in order, so the write front advances through memory as one compact
// window; measured the fastest SM write pattern on B200 (profiles/r2_write_ceiling.md).
constexpr uint64_t kFillChunk = 2048;  // u64 per CTA
__global__ void __launch_bounds__(128) fill_probe_kernel(uint64_t *p) {
    const uint64_t base = (uint64_t)blockIdx.x * kFillChunk;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint64_t i = base + k * 512 + threadIdx.x * 4;
        st4(p + i, mix(i + 1), mix(i + 2), mix(i + 3), mix(i + 4));
    }
}

// Time `launch` `reps` times (after one warm-up) with CUDA events; best GB/s of `bytes`.
template <typename F>
double best_gbs(uint64_t bytes, int reps, F launch) {
    cudaEvent_t a, b;
    if (cudaEventCreate(&a) != cudaSuccess) return -1;
    if (cudaEventCreate(&b) != cudaSuccess) {
        cudaEventDestroy(a);
        return -1;
    }
    double best = 0;
    for (int r = 0; r < reps + 1; ++r) {
        cudaEventRecord(a);
        launch(r);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (r) best = std::max(best, bytes / (ms * 1e-3) / 1e9);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return best;
}

}  // namespace probek

extern "C" {

// ---------------------------------------------------------------------------- probes
double prng_probe_memset_gbs(uint64_t bytes, int reps) {
    void *p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return -1;
    const double best = probek::best_gbs(bytes, reps, [&](int r) { cudaMemsetAsync(p, r & 0xff, bytes); });
    cudaFree(p);
    return cudaGetLastError() == cudaSuccess ? best : -1;
}

double prng_probe_memset_sustained_gbs(uint64_t bytes, int reps) {
    void *p = nullptr;
    if (reps < 1 || cudaMalloc(&p, bytes) != cudaSuccess) return -1;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaMemset(p, 1, bytes);
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) cudaMemsetAsync(p, r & 0xff, bytes);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(p);
    return cudaGetLastError() == cudaSuccess ? (double)bytes * reps / (ms * 1e-3) / 1e9 : -1;
}

double prng_probe_store_gbs(uint64_t bytes, int reps) {
    uint64_t *p = nullptr;
    bytes &= ~31ull;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return -1;
    int dev = 0, sms = 0, bps = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, probek::store_probe_kernel, probek::kBlock, 0);
    const double best = probek::best_gbs(bytes, reps, [&](int) {
        probek::store_probe_kernel<<<sms * std::max(bps, 1), probek::kBlock>>>(p, bytes / 32);
    });
    cudaFree(p);
    return cudaGetLastError() == cudaSuccess ? best : -1;
}

double prng_probe_fill_gbs(uint64_t bytes, int reps) {
    uint64_t *p = nullptr;
    const uint64_t chunks = bytes / (probek::kFillChunk * 8);
    if (chunks == 0 || chunks > 0x7FFFFFFFull) return -1;
    bytes = chunks * probek::kFillChunk * 8;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return -1;
    const double best =
        probek::best_gbs(bytes, reps, [&](int) { probek::fill_probe_kernel<<<(unsigned)chunks, 128>>>(p); });
    cudaFree(p);
    return cudaGetLastError() == cudaSuccess ? best : -1;
}

// D2H of `bytes` from device memory into a pinned (or pageable) host buffer, split over
// `nstreams` streams.  sustained = 0: best of `reps` single copies, each timed alone.
// sustained = 1: `reps` copies back to back timed as one interval (for several ranks
// copying at the same time, each rank's share of the shared host links).
static double d2h_probe(uint64_t bytes, int reps, int pinned, int nstreams, int sustained) {
    if (nstreams < 1) nstreams = 1;
    if (reps < 1) reps = 1;
    void *d = nullptr, *hbuf = nullptr;
    if (cudaMalloc(&d, bytes) != cudaSuccess) return -1;
    cudaMemset(d, 7, bytes);
    if (pinned) {
        if (cudaHostAlloc(&hbuf, bytes, cudaHostAllocDefault) != cudaSuccess) {
            cudaFree(d);
            return -1;
        }
    } else {
        hbuf = std::malloc(bytes);
        if (!hbuf) {
            cudaFree(d);
            return -1;
        }
        std::memset(hbuf, 0, bytes);
    }
    std::vector<cudaStream_t> ss(nstreams);
    for (auto &s : ss) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    const uint64_t chunk = (bytes / nstreams) & ~4095ull;
    auto copy_once = [&]() {
        for (int i = 0; i < nstreams; ++i) {
            const uint64_t off = i * chunk, len = (i == nstreams - 1) ? bytes - off : chunk;
            cudaMemcpyAsync((char *)hbuf + off, (char *)d + off, len, cudaMemcpyDeviceToHost, ss[i]);
        }
    };
    double best = 0;
    cudaDeviceSynchronize();
    if (sustained) {
        copy_once();  // warm-up
        for (auto &s : ss) cudaStreamSynchronize(s);
        const double t0 = probek::now_s();
        for (int r = 0; r < reps; ++r) copy_once();
        for (auto &s : ss) cudaStreamSynchronize(s);
        best = (double)bytes * reps / (probek::now_s() - t0) / 1e9;
    } else {
        for (int r = 0; r < reps + 1; ++r) {
            cudaDeviceSynchronize();
            const double t0 = probek::now_s();
            copy_once();
            for (auto &s : ss) cudaStreamSynchronize(s);
            const double dt = probek::now_s() - t0;
            if (r) best = std::max(best, bytes / dt / 1e9);
        }
    }
    for (auto &s : ss) cudaStreamDestroy(s);
    if (pinned)
        cudaFreeHost(hbuf);
    else
        std::free(hbuf);
    cudaFree(d);
    return cudaGetLastError() == cudaSuccess ? best : -1;
}

double prng_probe_d2h_gbs(uint64_t bytes, int reps, int pinned, int nstreams) {
    return d2h_probe(bytes, reps, pinned, nstreams, 0);
}

double prng_probe_d2h_sustained_gbs(uint64_t bytes, int reps) { return d2h_probe(bytes, reps, 1, 1, 1); }

}  // extern "C"
