// prng_probes.cu -- same-box roofline denominators and research probes:
// memset fill, plain store kernels, copy-engine D2D sweep, pinned / pageable D2H.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "engine_internal.h"

using namespace prng_detail;

namespace probek {

// Self-contained store helpers (the probes measure the hardware, not the method).
__device__ __forceinline__ void st2(uint64_t *p, uint64_t a, uint64_t b) {
    asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void st4(uint64_t *p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
__device__ __forceinline__ uint64_t mix(uint64_t x) {  // any cheap bit mixer will do for data
    x ^= x << 13;
    x ^= x >> 7;
    x ^= x << 17;
    return x;
}

// ---------------------------------------------------------------- roofline probe kernel
// Pure 32-byte grid-stride store stream: the same-box SM write ceiling.  pattern 0: the
// index (i, i+1, ...), 1: zeros, 2: pseudo-random (xorshift64 of the index) -- to see
// whether the data values change the write rate (e.g. compression of constant data).
__global__ void __launch_bounds__(256) store_probe_kernel(uint64_t *p, uint64_t n4, int pattern) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
        if (pattern == 1) {
            st4(p + 4 * i, 0, 0, 0, 0);
        } else if (pattern == 2) {
            const uint64_t x = mix(i * 0x9E3779B97F4A7C15ull + 1);
            st4(p + 4 * i, x, x ^ 0xA5A5A5A5A5A5A5A5ull, x * 3, ~x);
        } else {
            st4(p + 4 * i, i, i + 1, i + 2, i + 3);
        }
    }
}


// Store-pattern microbenchmark (research probe, not on the path): 16-byte stores.
//   mode 0: grid-stride sweep (consecutive warps adjacent, the grid sweeps forward)
//   mode 1: mode 0 + a CTA barrier after every warp-store round
//   mode 2: blocked -- CTA b sweeps its own contiguous 1/gridDim of the buffer
//   mode 3: mode 2 + a CTA barrier after every round
//   mode 4: "slot-strided" like the generator: the buffer is `slots` rows; each round a
//           CTA writes its 4 KiB-ish chunk in row r mod slots, advancing one row per round
__global__ void __launch_bounds__(256) store_pattern_kernel(uint64_t *p, uint64_t n2, int mode, uint64_t slots) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    if (mode <= 1) {
        for (uint64_t i = tid; i < n2; i += nthreads) {
            st2(p + 2 * i, i, ~i);
            if (mode == 1) __syncthreads();
        }
    } else if (mode >= 100) {
        // mode 100 + k: grid-stride with k dependent xorshift steps between stores (pacing)
        uint64_t x = tid + 1;
        for (uint64_t i = tid; i < n2; i += nthreads) {
            for (int j = 0; j < mode - 100; ++j) x = mix(x);
            st2(p + 2 * i, i, x);
        }
    } else if (mode <= 3) {
        const uint64_t per = (n2 + gridDim.x - 1) / gridDim.x;
        const uint64_t b0 = blockIdx.x * per, b1 = b0 + per < n2 ? b0 + per : n2;
        for (uint64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
            st2(p + 2 * i, i, ~i);
            if (mode == 3) __syncthreads();
        }
    } else {
        // row-major [slots][cols]: CTA b owns columns [b*blockDim, (b+1)*blockDim) of a
        // "piece" and walks rows; pieces advance after `slots` rows (like the generator).
        const uint64_t cols = n2 / slots;  // vec2 elements per row
        const uint64_t piece_w = blockDim.x;
        const uint64_t npieces = cols / (piece_w * gridDim.x);
        for (uint64_t pc = 0; pc < npieces; ++pc) {
            const uint64_t col = (pc * gridDim.x + blockIdx.x) * piece_w + threadIdx.x;
            for (uint64_t r = 0; r < slots; ++r) {
                st2(p + 2 * (r * cols + col), r, col);
                __syncthreads();
            }
        }
    }
}

}  // namespace probek

extern "C" {

// ---------------------------------------------------------------------------- probes
double prng_probe_memset_gbs(uint64_t bytes, int reps) {
    void *p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return -1;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double best = 0;
    cudaMemset(p, 1, bytes);
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a);
        cudaMemsetAsync(p, r & 0xff, bytes);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        best = std::max(best, bytes / (ms * 1e-3) / 1e9);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
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

double prng_probe_store_gbs(uint64_t bytes, int reps) { return prng_probe_store_pattern_gbs(bytes, reps, 0, 0); }

double prng_probe_store_pattern_gbs(uint64_t bytes, int reps, int pattern, int warps_per_sm) {
    uint64_t *p = nullptr;
    bytes &= ~31ull;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return -1;
    int dev = 0, sms = 0, bps = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, probek::store_probe_kernel, kBlock, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double best = 0;
    for (int r = 0; r < reps + 1; ++r) {
        cudaEventRecord(a);
        if (warps_per_sm > 0)
            probek::store_probe_kernel<<<sms, 32 * std::min(warps_per_sm, 32), 0>>>(p, bytes / 32, pattern);
        else
            probek::store_probe_kernel<<<sms * std::max(bps, 1), kBlock>>>(p, bytes / 32, pattern);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (r) best = std::max(best, bytes / (ms * 1e-3) / 1e9);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(p);
    return cudaGetLastError() == cudaSuccess ? best : -1;
}

// Copy-engine write probe: a `chunk`-byte (L2-resident) source copied D2D over a `total`-byte
// destination, chunk by chunk (cudaMemcpyAsync), i.e. the DRAM sees a sequential write
// sweep fed from L2.  Returns destination GB/s (best of reps).
double prng_probe_d2d_sweep_gbs(uint64_t chunk, uint64_t total, int reps) {
    void *src = nullptr, *dst = nullptr;
    if (cudaMalloc(&src, chunk) != cudaSuccess) return -1;
    if (cudaMalloc(&dst, total) != cudaSuccess) {
        cudaFree(src);
        return -1;
    }
    cudaMemset(src, 3, chunk);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double best = 0;
    for (int r = 0; r < reps + 1; ++r) {
        cudaEventRecord(a);
        for (uint64_t off = 0; off + chunk <= total; off += chunk)
            cudaMemcpyAsync((char *)dst + off, src, chunk, cudaMemcpyDeviceToDevice);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (r) best = std::max(best, (total / chunk) * (double)chunk / (ms * 1e-3) / 1e9);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(src);
    cudaFree(dst);
    return cudaGetLastError() == cudaSuccess ? best : -1;
}

double prng_probe_store_mode_gbs(uint64_t bytes, int reps, int mode, int warps_per_cta, int ctas_per_sm,
                                 uint64_t slots) {
    uint64_t *p = nullptr;
    bytes &= ~15ull;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return -1;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double best = 0;
    uint64_t done = bytes;
    for (int r = 0; r < reps + 1; ++r) {
        cudaEventRecord(a);
        probek::store_pattern_kernel<<<sms * ctas_per_sm, 32 * warps_per_cta>>>(p, bytes / 16, mode,
                                                                                 slots ? slots : 1);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (mode == 4) {  // bytes actually written: whole pieces only
            const uint64_t cols = bytes / 16 / (slots ? slots : 1);
            const uint64_t pw = 32ull * warps_per_cta * sms * ctas_per_sm;
            done = (cols / pw) * pw * (slots ? slots : 1) * 16;
        }
        if (r) best = std::max(best, done / (ms * 1e-3) / 1e9);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(p);
    return cudaGetLastError() == cudaSuccess ? best : -1;
}

// Research probe: do the SM store path and the copy engine add up?  An SM store kernel
// (grid-stride, `sm_warps` warps per SM) over `sm_bytes` on one stream while the copy
// engine sweeps `ce_bytes` from an L2-resident `ce_chunk` source on another; returns the
// combined destination GB/s (best of reps) and, via the out pointers, each side alone.
double prng_probe_concurrent_gbs(uint64_t sm_bytes, uint64_t ce_bytes, uint64_t ce_chunk, int sm_warps, int reps,
                                 double *sm_alone, double *ce_alone) {
    uint64_t *a = nullptr, *src = nullptr, *b = nullptr;
    if (cudaMalloc(&a, sm_bytes) != cudaSuccess) return -1;
    if (cudaMalloc(&b, ce_bytes) != cudaSuccess || cudaMalloc(&src, ce_chunk) != cudaSuccess) {
        cudaFree(a);
        if (b) cudaFree(b);
        return -1;
    }
    cudaMemset(src, 5, ce_chunk);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t e0, e1, e2;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventCreate(&e2);
    auto sm_launch = [&](cudaStream_t s) {
        probek::store_probe_kernel<<<sms, 32 * sm_warps, 0, s>>>(a, sm_bytes / 32, 0);
    };
    auto ce_launch = [&](cudaStream_t s) {
        for (uint64_t off = 0; off + ce_chunk <= ce_bytes; off += ce_chunk)
            cudaMemcpyAsync((char *)b + off, src, ce_chunk, cudaMemcpyDeviceToDevice, s);
    };
    const uint64_t ce_done = (ce_bytes / ce_chunk) * ce_chunk;
    double best = 0, best_sm = 0, best_ce = 0;
    for (int r = 0; r < reps + 1; ++r) {
        float ms = 0;
        // SM alone
        cudaEventRecord(e0, s1);
        sm_launch(s1);
        cudaEventRecord(e1, s1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (r) best_sm = std::max(best_sm, sm_bytes / (ms * 1e-3) / 1e9);
        // CE alone
        cudaEventRecord(e0, s2);
        ce_launch(s2);
        cudaEventRecord(e1, s2);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (r) best_ce = std::max(best_ce, ce_done / (ms * 1e-3) / 1e9);
        // both at once: both streams start after e0, the region ends when both are done
        cudaDeviceSynchronize();
        cudaEventRecord(e0, s1);
        cudaStreamWaitEvent(s2, e0, 0);
        sm_launch(s1);
        ce_launch(s2);
        cudaEventRecord(e1, s1);
        cudaEventRecord(e2, s2);
        cudaEventSynchronize(e1);
        cudaEventSynchronize(e2);
        float m1 = 0, m2 = 0;
        cudaEventElapsedTime(&m1, e0, e1);
        cudaEventElapsedTime(&m2, e0, e2);
        if (r) best = std::max(best, (sm_bytes + ce_done) / (std::max(m1, m2) * 1e-3) / 1e9);
    }
    if (sm_alone) *sm_alone = best_sm;
    if (ce_alone) *ce_alone = best_ce;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    cudaStreamDestroy(s1);
    cudaStreamDestroy(s2);
    cudaFree(a);
    cudaFree(b);
    cudaFree(src);
    return cudaGetLastError() == cudaSuccess ? best : -1;
}

double prng_probe_d2h_gbs(uint64_t bytes, int reps, int pinned, int nstreams) {
    if (nstreams < 1) nstreams = 1;
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
    double best = 0;
    const uint64_t chunk = (bytes / nstreams) & ~4095ull;
    for (int r = 0; r < reps + 1; ++r) {
        cudaDeviceSynchronize();
        const double t0 = now_s();
        for (int i = 0; i < nstreams; ++i) {
            const uint64_t off = i * chunk, len = (i == nstreams - 1) ? bytes - off : chunk;
            cudaMemcpyAsync((char *)hbuf + off, (char *)d + off, len, cudaMemcpyDeviceToHost, ss[i]);
        }
        for (auto &s : ss) cudaStreamSynchronize(s);
        const double dt = now_s() - t0;
        if (r) best = std::max(best, bytes / dt / 1e9);
    }
    for (auto &s : ss) cudaStreamDestroy(s);
    if (pinned)
        cudaFreeHost(hbuf);
    else
        std::free(hbuf);
    cudaFree(d);
    return cudaGetLastError() == cudaSuccess ? best : -1;
}

}  // extern "C"
