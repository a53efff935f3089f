// die_probe.cu -- research probe (session 2): does die locality matter for SM write streams
// on B200 (two dies joined by NV-HBI, HBM interleaved over both)?
//
// Part 1 (latency map): every CTA (one thread, records %smid) times an L2-hit load of each
// 4 KiB chunk of a 64 MiB buffer (the buffer is touched first, so all chunks are in L2;
// the timed load's latency depends on which die's L2 slice holds the line).
// Output: lat[cta][chunk] cycles + smid[cta].  The analysis (die_probe.py) splits SMs and
// chunks into two groups if the latencies are bimodal.
//
// Part 2 (write bandwidth by locality): given a chunk -> group map (from part 1, applied
// modulo the map period), each SM writes only chunks of its own group, only chunks of the
// other group, or all chunks, over a 16 GiB buffer; GB/s with CUDA events.
//
// Build + run (GPU box):  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/die_probe
//                         tools/experiments_r1/die_probe.cu && /tmp/die_probe lat > lat.csv
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess) {                                                   \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));               \
            exit(1);                                                               \
        }                                                                          \
    } while (0)

__device__ __forceinline__ uint32_t smid() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

constexpr int kChunk = 4096;

__global__ void lat_kernel(const uint64_t *buf, int nchunks, uint32_t *lat, uint32_t *sm) {
    if (threadIdx.x) return;
    sm[blockIdx.x] = smid();
    uint64_t acc = 0;
    // touch everything once (brings the lines into L2)
    for (int c = 0; c < nchunks; ++c) {
        uint64_t v;
        asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(buf + (size_t)c * kChunk / 8));
        acc += v;
    }
    for (int c = 0; c < nchunks; ++c) {
        const uint64_t *p = buf + (size_t)c * kChunk / 8 + (acc & 1);  // dependent address
        long long t0 = clock64();
        uint64_t v;
        asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
        acc += v;
        long long t1 = clock64();
        // force completion before t1 is taken: t1 depends on nothing, so fold v into it
        lat[(size_t)blockIdx.x * nchunks + c] = (uint32_t)(t1 - t0) + (uint32_t)(acc == 0x5555);
    }
}

// mode 0: all chunks; 1: only chunks whose group == the SM's group; 2: only the other group.
__global__ void __launch_bounds__(128) write_kernel(uint64_t *buf, size_t nchunks, const uint8_t *chunk_group,
                                                    int period, const uint8_t *sm_group, int mode, int reps,
                                                    unsigned long long *bytes) {
    const uint32_t g = sm_group[smid()];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // each CTA walks chunks c = blockIdx.x, + gridDim.x, ...; a warp writes 1 KiB of it
    for (int r = 0; r < reps; ++r)
        for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
            const uint32_t cg = chunk_group[c % period];
            if (mode == 1 && cg != g) continue;
            if (mode == 2 && cg == g) continue;
            if (threadIdx.x == 0) atomicAdd(bytes, (unsigned long long)kChunk);
            uint64_t *p = buf + c * (kChunk / 8) + warp * 128 + lane * 4;
            asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(c), "l"(c + 1), "l"(c + 2),
                         "l"((uint64_t)r)
                         : "memory");
        }
}

int main(int argc, char **argv) {
    const char *what = argc > 1 ? argv[1] : "lat";
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    if (!strcmp(what, "lat")) {
        const int nchunks = 16384;  // 64 MiB: fits in L2, so the timed loads are L2 hits
        uint64_t *buf;
        CK(cudaMalloc(&buf, (size_t)nchunks * kChunk));
        CK(cudaMemset(buf, 0, (size_t)nchunks * kChunk));
        const int nblk = nsm;  // one single-thread CTA per SM (occupancy spreads them)
        uint32_t *lat, *sm;
        CK(cudaMalloc(&lat, (size_t)nblk * nchunks * 4));
        CK(cudaMalloc(&sm, nblk * 4));
        lat_kernel<<<nblk, 32>>>(buf, nchunks, lat, sm);
        CK(cudaDeviceSynchronize());
        std::vector<uint32_t> hl((size_t)nblk * nchunks), hs(nblk);
        CK(cudaMemcpy(hl.data(), lat, hl.size() * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(hs.data(), sm, hs.size() * 4, cudaMemcpyDeviceToHost));
        // reference CTA: the one on the lowest smid; its latency histogram and split
        int ref = 0;
        for (int b2 = 1; b2 < nblk; ++b2)
            if (hs[b2] < hs[ref]) ref = b2;
        std::vector<uint32_t> r(hl.begin() + (size_t)ref * nchunks, hl.begin() + (size_t)(ref + 1) * nchunks);
        std::vector<uint32_t> srt = r;
        std::sort(srt.begin(), srt.end());
        printf("ref smid %u latency percentiles (cycles): p1 %u p10 %u p25 %u p50 %u p75 %u p90 %u p99 %u\n", hs[ref],
               srt[nchunks / 100], srt[nchunks / 10], srt[nchunks / 4], srt[nchunks / 2], srt[3 * nchunks / 4],
               srt[9 * nchunks / 10], srt[99 * nchunks / 100]);
        // histogram in 20-cycle bins
        std::vector<int> hist(200, 0);
        for (uint32_t v : r) hist[std::min<uint32_t>(v / 20, 199)]++;
        printf("histogram (20-cycle bins, count>0):");
        for (int i = 0; i < 200; ++i)
            if (hist[i]) printf(" %d:%d", i * 20, hist[i]);
        printf("\n");
        // split at the largest gap between the two most populated regions: use the median
        // of the sorted latencies between p10 and p90 as the threshold
        const uint32_t thr = (srt[nchunks / 10] + srt[9 * nchunks / 10]) / 2;
        std::vector<uint8_t> cls(nchunks);
        int n0 = 0;
        for (int c = 0; c < nchunks; ++c) n0 += (cls[c] = r[c] <= thr ? 0 : 1) == 0;
        printf("threshold %u: %d chunks near (class 0), %d far (class 1)\n", thr, n0, nchunks - n0);
        // period of the class pattern (powers of two)
        for (int per = 1; per <= nchunks / 2; per *= 2) {
            int mism = 0;
            for (int c = per; c < nchunks; ++c) mism += cls[c] != cls[c % per];
            if (mism * 100 < nchunks) {
                printf("class pattern repeats with period %d chunks (%d KiB), %d mismatches\n", per, per * 4, mism);
                break;
            }
        }
        printf("first 64 chunk classes: ");
        for (int c = 0; c < 64; ++c) printf("%d", cls[c]);
        printf("\n");
        // SM groups: mean latency on class-0 vs class-1 chunks
        std::vector<uint8_t> sgrp(256, 0);
        int ng[2] = {0, 0};
        printf("smid:group(mean0/mean1)");
        for (int b2 = 0; b2 < nblk; ++b2) {
            double m[2] = {0, 0};
            int k[2] = {0, 0};
            for (int c = 0; c < nchunks; ++c) {
                m[cls[c]] += hl[(size_t)b2 * nchunks + c];
                k[cls[c]]++;
            }
            m[0] /= std::max(1, k[0]);
            m[1] /= std::max(1, k[1]);
            const int g = m[0] <= m[1] ? 0 : 1;
            sgrp[hs[b2]] = (uint8_t)g;
            ng[g]++;
            printf(" %u:%d(%.0f/%.0f)", hs[b2], g, m[0], m[1]);
        }
        printf("\nSM groups: %d / %d\n", ng[0], ng[1]);
        // groups.bin for the write test: period = 512 chunks (2 MiB) of classes, then SM groups
        FILE *f = fopen(argc > 2 ? argv[2] : "groups.bin", "wb");
        const int per = 512;
        fwrite(&per, 4, 1, f);
        fwrite(cls.data(), 1, per, f);
        fwrite(sgrp.data(), 1, nsm, f);
        fclose(f);
        return 0;
    }
    // write <groups.bin: period bytes of chunk groups, then nsm bytes of SM groups>
    if (!strcmp(what, "write") && argc > 2) {
        FILE *f = fopen(argv[2], "rb");
        if (!f) return 2;
        int period = 0;
        if (fread(&period, 4, 1, f) != 1) return 2;
        std::vector<uint8_t> cgrp(period), sgrp(256, 0);
        if (fread(cgrp.data(), 1, period, f) != (size_t)period) return 2;
        if (fread(sgrp.data(), 1, nsm, f) != (size_t)nsm) return 2;
        fclose(f);
        uint8_t *dc, *ds;
        CK(cudaMalloc(&dc, period));
        CK(cudaMalloc(&ds, 256));
        CK(cudaMemcpy(dc, cgrp.data(), period, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ds, sgrp.data(), 256, cudaMemcpyHostToDevice));
        const size_t bytes = 16ull << 30, nchunks = bytes / kChunk;
        uint64_t *buf;
        CK(cudaMalloc(&buf, bytes));
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        unsigned long long *dbytes;
        CK(cudaMalloc(&dbytes, 8));
        for (int rep = 0; rep < 3; ++rep)
            for (int mode = 0; mode < 3; ++mode) {
                write_kernel<<<nsm * 4, 128>>>(buf, nchunks, dc, period, ds, mode, 1, dbytes);  // warm
                CK(cudaMemset(dbytes, 0, 8));
                cudaEventRecord(a);
                write_kernel<<<nsm * 4, 128>>>(buf, nchunks, dc, period, ds, mode, 2, dbytes);
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                unsigned long long hb = 0;
                CK(cudaMemcpy(&hb, dbytes, 8, cudaMemcpyDeviceToHost));
                printf("mode %d (%s) rep %d: %.1f GB/s over %.2f GB\n", mode,
                       mode == 0 ? "all chunks" : mode == 1 ? "own-group chunks" : "other-group chunks", rep,
                       hb / (ms * 1e-3) / 1e9, hb / 1e9);
            }
        return 0;
    }
    fprintf(stderr, "usage: die_probe lat | write groups.bin\n");
    return 2;
}
