// prng_pipeline.cu -- a4 + a5: the end-to-end modes of prng_generate (device double buffer,
// side copy stream, pinned / pageable / mapped host buffers, sink) and prng_generate_host
// (D2H straight into a caller's -- possibly shared, multi-rank -- host array).
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "engine_internal.h"

using namespace prng_detail;

// ---------------------------------------------------------------------------- end to end
// Device double buffer of the end-to-end paths: 2 halves x T slots.
static int ensure_dbuf(prng *h, uint64_t T, prng_err_t *err) {
    const uint64_t pitch = pitch_for(h->count);
    if (!h->d_buf || h->buf_T != T || h->buf_pitch != pitch) {
        if (h->d_buf) cudaFree(h->d_buf);
        h->d_buf = nullptr;
        CU(cudaMalloc(&h->d_buf, 2 * T * pitch * sizeof(uint64_t)));
        h->buf_T = T;
        h->buf_pitch = pitch;
    }
    return PRNG_OK;
}

static int ensure_e2e(prng *h, uint64_t T, int halves, int kind, bool need_dbuf, prng_err_t *err) {
    if (need_dbuf)
        if (int rc = ensure_dbuf(h, T, err)) return rc;
    if (h->h_T != T || h->h_halves < halves || h->h_kind != kind) {
        for (int i = 0; i < 2; ++i) {
            free_host(h->h_kind, h->h_buf[i], h->h_T * h->count * sizeof(uint64_t));
            h->h_buf[i] = h->h_dev[i] = nullptr;
        }
        h->h_kind = kind;
        h->h_T = T;
        h->h_halves = 0;
        const size_t bytes = T * h->count * sizeof(uint64_t);
        for (int i = 0; i < halves; ++i) {
            void *p = nullptr;
            switch (kind) {
                case HK_PINNED: CU(cudaHostAlloc(&p, bytes, cudaHostAllocDefault)); break;
                case HK_PINNED_WC: CU(cudaHostAlloc(&p, bytes, cudaHostAllocWriteCombined)); break;
                case HK_MAPPED: CU(cudaHostAlloc(&p, bytes, cudaHostAllocMapped)); break;
                case HK_HUGE_REGISTERED: {
                    // anonymous mapping advised onto 2 MiB transparent huge pages, then pinned
                    p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
                    if (p == MAP_FAILED) return set_err(err, PRNG_ENOMEM, "mmap(%zu)", bytes);
                    madvise(p, bytes, MADV_HUGEPAGE);
                    std::memset(p, 0, bytes);
                    cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterDefault);
                    if (e != cudaSuccess) {
                        munmap(p, bytes);
                        return set_err(err, PRNG_ECUDA, "cudaHostRegister: %s", cudaGetErrorString(e));
                    }
                    break;
                }
                default:
                    p = std::malloc(bytes);
                    if (!p) return set_err(err, PRNG_ENOMEM, "malloc(%zu)", bytes);
            }
            h->h_buf[i] = (uint64_t *)p;
            if (kind == HK_MAPPED) CU(cudaHostGetDevicePointer((void **)&h->h_dev[i], p, 0));
            h->h_halves = i + 1;
        }
    }
    return PRNG_OK;
}

// O3 (zero-copy): the generation kernel stores each batch straight into a mapped pinned
// host half over PCIe -- no device ring, no copy engine; the store IS the transfer.
// sink(j) runs while gen(j+1) writes the other half; gen(j+2) is enqueued after sink(j).
static int generate_zerocopy(prng *h, uint64_t numiter, uint64_t T, uint64_t T_alloc, prng_sink_fn sink,
                             void *user, prng_err_t *err) {
    if (h->count % 4) return set_err(err, PRNG_EINVAL, "zero-copy mode needs count %% 4 == 0 (32-B aligned rows)");
    if (int rc = ensure_e2e(h, T_alloc, 2, HK_MAPPED, false, err)) return rc;
    const double t0 = now_s();  // wall time of the profiled call, allocations excluded
    const uint64_t nb = (numiter + T - 1) / T;
    const uint64_t pos0 = h->pos;
    auto iters_of = [&](uint64_t j) { return (uint32_t)std::min<uint64_t>(T, numiter - j * T); };
    if (int rc = pipeline_events(h, err)) return rc;
    cudaEvent_t *const ev = h->pev;  // ev[0], ev[1]: gen(j) done, per host half
    int rc = PRNG_OK;
    auto gen = [&](uint64_t j) -> int {
        if (int r = launch_batch(h, h->h_dev[j & 1], h->count, T, 0, iters_of(j), pos0 + j * T == 0, h->s_gen, err))
            return r;
        cudaError_t e = cudaEventRecord(ev[j & 1], h->s_gen);
        return e == cudaSuccess ? PRNG_OK : set_err(err, PRNG_ECUDA, "cudaEventRecord: %s", cudaGetErrorString(e));
    };
    for (uint64_t j = 0; j < std::min<uint64_t>(nb, 2) && !rc; ++j) rc = gen(j);
    for (uint64_t j = 0; j < nb && !rc; ++j) {
        cudaError_t e = cudaEventSynchronize(ev[j & 1]);
        if (e != cudaSuccess) {
            rc = set_err(err, PRNG_ECUDA, "cudaEventSynchronize: %s", cudaGetErrorString(e));
            break;
        }
        const double a = now_s();
        int r = sink(user, pos0 + j * T, iters_of(j), h->gid_begin, h->count, h->h_buf[j & 1]);
        if (h->profile) h->host_iv.push_back({PRNG_EV_OUT, a - h->host_origin, now_s() - h->host_origin});
        if (r != 0) {
            rc = set_err(err, PRNG_ESINK, "sink returned %d at batch %llu", r, (unsigned long long)j);
            break;
        }
        if (j + 2 < nb) rc = gen(j + 2);
    }
    const cudaError_t es = cudaStreamSynchronize(h->s_gen);
    if (!rc && es != cudaSuccess) rc = set_err(err, PRNG_ECUDA, "generation stream: %s", cudaGetErrorString(es));
    if (rc) {
        h->poisoned = true;
        return rc;
    }
    h->pos = pos0 + numiter;
    h->wall_s += now_s() - t0;
    return PRNG_OK;
}

static int enqueue_copy(prng *h, uint64_t *hdst, const uint64_t *dsrc, uint64_t iters, cudaStream_t s,
                        prng_err_t *err) {
    if (int rc = prof_begin(h, s, PRNG_EV_READ_BUFFER, err)) return rc;
    const size_t row = h->count * sizeof(uint64_t);
    if (h->buf_pitch == h->count) {
        CU(cudaMemcpyAsync(hdst, dsrc, row * iters, cudaMemcpyDeviceToHost, s));
    } else {
        CU(cudaMemcpy2DAsync(hdst, row, dsrc, h->buf_pitch * sizeof(uint64_t), row, iters, cudaMemcpyDeviceToHost, s));
    }
    return prof_end(h, s, err);
}

int prng_detail::generate_e2e(prng *h, uint64_t numiter, prng_sink_fn sink, void *user, prng_err_t *err) {
    uint64_t T = (uint64_t)h->batch_iters;
    const uint64_t row = h->count * sizeof(uint64_t);
    if (T == 0) T = std::max<uint64_t>(1, (256ull << 20) / row);  // ~256 MiB per batch
    const uint64_t T_alloc = T;  // buffers are sized for full batches: no re-allocation per call
    T = std::min<uint64_t>(T, numiter);
    const int mode = h->mode;
    if (mode == PRNG_MODE_ZEROCOPY) {
        return generate_zerocopy(h, numiter, T, T_alloc, sink, user, err);
    }
    const int halves = (mode == PRNG_MODE_OVERLAP2 || mode == PRNG_MODE_PAGEABLE) ? 2 : 1;
    if (int rc = ensure_e2e(h, T_alloc, halves, mode == PRNG_MODE_PAGEABLE ? HK_PAGEABLE : h->host_mem, true, err))
        return rc;
    const uint64_t nb = (numiter + T - 1) / T;
    const uint64_t pitch = h->buf_pitch;
    auto iters_of = [&](uint64_t j) { return (uint32_t)std::min<uint64_t>(T, numiter - j * T); };
    auto dslot = [&](uint64_t j) { return (mode == PRNG_MODE_SERIAL ? 0 : (j & 1)) * T; };
    const uint64_t pos0 = h->pos;
    const double t0 = now_s();

    auto run_sink = [&](uint64_t j, const uint64_t *data) -> int {
        const double a = now_s();
        int r = sink ? sink(user, pos0 + j * T, iters_of(j), h->gid_begin, h->count, data) : 0;
        if (h->profile) h->host_iv.push_back({PRNG_EV_OUT, a - h->host_origin, now_s() - h->host_origin});
        if (r != 0) {
            h->poisoned = true;
            return set_err(err, PRNG_ESINK, "sink returned %d at batch %llu", r, (unsigned long long)j);
        }
        return PRNG_OK;
    };

    if (mode == PRNG_MODE_SERIAL) {
        // S0: everything on one stream, one buffer each side: gen -> read -> out -> gen ...
        for (uint64_t j = 0; j < nb; ++j) {
            if (int rc = launch_batch(h, h->d_buf, pitch, 2 * T, 0, iters_of(j), pos0 + j * T == 0, h->s_gen, err))
                return rc;
            if (int rc = enqueue_copy(h, h->h_buf[0], h->d_buf, iters_of(j), h->s_gen, err)) return rc;
            CU(cudaStreamSynchronize(h->s_gen));
            if (int rc = run_sink(j, h->h_buf[0])) return rc;
        }
        h->pos = pos0 + numiter;
        h->wall_s += now_s() - t0;
        return PRNG_OK;
    }

    // Overlapped modes (S1, O1, O2): gen stream + copy stream + events.
    const int R = 8;  // event ring; at most gen(j+4) / copy(j+2) ahead of the host at batch j
    if (int rc = pipeline_events(h, err)) return rc;
    cudaEvent_t *const ev_gen = h->pev, *const ev_cp = h->pev + R;
    static_assert(2 * R <= prng::kPipeEvents, "event pool too small");
    int rc = PRNG_OK;
    uint64_t gen_enq = 0, cp_enq = 0;  // batches enqueued so far
    auto enqueue_gen = [&](uint64_t j) -> int {
        // gen(j) overwrites device half j%2, last read by copy(j-2)  (WAR, A15)
        if (j >= 2) {
            cudaError_t e = cudaStreamWaitEvent(h->s_gen, ev_cp[(j - 2) % R], 0);
            if (e != cudaSuccess) return set_err(err, PRNG_ECUDA, "cudaStreamWaitEvent: %s", cudaGetErrorString(e));
        }
        if (int r = launch_batch(h, h->d_buf, pitch, 2 * T, dslot(j), iters_of(j), pos0 + j * T == 0, h->s_gen, err))
            return r;
        cudaError_t e = cudaEventRecord(ev_gen[j % R], h->s_gen);
        if (e != cudaSuccess) return set_err(err, PRNG_ECUDA, "cudaEventRecord: %s", cudaGetErrorString(e));
        gen_enq = j + 1;
        return PRNG_OK;
    };
    auto enqueue_cp = [&](uint64_t j) -> int {
        // copy(j) reads device half j%2 after gen(j) wrote it  (RAW, A15)
        cudaError_t e = cudaStreamWaitEvent(h->s_copy, ev_gen[j % R], 0);
        if (e != cudaSuccess) return set_err(err, PRNG_ECUDA, "cudaStreamWaitEvent: %s", cudaGetErrorString(e));
        if (int r = enqueue_copy(h, h->h_buf[j % halves], h->d_buf + dslot(j) * pitch, iters_of(j), h->s_copy, err))
            return r;
        e = cudaEventRecord(ev_cp[j % R], h->s_copy);
        if (e != cudaSuccess) return set_err(err, PRNG_ECUDA, "cudaEventRecord: %s", cudaGetErrorString(e));
        cp_enq = j + 1;
        return PRNG_OK;
    };

    // Prologue: gen(0), copy(0), gen(1), [copy(1) if a second host half], gen(2), gen(3).
    for (uint64_t j = 0; j < std::min<uint64_t>(nb, 2) && !rc; ++j) {
        rc = enqueue_gen(j);
        if (!rc && j < (uint64_t)halves) rc = enqueue_cp(j);
    }
    while (!rc && gen_enq < nb && gen_enq < cp_enq + 2) rc = enqueue_gen(gen_enq);

    for (uint64_t j = 0; j < nb && !rc; ++j) {
        cudaError_t e = cudaEventSynchronize(ev_cp[j % R]);
        if (e != cudaSuccess) {
            rc = set_err(err, PRNG_ECUDA, "cudaEventSynchronize: %s", cudaGetErrorString(e));
            break;
        }
        rc = run_sink(j, h->h_buf[j % halves]);
        if (rc) break;
        // host half j%halves is free again: queue the next copy into it, then the next gen
        if (cp_enq < nb) rc = enqueue_cp(cp_enq);
        while (!rc && gen_enq < nb && gen_enq < cp_enq + 2) rc = enqueue_gen(gen_enq);
    }
    if (rc) {
        cudaStreamSynchronize(h->s_gen);
        cudaStreamSynchronize(h->s_copy);
        h->poisoned = true;
        return rc;
    }
    const cudaError_t es = cudaStreamSynchronize(h->s_gen);
    if (es != cudaSuccess) {
        h->poisoned = true;
        return set_err(err, PRNG_ECUDA, "generation stream: %s", cudaGetErrorString(es));
    }
    h->pos = pos0 + numiter;
    h->wall_s += now_s() - t0;
    return PRNG_OK;
}

extern "C" {

// ---------------------------------------------------------------------------- host array
// a4 + a5, multi-rank form (BASELINE north_star: "each rank generates its own gid range and
// writes its slice of the host output directly"): D2H straight into the caller's host array
// -- no staging buffer, no sink.  Iteration k of this call lands in row k mod dst_rows:
// dst[(k mod dst_rows) * dst_pitch + j], j < count.  For a shared array the caller passes
// dst = array + gid_begin and dst_pitch = numrn_total, so every rank fills its own columns.
int prng_generate_host(prng_t *h, uint64_t numiter, uint64_t *dst, uint64_t dst_pitch, uint64_t dst_rows,
                       prng_err_t *err) {
    if (int rc = check_handle(h, err, true)) return rc;
    if (numiter < 1 || !dst || dst_pitch < h->count || dst_rows < 1)
        return set_err(err, PRNG_EINVAL, "numiter >= 1, dst != NULL, dst_pitch >= count, dst_rows >= 1");
    if (int rc = ensure_origin(h, err)) return rc;
    const uint64_t row = h->count * sizeof(uint64_t);
    uint64_t T = (uint64_t)h->batch_iters;
    if (T == 0) T = std::max<uint64_t>(1, (256ull << 20) / row);
    if (int rc = ensure_dbuf(h, T, err)) return rc;
    T = std::min<uint64_t>(T, numiter);
    // pin the destination for the DMA engine unless it already is (registered / cudaHostAlloc)
    const size_t span = ((std::min<uint64_t>(dst_rows, numiter) - 1) * dst_pitch + h->count) * sizeof(uint64_t);
    cudaPointerAttributes attr;
    bool registered_here = false;
    if (cudaPointerGetAttributes(&attr, dst) != cudaSuccess || attr.type != cudaMemoryTypeHost) {
        cudaGetLastError();
        CU(cudaHostRegister(dst, span, cudaHostRegisterDefault));
        registered_here = true;
    }
    const uint64_t nb = (numiter + T - 1) / T, pitch = h->buf_pitch, pos0 = h->pos;
    auto iters_of = [&](uint64_t j) { return (uint32_t)std::min<uint64_t>(T, numiter - j * T); };
    const int R = 4;
    if (int r = pipeline_events(h, err)) {
        if (registered_here) cudaHostUnregister(dst);
        return r;
    }
    cudaEvent_t *const ev_gen = h->pev, *const ev_cp = h->pev + R;
    int rc = PRNG_OK;
    // every CUDA call of the pipeline is checked: a failed record / wait would otherwise let
    // a copy run before its generation (or a generation overwrite a half still being read)
    auto chk = [&](cudaError_t e, const char *what) -> int {
        e = fault_point(h, e);
        if (e == cudaSuccess) return PRNG_OK;
        return set_err(err, e == cudaErrorMemoryAllocation ? PRNG_ENOMEM : PRNG_ECUDA, "%s: %s", what,
                       cudaGetErrorString(e));
    };
    const double t0 = now_s();
    for (uint64_t j = 0; j < nb && !rc; ++j) {
        // gen(j) into device half j%2, after copy(j-2) has drained it (WAR, A15)
        if (j >= 2 && (rc = chk(cudaStreamWaitEvent(h->s_gen, ev_cp[(j - 2) % R], 0), "cudaStreamWaitEvent(gen)")))
            break;
        rc = launch_batch(h, h->d_buf, pitch, 2 * T, (j & 1) * T, iters_of(j), pos0 + j * T == 0, h->s_gen, err);
        if (rc) break;
        if ((rc = chk(cudaEventRecord(ev_gen[j % R], h->s_gen), "cudaEventRecord(gen)"))) break;
        // copy(j): rows (pos0 + j*T + t) mod dst_rows, split where the host ring wraps
        if ((rc = chk(cudaStreamWaitEvent(h->s_copy, ev_gen[j % R], 0), "cudaStreamWaitEvent(copy)"))) break;
        if ((rc = prof_begin(h, h->s_copy, PRNG_EV_READ_BUFFER, err))) break;
        uint64_t t = 0;
        while (t < iters_of(j)) {
            const uint64_t r0 = (j * T + t) % dst_rows;  // destination row of call iteration j*T + t
            const uint64_t nrows = std::min<uint64_t>(iters_of(j) - t, dst_rows - r0);
            rc = chk(cudaMemcpy2DAsync(dst + r0 * dst_pitch, dst_pitch * sizeof(uint64_t),
                                       h->d_buf + ((j & 1) * T + t) * pitch, pitch * sizeof(uint64_t), row, nrows,
                                       cudaMemcpyDeviceToHost, h->s_copy),
                     "cudaMemcpy2DAsync");
            if (rc) break;
            t += nrows;
        }
        if (rc) break;
        if ((rc = prof_end(h, h->s_copy, err))) break;
        if ((rc = chk(cudaEventRecord(ev_cp[j % R], h->s_copy), "cudaEventRecord(copy)"))) break;
        // keep at most two batches in flight per stream (the event ring has R = 4 entries)
        if (j >= 2 && (rc = chk(cudaEventSynchronize(ev_cp[(j - 2) % R]), "cudaEventSynchronize"))) break;
    }
    const cudaError_t eg = cudaStreamSynchronize(h->s_gen);
    const cudaError_t ec = cudaStreamSynchronize(h->s_copy);
    if (registered_here) cudaHostUnregister(dst);
    if (!rc) rc = chk(eg, "generation stream");
    if (!rc) rc = chk(ec, "copy stream");
    if (rc) {
        h->poisoned = true;
        return rc;
    }
    h->pos = pos0 + numiter;
    h->wall_s += now_s() - t0;
    return ok(err);
}

}  // extern "C"
