// Host <-> device transfers for PAGEABLE host memory.
//
// The drop-in's callers hand over plain numpy arrays (GridBuffer.data,
// core.py:232-373; the box of sweep()).  cudaMemcpy from / to pageable memory
// stages through the driver's own bounce buffers on one thread: measured on the
// C5 box (3.65 GB) 10.5 GB/s up and 3.5-4.2 GB/s down (the freshly allocated
// output array also takes its page faults inside the copy) -- 1.26 s around a
// 0.10 s sweep.  Here pageable transfers run through two pinned bounce
// buffers: a few host threads copy chunk i+1 between the caller's array and
// one buffer (first-touch faults spread over the threads) while the copy
// engine moves chunk i from / to the other.  Pinned host memory (the bench's
// pipelined path, torch pinned tensors) is detected and copied directly.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "plan.hpp"

namespace sbh {
namespace {

constexpr size_t kChunk = 32u << 20;   // bytes per bounce buffer

struct Bounce {
    std::mutex mu;            // one pageable transfer at a time per process
    void* buf[2] = {nullptr, nullptr};
    void* buf2[2] = {nullptr, nullptr};   // second pair (streamed sweeps: up and down at once)
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int device = -1;
};
Bounce g_bounce;

int bounce_ready(int device) {
    Bounce& b = g_bounce;
    if (b.buf[0] && b.device == device) return SB_OK;
    for (int i = 0; i < 2; i++) {   // (events belong to a device: re-create on a device change)
        if (b.ev[i]) cudaEventDestroy(b.ev[i]);
        b.ev[i] = nullptr;
        if (!b.buf[i]) SB_CUDA(cudaHostAlloc(&b.buf[i], kChunk, cudaHostAllocPortable));
        SB_CUDA(cudaEventCreateWithFlags(&b.ev[i], cudaEventDisableTiming));
    }
    b.device = device;
    return SB_OK;
}

int host_threads() {
    static const int n = [] {
        const int env = (int)env_double("SB200_XFER_THREADS", 0);
        if (env > 0) return std::min(env, 64);
        const unsigned hw = std::thread::hardware_concurrency();
        return (int)std::max(1u, std::min(16u, hw));   // (C5 box, 16-thread host: 8 threads 413 ms per call, 16: 348)
    }();
    return n;
}

// One thread's share of a copy.  Large pieces go through non-temporal stores (the
// destination is either a bounce buffer the copy engine reads next or the caller's array,
// not data this core will touch again): no read-for-ownership of the destination lines,
// 2 instead of 3 memory transfers per byte.  SB200_XFER_NT=0: plain memcpy.
#if defined(__x86_64__)
#include <immintrin.h>
__attribute__((target("avx2"))) void copy_nt_avx2(char* dst, const char* src, size_t n) {
    const size_t head = (32 - (reinterpret_cast<uintptr_t>(dst) & 31)) & 31;
    if (head >= n) {
        std::memcpy(dst, src, n);
        return;
    }
    std::memcpy(dst, src, head);
    dst += head;
    src += head;
    n -= head;
    size_t i = 0;
    for (; i + 128 <= n; i += 128) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 32));
        const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 64));
        const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 96), d);
    }
    _mm_sfence();
    if (i < n) std::memcpy(dst + i, src + i, n - i);
}
#endif

void copy_bytes(char* dst, const char* src, size_t n) {
#if defined(__x86_64__)
    static const bool nt = env_double("SB200_XFER_NT", 1) != 0 && __builtin_cpu_supports("avx2");
    if (nt && n >= 4096) {
        copy_nt_avx2(dst, src, n);
        return;
    }
#endif
    std::memcpy(dst, src, n);
}

}  // namespace

// rows x row_bytes from src (pitch sp) to dst (pitch dp), split over the host threads
void parallel_copy_rows(char* dst, size_t dp, const char* src, size_t sp, size_t row_bytes, size_t rows, int share) {
    // `share` > 1: this caller takes 1/share of the host threads (two directions at once)
    const int cap = std::max(1, host_threads() / std::max(1, share));
    const int nt = (int)std::min<size_t>((size_t)cap, std::max<size_t>(1, rows * row_bytes / (1u << 20)));
    auto work = [=](int t) {
        if (dp == row_bytes && sp == row_bytes) {      // contiguous: split by bytes (64 B granules)
            const size_t total = rows * row_bytes;
            const size_t per = ((total + nt - 1) / nt + 63) / 64 * 64;
            const size_t lo = std::min(total, per * t), hi = std::min(total, per * (t + 1));
            if (hi > lo) copy_bytes(dst + lo, src + lo, hi - lo);
        } else {
            const size_t per = (rows + nt - 1) / nt;
            const size_t lo = std::min(rows, per * t), hi = std::min(rows, per * (t + 1));
            for (size_t r = lo; r < hi; r++) copy_bytes(dst + r * dp, src + r * sp, row_bytes);
        }
    };
    if (nt <= 1) {
        work(0);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(nt - 1);
    for (int t = 1; t < nt; t++) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
}

// Both bounce pairs for one caller (sb_sweep_host), under the process-wide transfer lock
// until xfer_release().
int xfer_acquire(int device, void* up[2], void* down[2], size_t* chunk_bytes) {
    g_bounce.mu.lock();
    int rc = bounce_ready(device);
    for (int i = 0; i < 2 && rc == SB_OK; i++)
        if (!g_bounce.buf2[i] && cudaHostAlloc(&g_bounce.buf2[i], kChunk, cudaHostAllocPortable) != cudaSuccess)
            rc = fail(SB_ERR_NOMEM, "pinned bounce buffer allocation failed");
    if (rc != SB_OK) {
        g_bounce.mu.unlock();
        return rc;
    }
    for (int i = 0; i < 2; i++) {
        up[i] = g_bounce.buf[i];
        down[i] = g_bounce.buf2[i];
    }
    *chunk_bytes = kChunk;
    return SB_OK;
}
void xfer_release() { g_bounce.mu.unlock(); }

// Pinned (cudaHostAlloc / cudaHostRegister) or managed memory: the copy engines read it directly.
bool host_is_pinned(const void* p) {
    static const int force = (int)env_double("SB200_XFER_BOUNCE", 1);   // 0: always the plain cudaMemcpy path
    if (!force) return true;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

// Pageable host rows (pitch host_pitch) -> contiguous device rows, stream-ordered on `st`;
// returns when the last chunk has been handed to the copy engine out of a bounce buffer
// (the caller's array is no longer read).
int h2d_pageable_rows(void* dst, const void* host, size_t host_pitch, size_t row_bytes, size_t rows, int device,
                      cudaStream_t st) {
    std::lock_guard<std::mutex> lock(g_bounce.mu);
    const int rc = bounce_ready(device);
    if (rc != SB_OK) return rc;
    Bounce& b = g_bounce;
    if (row_bytes > kChunk) return fail(SB_ERR_ARG, "row of %zu bytes exceeds the transfer chunk", row_bytes);
    const size_t rpc = std::max<size_t>(1, kChunk / row_bytes);   // rows per chunk
    int slot = 0;
    for (size_t r0 = 0; r0 < rows; r0 += rpc, slot ^= 1) {
        const size_t nr = std::min(rpc, rows - r0);
        SB_CUDA(cudaEventSynchronize(b.ev[slot]));      // the copy that last read this buffer is done
        parallel_copy_rows(static_cast<char*>(b.buf[slot]), row_bytes, static_cast<const char*>(host) + r0 * host_pitch,
                           host_pitch, row_bytes, nr);
        SB_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + r0 * row_bytes, b.buf[slot], nr * row_bytes,
                                cudaMemcpyHostToDevice, st));
        SB_CUDA(cudaEventRecord(b.ev[slot], st));
    }
    // the bounce buffers are shared: the next transfer may overwrite them
    SB_CUDA(cudaEventSynchronize(b.ev[0]));
    SB_CUDA(cudaEventSynchronize(b.ev[1]));
    return SB_OK;
}

// Contiguous pageable bytes: pieces of 4 MB as rows, then the remainder.
int h2d_pageable(void* dst, const void* src, size_t bytes, int device, cudaStream_t st) {
    const size_t piece = 4u << 20, full = bytes / piece;
    int rc = h2d_pageable_rows(dst, src, piece, piece, full, device, st);
    if (rc == SB_OK && bytes > full * piece)
        rc = h2d_pageable_rows(static_cast<char*>(dst) + full * piece, static_cast<const char*>(src) + full * piece,
                               bytes - full * piece, bytes - full * piece, 1, device, st);
    return rc;
}

// Pitched device rows -> compact pageable host rows; returns when `host` holds the data.
int d2h_pageable_rows(void* host, size_t host_pitch, const void* src, size_t src_pitch, size_t row_bytes, size_t rows,
                      int device, cudaStream_t st) {
    std::lock_guard<std::mutex> lock(g_bounce.mu);
    const int rc = bounce_ready(device);
    if (rc != SB_OK) return rc;
    Bounce& b = g_bounce;
    if (row_bytes > kChunk) return fail(SB_ERR_ARG, "row of %zu bytes exceeds the transfer chunk", row_bytes);
    const size_t rpc = std::max<size_t>(1, kChunk / row_bytes);   // rows per chunk
    auto issue = [&](size_t r0, int slot) -> int {
        const size_t nr = std::min(rpc, rows - r0);
        SB_CUDA(cudaMemcpy2DAsync(b.buf[slot], row_bytes, static_cast<const char*>(src) + r0 * src_pitch, src_pitch,
                                  row_bytes, nr, cudaMemcpyDeviceToHost, st));
        SB_CUDA(cudaEventRecord(b.ev[slot], st));
        return SB_OK;
    };
    if (rows == 0) return SB_OK;
    int rc2 = issue(0, 0);
    if (rc2 != SB_OK) return rc2;
    int slot = 0;
    for (size_t r0 = 0; r0 < rows; r0 += rpc, slot ^= 1) {
        if (r0 + rpc < rows) {                          // next chunk into the other buffer meanwhile
            rc2 = issue(r0 + rpc, slot ^ 1);
            if (rc2 != SB_OK) return rc2;
        }
        SB_CUDA(cudaEventSynchronize(b.ev[slot]));
        const size_t nr = std::min(rpc, rows - r0);
        parallel_copy_rows(static_cast<char*>(host) + r0 * host_pitch, host_pitch, static_cast<const char*>(b.buf[slot]),
                           row_bytes, row_bytes, nr);
    }
    return SB_OK;
}

}  // namespace sbh
