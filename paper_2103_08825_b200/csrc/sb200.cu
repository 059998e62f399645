// sb200 -- plan management, device layout, dispatch and the C ABI
// (include/sb200.h).  Host side of the B200 multistep stencil sweep.
//
// Device layout (private; the host convention is the compact halo box):
//   * unit axis x padded to a pitch px so interior x = 0 starts 128 B aligned
//     (512 B for 1D, whose single row also carries the kernel's read-ahead);
//   * outer axes keep their r-deep halo rows/planes, and the slab axis
//     (axis 0) keeps h_lo/h_hi = r (physical) or the ghost depth G (slab);
//   * two buffers (ping-pong), halo and ghost present in both.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <condition_variable>
#include <cstdio>
#include <mutex>
#include <thread>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "generic.cuh"
#include "plan.hpp"

namespace sbh {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

// Tuning knobs (development only; defaults are the measured best).
double env_double(const char* name, double dflt) {
    const char* v = getenv(name);
    return v ? atof(v) : dflt;
}


}  // namespace sbh

using namespace sbh;

namespace {

int validate_problem(const sb_problem* p) {
    if (!p) return fail(SB_ERR_ARG, "problem is NULL");
    if (p->d < 1 || p->d > 3) return fail(SB_ERR_SPEC, "dimension must be 1, 2 or 3, got %d", p->d);
    if (p->r < 1) return fail(SB_ERR_SPEC, "order must be positive, got %d", p->r);
    if (p->shape != SB_STAR && p->shape != SB_BOX)
        return fail(SB_ERR_SPEC, "shape must be star or box, got %d", p->shape);
    if (!p->offsets || !p->weights) return fail(SB_ERR_SPEC, "offsets/weights are NULL");
    const int d = p->d, r = p->r;
    int64_t expected = 1;
    if (p->shape == SB_STAR) {
        expected = 2 * d * r + 1;
    } else {
        for (int a = 0; a < d; a++) expected *= (2 * r + 1);
    }
    if (p->nw != expected)
        return fail(SB_ERR_SPEC, "%s stencil of d=%d r=%d needs %lld weights, got %d",
                    p->shape == SB_STAR ? "star" : "box", d, r, (long long)expected, p->nw);
    if (p->nw > sb::kGenericMaxW) return fail(SB_ERR_SPEC, "too many weights (%d)", p->nw);
    bool has_zero = false;
    for (int i = 0; i < p->nw; i++) {
        int nz = 0, mx = 0;
        for (int a = 0; a < d; a++) {
            const int c = p->offsets[i * d + a];
            nz += (c != 0);
            mx = std::max(mx, c < 0 ? -c : c);
        }
        if (mx > r) return fail(SB_ERR_SPEC, "offset %d outside radius %d", i, r);
        if (nz == 0) has_zero = true;
        if (p->shape == SB_STAR && nz > 1) return fail(SB_ERR_SPEC, "star stencil has a non-axis-aligned offset");
        if (i > 0) {  // strictly increasing lexicographic order
            int cmp = 0;
            for (int a = 0; a < d && cmp == 0; a++) {
                const int x = p->offsets[(i - 1) * d + a], y = p->offsets[i * d + a];
                cmp = (x < y) ? -1 : (x > y ? 1 : 0);
            }
            if (cmp >= 0) return fail(SB_ERR_SPEC, "offsets not in canonical (lexicographic) order at %d", i);
        }
    }
    if (!has_zero) return fail(SB_ERR_SPEC, "zero offset missing from weight table");
    for (int a = 0; a < d; a++)
        if (p->dims[a] <= 0) return fail(SB_ERR_GRID, "extents must be positive (axis %d)", a);
    if (p->dtype != SB_F64 && p->dtype != SB_F32) return fail(SB_ERR_ARG, "dtype must be SB_F64 or SB_F32");
    if (p->arith != SB_ARITH_EXACT && p->arith != SB_ARITH_FMA) return fail(SB_ERR_ARG, "arith must be EXACT or FMA");
    if (p->k < 0 || p->k > 64) return fail(SB_ERR_ARG, "fusion depth k=%d out of range", p->k);
    if (p->ghost_lo < 0 || p->ghost_hi < 0) return fail(SB_ERR_GRID, "ghost depth must be >= 0");
    if ((p->ghost_lo > 0 && p->ghost_lo < r) || (p->ghost_hi > 0 && p->ghost_hi < r))
        return fail(SB_ERR_GRID, "ghost depth must be >= r=%d", r);
    if (p->kernel < SB_KERNEL_AUTO || p->kernel > SB_KERNEL_FUSED) return fail(SB_ERR_ARG, "bad kernel choice");
    return SB_OK;
}

// Fused kernel available for this stencil class (0 = none).
int fused_kind(const sb_plan* P) {
    if (P->d == 1 && (P->r == 1 || P->r == 2)) return KK_FUSED1D;
    if (P->d == 3 && P->r == 1) return KK_FUSED3D;   // 7-point star or 27-point box
    if (P->d == 2 && P->r == 1) return KK_FUSED2D;   // 5-point star or 9-point box
    return 0;
}

// Supported fused depths (template instantiations) per kernel.
bool fused_k_ok(const sb_plan* P, int kind, int k) {
    if (kind == KK_FUSED3D) return k >= 1 && k <= 4;
    if (kind == KK_FUSED2D) return k == 1 || k == 2 || k == 4 || k == 8 || ((k == 16 || k == 32) && sep2d_ok(P, k));
    if (k == 32 || k == 64) return compose1d_ok(P, k, 16);   // composed path only
    return k == 1 || k == 2 || k == 4 || k == 8 || k == 16;
}

int largest_fused_k(int kind, int64_t steps, int kmax) {
    if (kind == KK_FUSED3D) return (int)std::min<int64_t>(steps, kmax);
    int k = 1;
    while (k * 2 <= kmax && k * 2 <= steps) k *= 2;
    return k;
}

int default_k(int kind, const sb_plan* P) {
    if (kind == KK_FUSED3D) return 2;   // measured best for both 3D stencils (C4, C5)
    if (kind == KK_FUSED2D) {
        // rank-1 weights in FMA mode: the separable composed path (K2c); else the
        // level-by-level kernel's measured best (C3 k=4)
        const int ks = (int)env_double("SB200_SEP2D_K", 32);
        if ((ks == 16 || ks == 32) && sep2d_ok(P, ks)) return ks;
        return 4;
    }
    // 1D: the deepest composed depth in FMA mode (C2 k=32: ~3960 vs k=16: ~3670;
    // C1 k=64: one launch for T=64), else the level-by-level kernel's 16
    if (compose1d_ok(P, 64, 16)) return 64;
    if (compose1d_ok(P, 32, 16)) return 32;
    return 16;
}

// ---------------------------------------------------------------- launches

template <typename T, bool FMA>
int launch_generic_box(sb_plan* P, const T* src, T* dst, const sb::Box3& b) {
    if (b.ext[0] <= 0 || b.ext[1] <= 0 || b.ext[2] <= 0) return SB_OK;
    const int64_t rows = b.ext[0] * b.ext[1];
    dim3 grid((unsigned)((b.ext[2] + sb::kGenericThreads - 1) / sb::kGenericThreads),
              (unsigned)std::min<int64_t>(rows, 65535));
    sb::generic_step_kernel<T, FMA><<<grid, sb::kGenericThreads, 0, P->stream>>>(
        src, dst, P->g, b, P->nw, P->d_lin, reinterpret_cast<const T*>(P->d_w));
    SB_CUDA(cudaGetLastError());
    return SB_OK;
}

// Whole interior; on the slab axis positions [lo, hi) (ghost planes included).
template <typename T, bool FMA>
int launch_generic(sb_plan* P, const T* src, T* dst, int64_t lo, int64_t hi) {
    sb::Box3 b;
    for (int a = 0; a < 3; a++) {
        b.base[a] = 0;
        b.ext[a] = P->g.n[a];
    }
    b.base[P->g.slab_axis] = lo;
    b.ext[P->g.slab_axis] = hi - lo;
    return launch_generic_box<T, FMA>(P, src, dst, b);
}

// One launch advancing k levels from buf[cur] into buf[cur^1].
template <typename T, bool FMA>
int launch_one(sb_plan* P, int k, int level_in_run, int64_t* launches, bool swap = true) {
    const T* src = reinterpret_cast<const T*>(P->buf[P->cur]);
    T* dst = reinterpret_cast<T*>(P->buf[P->cur ^ 1]);
    int rc;
    if (P->kind == KK_FUSED1D) {
        rc = launch_fused1d(P, P->cur, k);
    } else if (P->kind == KK_FUSED3D) {
        rc = launch_fused3d(P, P->cur, k);
    } else if (P->kind == KK_FUSED2D) {
        rc = launch_fused2d(P, P->cur, k);
    } else {
        // generic: one level; on slab sides the valid range shrinks by r per level
        const int64_t n0 = P->dims[0];
        int64_t lo = P->phys_lo ? 0 : -P->hlo + (int64_t)P->r * (level_in_run + 1);
        int64_t hi = P->phys_hi ? n0 : n0 + P->hhi - (int64_t)P->r * (level_in_run + 1);
        if (P->zr_hi >= 0) {   // range launch: interior planes [zr_lo, zr_hi) only
            lo = P->zr_lo;
            hi = P->zr_hi;
        }
        rc = launch_generic<T, FMA>(P, src, dst, lo, hi);
    }
    if (rc != SB_OK) return rc;
    if (swap) P->cur ^= 1;
    ++*launches;
    P->kernels_launched++;
    return SB_OK;
}

template <typename T, bool FMA>
int run_steps(sb_plan* P, int64_t steps, int64_t* launches, int* k_used) {
    const bool slab = !(P->phys_lo && P->phys_hi);
    int64_t done = 0;
    *k_used = 1;
    if (P->kind == KK_GENERIC) {
        for (int64_t t = 0; t < steps; t++) {
            int rc = launch_one<T, FMA>(P, 1, slab ? (int)t : 0, launches);
            if (rc != SB_OK) return rc;
        }
        return SB_OK;
    }
    if (slab) {
        // A slab plan runs one fused launch per exchange interval.
        if (steps <= 64 && fused_k_ok(P, P->kind, (int)steps)) {
            *k_used = (int)steps;
            return launch_one<T, FMA>(P, (int)steps, 0, launches);
        }
        const int saved = P->kind;
        P->kind = KK_GENERIC;
        int rc = SB_OK;
        for (int64_t t = 0; t < steps && rc == SB_OK; t++) rc = launch_one<T, FMA>(P, 1, (int)t, launches);
        P->kind = saved;
        return rc;
    }
    *k_used = P->k;
    while (done < steps) {
        const int kk = (steps - done >= P->k) ? P->k : largest_fused_k(P->kind, steps - done, P->k);
        int rc = launch_one<T, FMA>(P, kk, 0, launches);
        if (rc != SB_OK) return rc;
        done += kk;
    }
    return SB_OK;
}

int dispatch_run(sb_plan* P, int64_t steps, int64_t* launches, int* k_used) {
    const bool fma = P->arith == SB_ARITH_FMA;
    if (P->dtype == SB_F64)
        return fma ? run_steps<double, true>(P, steps, launches, k_used)
                   : run_steps<double, false>(P, steps, launches, k_used);
    return fma ? run_steps<float, true>(P, steps, launches, k_used)
               : run_steps<float, false>(P, steps, launches, k_used);
}

// CUDA-graph replay of repeated sweeps.  The first sweep of a given
// (steps, starting buffer) runs eagerly (it also performs every first-use
// setup: schedules, smem attributes, tensor maps); the second is captured
// from the plan stream (side-stream fork/join included) and instantiated;
// later ones replay it with a single cudaGraphLaunch -- the host cost of a
// short sweep (C1: one composed launch + its boundary windows + 4 event
// calls) drops to one call.  SB200_GRAPHS=0 disables it.
int run_graphed(sb_plan* P, int64_t steps, int64_t* launches, int* k_used) {
    static const bool enabled = env_double("SB200_GRAPHS", 1) != 0 && !getenv("SB200_TRACE");
    if (!enabled || steps == 0) return dispatch_run(P, steps, launches, k_used);
    SweepGraph* g = nullptr;
    for (auto& e : P->graphs)
        if (e.steps == steps && e.cur0 == P->cur) g = &e;
    if (!g) {
        if (P->graphs.size() >= 16) return dispatch_run(P, steps, launches, k_used);
        SweepGraph e;
        e.steps = steps;
        e.cur0 = P->cur;
        P->graphs.push_back(e);
        g = &P->graphs.back();
    }
    // a sweep that is one launch gains nothing from a graph, and direct launches
    // keep programmatic dependent launch across consecutive sweeps (C1: 10.5 vs
    // 12.4 us per sweep measured)
    if (g->failed || ++g->hits < 2 || g->launches == 1) {
        const int rc = dispatch_run(P, steps, launches, k_used);
        if (g->hits == 1) g->launches = *launches;
        return rc;
    }
    if (!g->exec) {
        const int cur_before = P->cur;
        const int64_t kernels_before = P->kernels_launched;
        cudaGraph_t graph = nullptr;
        SB_CUDA(cudaStreamBeginCapture(P->stream, cudaStreamCaptureModeThreadLocal));
        const int rc = dispatch_run(P, steps, &g->launches, &g->k_used);
        const cudaError_t ec = cudaStreamEndCapture(P->stream, &graph);
        g->cur1 = P->cur;
        g->kernels = P->kernels_launched - kernels_before;
        g->last_kernel = P->last_kernel;
        P->cur = cur_before;                       // nothing has executed yet
        P->kernels_launched = kernels_before;
        if (rc != SB_OK || ec != cudaSuccess ||
            cudaGraphInstantiate(&g->exec, graph, 0) != cudaSuccess) {
            if (graph) cudaGraphDestroy(graph);
            cudaGetLastError();                    // clear; fall back to eager launches
            g->failed = true;
            g->exec = nullptr;
            return dispatch_run(P, steps, launches, k_used);
        }
        cudaGraphDestroy(graph);
    }
    SB_CUDA(cudaGraphLaunch(g->exec, P->stream));
    P->cur = g->cur1;
    P->kernels_launched += g->kernels;
    P->last_kernel = g->last_kernel;
    *launches = g->launches;
    *k_used = g->k_used;
    return SB_OK;
}

template <typename T, bool FMA>
int launch_range_t(sb_plan* P, int k, bool finish) {
    int64_t launches = 0;
    return launch_one<T, FMA>(P, k, 0, &launches, finish);
}

const char* kernel_name(const sb_plan* P) {
    if (P->last_kernel) return P->last_kernel;
    if (P->kind == KK_FUSED1D) return "fused1d_kernel";
    if (P->kind == KK_FUSED3D) return "fused3d_kernel";
    if (P->kind == KK_FUSED2D) return "fused2d_kernel";
    return "generic_step_kernel";
}

int max_slab_steps(const sb_plan* P) {
    int64_t m = INT32_MAX;
    if (!P->phys_lo) m = std::min<int64_t>(m, P->hlo / P->r);
    if (!P->phys_hi) m = std::min<int64_t>(m, P->hhi / P->r);
    return (int)m;
}

}  // namespace

// ===================================================================== C ABI
namespace sbh {

// Host box -> buf[0], then the halo/ghost into buf[1] too (kernels never
// write it).  1D copies only the two ends (pad + halo); 2D/3D copy the whole
// buffer (cheap next to those sweeps).  Stream-ordered, no host sync.
int enqueue_upload(sb_plan* P, const void* host, size_t bytes);
int enqueue_download(sb_plan* P, void* host, size_t bytes);

// The host box as uniformly pitched rows (pitch >= the row's bytes): a NATURAL
// GridBuffer.data whose halo equals the stencil order (core.py:232-373) is one.
int enqueue_upload_pitched(sb_plan* P, const void* host, size_t pitch) {
    if (!P || !host) return fail(SB_ERR_ARG, "NULL argument");
    const size_t rb = (size_t)P->host_row_elems * P->es;
    if (pitch < rb) return fail(SB_ERR_GRID, "host pitch %zu below the row size %zu", pitch, rb);
    if (pitch == rb || P->host_rows == 1) return enqueue_upload(P, host, (size_t)P->host_elems * P->es);
    SB_CUDA(cudaSetDevice(P->device));
    char* dst = reinterpret_cast<char*>(P->buf[0]) + P->host_dst_offset * P->es;
    if (host_is_pinned(host)) {
        SB_CUDA(cudaMemcpy2DAsync(P->buf[1], rb, host, pitch, rb, P->host_rows, cudaMemcpyHostToDevice, P->stream));
    } else {
        const int rc = h2d_pageable_rows(P->buf[1], host, pitch, rb, (size_t)P->host_rows, P->device, P->stream);
        if (rc != SB_OK) return rc;
    }
    SB_CUDA(cudaMemcpy2DAsync(dst, P->px * P->es, P->buf[1], rb, rb, P->host_rows, cudaMemcpyDeviceToDevice, P->stream));
    return finish_upload(P);
}

int enqueue_download_pitched(sb_plan* P, void* host, size_t pitch) {
    if (!P || !host) return fail(SB_ERR_ARG, "NULL argument");
    if (!P->uploaded) return fail(SB_ERR_STATE, "download before upload");
    const size_t rb = (size_t)P->host_row_elems * P->es;
    if (pitch < rb) return fail(SB_ERR_GRID, "host pitch %zu below the row size %zu", pitch, rb);
    if (pitch == rb || P->host_rows == 1) return enqueue_download(P, host, (size_t)P->host_elems * P->es);
    SB_CUDA(cudaSetDevice(P->device));
    const char* src = reinterpret_cast<const char*>(P->buf[P->cur]) + P->host_dst_offset * P->es;
    if (!host_is_pinned(host))
        return d2h_pageable_rows(host, pitch, src, (size_t)P->px * P->es, rb, (size_t)P->host_rows, P->device, P->stream);
    SB_CUDA(cudaMemcpy2DAsync(host, pitch, src, P->px * P->es, rb, P->host_rows, cudaMemcpyDeviceToHost, P->stream));
    return SB_OK;
}

int enqueue_upload(sb_plan* P, const void* host, size_t bytes) {
    if (!P || !host) return fail(SB_ERR_ARG, "NULL argument");
    if (bytes != (size_t)P->host_elems * P->es)
        return fail(SB_ERR_GRID, "host box has %zu bytes, expected %lld", bytes,
                    (long long)(P->host_elems * (int64_t)P->es));
    SB_CUDA(cudaSetDevice(P->device));
    char* dst = reinterpret_cast<char*>(P->buf[0]) + P->host_dst_offset * P->es;
    static const int staged = (int)env_double("SB200_STAGED_UPLOAD", 1);
    const bool pinned = host_is_pinned(host);
    if (!pinned && P->d == 1) {
        // pageable 1D line: contiguous on both sides, through the pinned bounce buffers
        const int rc = h2d_pageable(dst, host, bytes, P->device, P->stream);
        if (rc != SB_OK) return rc;
    } else if (!pinned) {
        // pageable box: the contiguous copy into buf[1] through the bounce buffers (hostxfer.cu:
        // C5 upload 345 -> ~110 ms), then the same device-side re-layout
        const int rc = h2d_pageable(P->buf[1], host, bytes, P->device, P->stream);
        if (rc != SB_OK) return rc;
        SB_CUDA(cudaMemcpy2DAsync(dst, P->px * P->es, P->buf[1], P->host_row_elems * P->es,
                                  P->host_row_elems * P->es, P->host_rows, cudaMemcpyDeviceToDevice, P->stream));
    } else if (P->d >= 2 && staged) {
        // Host -> device as ONE contiguous copy into buf[1] (free until the mirror
        // below), then the pitched re-layout device to device: a pitched H2D copy
        // whose destination rows start off the 128 B grid ran at 37.6 GB/s, a
        // contiguous one at 55.5 (C5 box, pinned host memory)
        SB_CUDA(cudaMemcpyAsync(P->buf[1], host, bytes, cudaMemcpyHostToDevice, P->stream));
        SB_CUDA(cudaMemcpy2DAsync(dst, P->px * P->es, P->buf[1], P->host_row_elems * P->es,
                                  P->host_row_elems * P->es, P->host_rows, cudaMemcpyDeviceToDevice, P->stream));
    } else {
        SB_CUDA(cudaMemcpy2DAsync(dst, P->px * P->es, host, P->host_row_elems * P->es,
                                  P->host_row_elems * P->es, P->host_rows, cudaMemcpyHostToDevice, P->stream));
    }
    return finish_upload(P);
}

// buf[0] holds the uploaded box: mirror the halo/ghost into buf[1] (kernels
// never write it) and make buf[0] current.
int finish_upload(sb_plan* P) {
    if (P->d == 1) {
        const size_t lo = (size_t)P->g.origin, hi = (size_t)(P->g.origin + P->g.n[2]);
        char* b0 = reinterpret_cast<char*>(P->buf[0]);
        char* b1 = reinterpret_cast<char*>(P->buf[1]);
        SB_CUDA(cudaMemcpyAsync(b1, b0, lo * P->es, cudaMemcpyDeviceToDevice, P->stream));
        SB_CUDA(cudaMemcpyAsync(b1 + hi * P->es, b0 + hi * P->es, (P->buf_elems - hi) * P->es,
                                cudaMemcpyDeviceToDevice, P->stream));
    } else {
        SB_CUDA(cudaMemcpyAsync(P->buf[1], P->buf[0], P->buf_elems * P->es, cudaMemcpyDeviceToDevice, P->stream));
    }
    P->cur = 0;
    P->uploaded = true;
    return SB_OK;
}

int enqueue_download(sb_plan* P, void* host, size_t bytes) {
    if (!P || !host) return fail(SB_ERR_ARG, "NULL argument");
    if (!P->uploaded) return fail(SB_ERR_STATE, "download before upload");
    if (bytes != (size_t)P->host_elems * P->es)
        return fail(SB_ERR_GRID, "host box has %zu bytes, expected %lld", bytes,
                    (long long)(P->host_elems * (int64_t)P->es));
    SB_CUDA(cudaSetDevice(P->device));
    const char* src = reinterpret_cast<const char*>(P->buf[P->cur]) + P->host_dst_offset * P->es;
    if (!host_is_pinned(host)) {
        // pageable destination (a numpy array): chunks through the pinned bounce buffers, copied
        // out by a few host threads while the next chunk arrives (C5 download 870-1050 -> ~150 ms);
        // returns with the data in `host`
        const size_t rb = (size_t)P->host_row_elems * P->es;
        if (P->host_rows == 1) {                    // one long line: pieces of 4 MB as rows
            const size_t piece = 4u << 20, full = rb / piece;
            int rc = d2h_pageable_rows(host, piece, src, piece, piece, full, P->device, P->stream);
            if (rc == SB_OK && rb > full * piece)
                rc = d2h_pageable_rows(static_cast<char*>(host) + full * piece, rb - full * piece, src + full * piece,
                                       rb - full * piece, rb - full * piece, 1, P->device, P->stream);
            return rc;
        }
        return d2h_pageable_rows(host, rb, src, (size_t)P->px * P->es, rb, (size_t)P->host_rows, P->device, P->stream);
    }
    SB_CUDA(cudaMemcpy2DAsync(host, P->host_row_elems * P->es, src, P->px * P->es,
                              P->host_row_elems * P->es, P->host_rows, cudaMemcpyDeviceToHost, P->stream));
    return SB_OK;
}

}  // namespace sbh

extern "C" {

const char* sb_last_error(void) { return g_err.c_str(); }
int sb_abi_version(void) { return SB200_ABI_VERSION; }

int sb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

void sb_plan_destroy(sb_plan* P) {
    if (!P) return;
    cudaSetDevice(P->device);
    for (auto e : P->rep_ev) cudaEventDestroy(e);
    for (int i = 0; i < 2; i++)
        if (P->buf[i]) cudaFree(P->buf[i]);
    if (P->d_lin) cudaFree(P->d_lin);
    if (P->d_w) cudaFree(P->d_w);
    if (P->d_counter) cudaFree(P->d_counter);
    if (P->d_trace) cudaFree(P->d_trace);
    if (P->stage) cudaFree(P->stage);
    if (P->tmp) cudaFree(P->tmp);
    for (auto& e : P->sched1d)
        if (e.d_chunks) cudaFree(e.d_chunks);
    for (auto& g : P->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    for (int i = 0; i < 2; i++)
        if (P->ev[i]) cudaEventDestroy(P->ev[i]);
    if (P->fork_ev) cudaEventDestroy(P->fork_ev);
    if (P->join_ev) cudaEventDestroy(P->join_ev);
    if (P->side_stream) cudaStreamDestroy(P->side_stream);
    if (P->own_stream) cudaStreamDestroy(P->own_stream);
    delete P;
}

// Host-side fields of a plan and its kernel choice / fused depth (no device
// resources); shared by sb_plan_create and sb_problem_k.
static int plan_host_setup(sb_plan* P, const sb_problem* prob) {
    P->d = prob->d;
    P->r = prob->r;
    P->shape = prob->shape;
    P->nw = prob->nw;
    P->dtype = prob->dtype;
    P->arith = prob->arith;
    P->kreq = prob->k;
    P->kernel_req = prob->kernel;
    P->device = prob->device;
    P->offsets.assign(prob->offsets, prob->offsets + (size_t)prob->nw * prob->d);
    P->weights.assign(prob->weights, prob->weights + prob->nw);
    for (int a = 0; a < P->d; a++) P->dims[a] = prob->dims[a];
    P->phys_lo = prob->ghost_lo == 0;
    P->phys_hi = prob->ghost_hi == 0;
    P->hlo = P->phys_lo ? P->r : prob->ghost_lo;
    P->hhi = P->phys_hi ? P->r : prob->ghost_hi;
    P->es = (P->dtype == SB_F64) ? 8 : 4;

    // ---- kernel choice
    const int fk = fused_kind(P);
    if (prob->kernel == SB_KERNEL_FUSED && !fk) {
        return fail(SB_ERR_ARG, "no fused kernel for d=%d r=%d shape=%d", prob->d, prob->r, prob->shape);
    }
    if (prob->kernel != SB_KERNEL_GENERIC && fk) {
        P->kind = fk;
        P->k = prob->k > 0 ? prob->k : default_k(fk, P);
        if (!fused_k_ok(P, fk, P->k)) {
            return fail(SB_ERR_ARG, "fused depth k=%d unsupported by the %s kernel", prob->k,
                        fk == KK_FUSED3D ? "3D (1..4)" : fk == KK_FUSED2D ? "2D (1, 2, 4, 8)"
                        : "1D (1, 2, 4, 8, 16; 32, 64 in FMA mode with r*k <= 64)");
        }
    } else {
        P->kind = KK_GENERIC;
        P->k = 1;
    }
    return SB_OK;
}

int sb_problem_k(const sb_problem* prob, int32_t* k) {
    if (!k) return fail(SB_ERR_ARG, "NULL argument");
    int rc = validate_problem(prob);
    if (rc != SB_OK) return rc;
    sb_plan tmp;
    rc = plan_host_setup(&tmp, prob);
    if (rc != SB_OK) return rc;
    *k = tmp.k;
    return SB_OK;
}

int sb_plan_create(sb_plan** out, const sb_problem* prob) {
    if (!out) return fail(SB_ERR_ARG, "plan output pointer is NULL");
    *out = nullptr;
    int rc = validate_problem(prob);
    if (rc != SB_OK) return rc;
    sb_plan* P = new (std::nothrow) sb_plan();
    if (!P) return fail(SB_ERR_NOMEM, "host allocation failed");
    rc = plan_host_setup(P, prob);
    if (rc != SB_OK) {
        delete P;
        return rc;
    }
    if (!(P->phys_lo && P->phys_hi)) {
        // slab: a launch of depth k needs ghost depth >= r*k on slab sides
        if (P->kind != KK_GENERIC && (int64_t)P->r * P->k > std::min(P->phys_lo ? INT32_MAX : P->hlo,
                                                                      P->phys_hi ? INT32_MAX : P->hhi)) {
            delete P;
            return fail(SB_ERR_GRID, "ghost depth must be >= r*k = %d", P->r * P->k);
        }
    }

    // ---- device geometry (canonical z, y, x)
    const int d = P->d, r = P->r;
    sb::Geom& g = P->g;
    const int64_t es = (int64_t)P->es;
    const int64_t line = 128 / es;
    if (d == 1) {
        const int64_t n = P->dims[0];
        const int64_t axl = round_up(std::max(P->hlo, (int64_t)r) + 256, 64);
        P->px = round_up(axl + n + std::max(P->hhi, (int64_t)r) + kRightPad1D, 64);
        g.n[0] = 1; g.n[1] = 1; g.n[2] = n;
        g.sy = P->px; g.sz = P->px;
        g.origin = axl;
        g.slab_axis = 2;
        P->buf_elems = (size_t)P->px;
        P->host_rows = 1;
        P->host_row_elems = P->hlo + n + P->hhi;
        P->host_dst_offset = axl - P->hlo;
    } else {
        const int64_t nx = P->dims[d - 1];
        const int64_t ax = round_up(std::max<int64_t>(r, line), line);
        P->px = round_up(ax + nx + r + line, line);
        g.n[2] = nx;
        if (d == 2) {
            const int64_t ny = P->dims[0];
            g.n[0] = 1; g.n[1] = ny;
            g.sy = P->px;
            const int64_t rows = P->hlo + ny + P->hhi;
            g.sz = rows * P->px;
            g.origin = P->hlo * P->px + ax;
            g.slab_axis = 1;
            P->buf_elems = (size_t)(rows * P->px);
            P->host_rows = rows;
        } else {
            const int64_t nz = P->dims[0], ny = P->dims[1];
            g.n[0] = nz; g.n[1] = ny;
            g.sy = P->px;
            g.sz = (ny + 2 * r) * P->px;
            const int64_t planes = P->hlo + nz + P->hhi;
            g.origin = P->hlo * g.sz + r * g.sy + ax;
            g.slab_axis = 0;
            P->buf_elems = (size_t)(planes * g.sz);
            P->host_rows = planes * (ny + 2 * r);
        }
        P->host_row_elems = nx + 2 * r;
        P->host_dst_offset = ax - r;
    }
    P->host_elems = P->host_rows * P->host_row_elems;

    // ---- device resources
    int ndev = sb_device_count();
    if (ndev <= 0) {
        delete P;
        return fail(SB_ERR_CUDA, "no CUDA device available (sb200 has no CPU fallback)");
    }
    if (P->device < 0 || P->device >= ndev) {
        delete P;
        return fail(SB_ERR_ARG, "device %d out of range (%d visible)", P->device, ndev);
    }
#define SB_CUDA_P(call)                                                                        \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) {                                                               \
            int code_ = (e_ == cudaErrorMemoryAllocation) ? SB_ERR_NOMEM : SB_ERR_CUDA;        \
            fail(code_, "%s failed: %s", #call, cudaGetErrorString(e_));                       \
            sb_plan_destroy(P);                                                                \
            return code_;                                                                      \
        }                                                                                      \
    } while (0)
    SB_CUDA_P(cudaSetDevice(P->device));
    SB_CUDA_P(cudaDeviceGetAttribute(&P->num_sms, cudaDevAttrMultiProcessorCount, P->device));
    SB_CUDA_P(cudaStreamCreateWithFlags(&P->own_stream, cudaStreamNonBlocking));
    P->stream = P->own_stream;
    SB_CUDA_P(cudaStreamCreateWithFlags(&P->side_stream, cudaStreamNonBlocking));
    SB_CUDA_P(cudaEventCreateWithFlags(&P->fork_ev, cudaEventDisableTiming));
    SB_CUDA_P(cudaEventCreateWithFlags(&P->join_ev, cudaEventDisableTiming));
    SB_CUDA_P(cudaEventCreate(&P->ev[0]));
    SB_CUDA_P(cudaEventCreate(&P->ev[1]));
    for (int i = 0; i < 2; i++) {
        SB_CUDA_P(cudaMalloc(&P->buf[i], P->buf_elems * P->es));
        SB_CUDA_P(cudaMemsetAsync(P->buf[i], 0, P->buf_elems * P->es, P->stream));
    }
    // generic tables: linear offsets + weights (in the plan dtype)
    std::vector<int64_t> lin(P->nw);
    for (int i = 0; i < P->nw; i++) {
        int64_t o = 0;
        for (int a = 0; a < d; a++) {
            const int ca = 3 - d + a;  // canonical axis
            const int64_t stride = (ca == 2) ? 1 : (ca == 1 ? g.sy : g.sz);
            o += (int64_t)P->offsets[i * d + a] * stride;
        }
        lin[i] = o;
    }
    SB_CUDA_P(cudaMalloc(&P->d_counter, 4 * sizeof(unsigned int)));
    SB_CUDA_P(cudaMemsetAsync(P->d_counter, 0, 4 * sizeof(unsigned int), P->stream));
    SB_CUDA_P(cudaMalloc(&P->d_lin, sizeof(int64_t) * P->nw));
    SB_CUDA_P(cudaMemcpyAsync(P->d_lin, lin.data(), sizeof(int64_t) * P->nw, cudaMemcpyHostToDevice, P->stream));
    SB_CUDA_P(cudaMalloc(&P->d_w, P->es * P->nw));
    std::vector<float> wf(P->weights.begin(), P->weights.end());
    SB_CUDA_P(cudaMemcpyAsync(P->d_w, P->dtype == SB_F64 ? (const void*)P->weights.data() : (const void*)wf.data(),
                              P->es * P->nw, cudaMemcpyHostToDevice, P->stream));
    // every setup operation is ordered on the plan stream: wait for that stream
    // only (no device-wide sync -- plans of concurrent host threads stay independent)
    SB_CUDA_P(cudaStreamSynchronize(P->stream));
#undef SB_CUDA_P
    *out = P;
    return SB_OK;
}

int sb_host_elems(const sb_plan* P, int64_t* elems) {
    if (!P || !elems) return fail(SB_ERR_ARG, "NULL argument");
    *elems = P->host_elems;
    return SB_OK;
}

int sb_upload(sb_plan* P, const void* host, size_t bytes) {
    const int rc = sbh::enqueue_upload(P, host, bytes);
    if (rc != SB_OK) return rc;
    SB_CUDA(cudaStreamSynchronize(P->stream));
    return SB_OK;
}

int sb_download(sb_plan* P, void* host, size_t bytes) {
    const int rc = sbh::enqueue_download(P, host, bytes);
    if (rc != SB_OK) return rc;
    SB_CUDA(cudaStreamSynchronize(P->stream));
    return SB_OK;
}

int sb_upload_pitched(sb_plan* P, const void* host, size_t pitch_bytes) {
    const int rc = sbh::enqueue_upload_pitched(P, host, pitch_bytes);
    if (rc != SB_OK) return rc;
    SB_CUDA(cudaStreamSynchronize(P->stream));
    return SB_OK;
}

int sb_download_pitched(sb_plan* P, void* host, size_t pitch_bytes) {
    const int rc = sbh::enqueue_download_pitched(P, host, pitch_bytes);
    if (rc != SB_OK) return rc;
    SB_CUDA(cudaStreamSynchronize(P->stream));
    return SB_OK;
}

int sb_upload_async(sb_plan* P, const void* host, size_t bytes) { return sbh::enqueue_upload(P, host, bytes); }

int sb_download_async(sb_plan* P, void* host, size_t bytes) { return sbh::enqueue_download(P, host, bytes); }

int sb_synchronize(sb_plan* P) {
    if (!P) return fail(SB_ERR_ARG, "NULL plan");
    SB_CUDA(cudaSetDevice(P->device));
    SB_CUDA(cudaStreamSynchronize(P->stream));
    SB_CUDA(cudaGetLastError());
    return SB_OK;
}

int sb_launch(sb_plan* P, int64_t steps) {
    if (!P) return fail(SB_ERR_ARG, "NULL plan");
    if (!P->uploaded) return fail(SB_ERR_STATE, "run before upload");
    if (steps < 0) return fail(SB_ERR_ARG, "steps must be >= 0");
    if (steps > max_slab_steps(P))
        return fail(SB_ERR_GRID, "slab plan can advance at most %d steps between exchanges", max_slab_steps(P));
    SB_CUDA(cudaSetDevice(P->device));
    int64_t launches = 0;
    int k_used = 1;
    return run_graphed(P, steps, &launches, &k_used);
}

int sb_launch_repeat(sb_plan* P, int64_t steps, int32_t repeats, int32_t per_sweep_events) {
    if (!P) return fail(SB_ERR_ARG, "NULL plan");
    if (repeats < 0) return fail(SB_ERR_ARG, "repeats must be >= 0");
    SB_CUDA(cudaSetDevice(P->device));
    const int nev = per_sweep_events ? repeats + 1 : 2;
    while ((int)P->rep_ev.size() < nev) {
        cudaEvent_t e = nullptr;
        SB_CUDA(cudaEventCreate(&e));
        P->rep_ev.push_back(e);
    }
    SB_CUDA(cudaEventRecord(P->rep_ev[0], P->stream));
    for (int i = 0; i < repeats; i++) {
        if (per_sweep_events && i > 0) SB_CUDA(cudaEventRecord(P->rep_ev[i], P->stream));
        const int rc = sb_launch(P, steps);
        if (rc != SB_OK) return rc;
    }
    SB_CUDA(cudaEventRecord(P->rep_ev[nev - 1], P->stream));
    P->rep_n = nev - 1;
    return SB_OK;
}

int sb_repeat_times(sb_plan* P, float* sweep_ms, int32_t cap) {
    if (!P || (!sweep_ms && cap > 0)) return fail(SB_ERR_ARG, "NULL argument");
    if (P->rep_n == 0) return fail(SB_ERR_STATE, "no sb_launch_repeat recorded");
    SB_CUDA(cudaSetDevice(P->device));
    SB_CUDA(cudaEventSynchronize(P->rep_ev[P->rep_n]));
    for (int i = 0; i < P->rep_n && i < cap; i++)
        SB_CUDA(cudaEventElapsedTime(&sweep_ms[i], P->rep_ev[i], P->rep_ev[i + 1]));
    return P->rep_n;
}

int sb_launch_range(sb_plan* P, int64_t steps, int64_t lo, int64_t hi, int32_t finish) {
    if (!P) return fail(SB_ERR_ARG, "NULL plan");
    if (!P->uploaded) return fail(SB_ERR_STATE, "run before upload");
    if (P->d < 2) return fail(SB_ERR_ARG, "range launches need d >= 2 (1D slabs exchange r*k points)");
    const int64_t n0 = P->dims[0];
    if (lo < 0 || hi > n0 || lo > hi) return fail(SB_ERR_ARG, "range [%lld, %lld) outside [0, %lld)",
                                                 (long long)lo, (long long)hi, (long long)n0);
    if (steps > max_slab_steps(P))
        return fail(SB_ERR_GRID, "slab plan can advance at most %d steps between exchanges", max_slab_steps(P));
    if (P->kind == KK_GENERIC ? steps != 1 : !fused_k_ok(P, P->kind, (int)steps))
        return fail(SB_ERR_ARG, "range launch depth %lld unsupported by the plan's kernel", (long long)steps);
    SB_CUDA(cudaSetDevice(P->device));
    P->zr_lo = lo;
    P->zr_hi = hi;
    int rc = SB_OK;
    if (hi > lo || finish) {
        const bool fma = P->arith == SB_ARITH_FMA;
        if (hi > lo) {
            if (P->dtype == SB_F64)
                rc = fma ? launch_range_t<double, true>(P, (int)steps, finish) : launch_range_t<double, false>(P, (int)steps, finish);
            else
                rc = fma ? launch_range_t<float, true>(P, (int)steps, finish) : launch_range_t<float, false>(P, (int)steps, finish);
        } else {
            P->cur ^= 1;   // empty last part: just complete the step
        }
    }
    P->zr_lo = 0;
    P->zr_hi = -1;
    return rc;
}

}  // extern "C"

// ---- streamed host-to-host sweep -----------------------------------------
//
// Host box in, `steps` steps, host box out, with the transfers overlapped with
// the sweep itself (3D whole-grid plans).  The grid is cut into B blocks of
// planes along z.  Launch j of the sweep (depth k_j, reach G_j = r k_j) runs
// block by block on ranges shifted down by S_j = G_0 + .. + G_{j-1}:
//     (j, b) computes planes [z_b - S_j, z_{b+1} - S_j)      (clipped to [0, n),
//                                                             the last block up to n)
// so it reads level-j planes up to z_{b+1} - S_j + G_j <= z_{b+1} - S_{j-1}, the end of
// what (j-1, b) produced (depths never increase), and down to planes block b-1
// produced earlier in the stream.  All launches of block b can therefore run as
// soon as the upload has passed plane z_{b+1} + G_0, and block b's final planes
// [z_b - S_{L-1}, z_{b+1} - S_{L-1}) can travel back while later blocks compute.
// Two ping-pong buffers suffice: (j, b) overwrites planes below z_{b+1} - S_j of
// the buffer that later blocks read from z_{b'} - S_j (b' > b) upwards.  Every
// launch is the plan's ordinary range launch, so the result is bit-identical to
// upload + run + download (tests/test_stream_sweep.py).
namespace {

struct StreamRes {   // per-call CUDA objects, released on every exit path
    cudaStream_t up = nullptr, down = nullptr;
    std::vector<cudaEvent_t> ev;
    bool locked = false;
    ~StreamRes() {
        for (auto e : ev) cudaEventDestroy(e);
        if (up) cudaStreamDestroy(up);
        if (down) cudaStreamDestroy(down);
        if (locked) sbh::xfer_release();
    }
    int event(cudaEvent_t* e) {
        SB_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        ev.push_back(*e);
        return SB_OK;
    }
};

template <typename T, bool FMA>
int stream_sweep_t(sb_plan* P, const char* in, size_t in_pitch, char* out, size_t out_pitch,
                   const std::vector<int>& ks, int nblocks) {
    const int64_t n = P->dims[0], r = P->r;
    const size_t rb = (size_t)P->host_row_elems * P->es;
    const int64_t R = P->host_rows / (n + 2 * r);              // rows per plane
    const size_t dpitch = (size_t)P->px * P->es;
    const int L = (int)ks.size();
    std::vector<int64_t> S(L + 1, 0);
    for (int j = 0; j < L; j++) S[j + 1] = S[j] + r * ks[j];
    StreamRes res;
    // pinned host memory is read / written by the copy engines directly; pageable memory goes
    // through the bounce buffers with host copy threads (hostxfer.cu)
    const bool pin_in = sbh::host_is_pinned(in), pin_out = sbh::host_is_pinned(out);
    void *bup[2] = {nullptr, nullptr}, *bdn[2] = {nullptr, nullptr};
    size_t chunk = (size_t)32 << 20;
    int rc = SB_OK;
    if (!pin_in || !pin_out) {
        rc = sbh::xfer_acquire(P->device, bup, bdn, &chunk);
        if (rc != SB_OK) return rc;
        res.locked = true;
    }
    SB_CUDA(cudaStreamCreateWithFlags(&res.up, cudaStreamNonBlocking));
    SB_CUDA(cudaStreamCreateWithFlags(&res.down, cudaStreamNonBlocking));
    const int64_t rows = P->host_rows;
    const int64_t rpc = std::max<int64_t>(1, (int64_t)(chunk / rb));
    const int64_t nchunks = (rows + rpc - 1) / rpc;
    cudaEvent_t start_ev, up_slot[2], dn_slot[2];
    if ((rc = res.event(&start_ev)) != SB_OK) return rc;
    for (int i = 0; i < 2; i++)
        if ((rc = res.event(&up_slot[i])) != SB_OK || (rc = res.event(&dn_slot[i])) != SB_OK) return rc;
    // the buffers may still be in use by earlier work on the plan stream
    SB_CUDA(cudaEventRecord(start_ev, P->stream));
    SB_CUDA(cudaStreamWaitEvent(res.up, start_ev, 0));
    char* b0 = reinterpret_cast<char*>(P->buf[0]) + P->host_dst_offset * P->es;
    char* b1 = reinterpret_cast<char*>(P->buf[1]) + P->host_dst_offset * P->es;

    // blocks and what each needs / yields (host plane index = interior plane + r)
    std::vector<int64_t> zb(nblocks + 1);
    for (int b = 0; b <= nblocks; b++) zb[b] = n * b / nblocks;
    auto need_rows = [&](int b) {       // upload progress block b waits for
        const int64_t planes = b == nblocks - 1 ? n + 2 * r : std::min<int64_t>(n + 2 * r, zb[b + 1] + r * ks[0] + r);
        return planes * R;
    };
    auto final_hi = [&](int b) {        // host planes [.., this) are final once block b is done
        if (b == nblocks - 1) return n + 2 * r;
        const int64_t f = std::min<int64_t>(n, std::max<int64_t>(0, zb[b + 1] - S[L - 1]));
        return f > 0 ? f + r : (int64_t)0;
    };

    struct Dl { int64_t r0, r1; cudaEvent_t after; };   // download row ranges, in order (`after`: the block's kernels)
    std::vector<Dl> dlq;                // (guarded by dl_mu: the downloader thread consumes it)
    std::mutex dl_mu;
    std::condition_variable dl_cv;
    bool dl_closed = false;
    size_t dl_issued = 0, dl_drained = 0;
    int64_t dl_planes = 0;              // host planes queued so far
    int dslot_issue = 0, dslot_drain = 0;
    int next_block = 0;
    const int final_buf = L & 1;

    auto enqueue_block = [&](int b, cudaEvent_t uploaded) -> int {
        SB_CUDA(cudaStreamWaitEvent(P->stream, uploaded, 0));
        for (int j = 0; j < L; j++) {
            const int64_t lo = b == 0 ? 0 : std::min<int64_t>(n, std::max<int64_t>(0, zb[b] - S[j]));
            const int64_t hi = b == nblocks - 1 ? n : std::min<int64_t>(n, std::max<int64_t>(0, zb[b + 1] - S[j]));
            if (hi <= lo) continue;
            P->cur = j & 1;
            P->zr_lo = lo;
            P->zr_hi = hi;
            int64_t launches = 0;
            const int rc2 = launch_one<T, FMA>(P, ks[j], 0, &launches, false);
            if (rc2 != SB_OK) return rc2;
        }
        cudaEvent_t done;
        int rc2 = res.event(&done);
        if (rc2 != SB_OK) return rc2;
        SB_CUDA(cudaEventRecord(done, P->stream));
        const int64_t hp = final_hi(b);
        if (hp > dl_planes) {
            {
                std::lock_guard<std::mutex> g(dl_mu);
                for (int64_t r0 = dl_planes * R; r0 < hp * R; r0 += rpc)
                    dlq.push_back({r0, std::min(r0 + rpc, hp * R), r0 == dl_planes * R ? done : nullptr});
            }
            dl_cv.notify_one();
            dl_planes = hp;
        }
        return SB_OK;
    };
    // The downloader thread: issues queued D2H chunks into the two bounce slots and copies
    // finished ones out to the caller's array, until the queue is closed and empty.  (One
    // thread feeding both directions measured no better than the plain sequence.)
    int dl_rc = SB_OK;
    auto downloader = [&]() {
        if (cudaSetDevice(P->device) != cudaSuccess) {
            dl_rc = SB_ERR_CUDA;
            return;
        }
        for (;;) {
            size_t avail;
            {
                std::unique_lock<std::mutex> g(dl_mu);
                dl_cv.wait(g, [&] { return dl_closed || dlq.size() > dl_issued || dl_issued > dl_drained; });
                avail = dlq.size();
                if (dl_closed && dl_drained == avail) return;
            }
            while (dl_issued < avail && (pin_out || dl_issued - dl_drained < 2)) {
                Dl d;
                {
                    std::lock_guard<std::mutex> g(dl_mu);
                    d = dlq[dl_issued];
                }
                const char* src = reinterpret_cast<const char*>(P->buf[final_buf]) + P->host_dst_offset * P->es +
                                  (size_t)d.r0 * dpitch;
                if (pin_out) {          // straight into the caller's rows; the stream is synchronised at the end
                    if ((d.after && cudaStreamWaitEvent(res.down, d.after, 0) != cudaSuccess) ||
                        cudaMemcpy2DAsync(out + (size_t)d.r0 * out_pitch, out_pitch, src, dpitch, rb, (size_t)(d.r1 - d.r0),
                                          cudaMemcpyDeviceToHost, res.down) != cudaSuccess) {
                        dl_rc = SB_ERR_CUDA;
                        return;
                    }
                    dl_issued++;
                    dl_drained++;
                    continue;
                }
                if ((d.after && cudaStreamWaitEvent(res.down, d.after, 0) != cudaSuccess) ||
                    cudaMemcpy2DAsync(bdn[dslot_issue], rb, src, dpitch, rb, (size_t)(d.r1 - d.r0), cudaMemcpyDeviceToHost,
                                      res.down) != cudaSuccess ||
                    cudaEventRecord(dn_slot[dslot_issue], res.down) != cudaSuccess) {
                    dl_rc = SB_ERR_CUDA;
                    return;
                }
                dslot_issue ^= 1;
                dl_issued++;
            }
            if (dl_drained < dl_issued) {
                if (cudaEventSynchronize(dn_slot[dslot_drain]) != cudaSuccess) {
                    dl_rc = SB_ERR_CUDA;
                    return;
                }
                Dl d;
                {
                    std::lock_guard<std::mutex> g(dl_mu);
                    d = dlq[dl_drained];
                }
                sbh::parallel_copy_rows(out + (size_t)d.r0 * out_pitch, out_pitch,
                                        static_cast<const char*>(bdn[dslot_drain]), rb, rb, (size_t)(d.r1 - d.r0), pin_in ? 1 : 2);
                dslot_drain ^= 1;
                dl_drained++;
            }
        }
    };
    std::thread dl_thread(downloader);
    auto finish_downloads = [&]() {     // close the queue and wait for the thread (every exit path)
        {
            std::lock_guard<std::mutex> g(dl_mu);
            dl_closed = true;
        }
        dl_cv.notify_one();
        if (dl_thread.joinable()) dl_thread.join();
    };
    struct Joiner {
        decltype(finish_downloads)& f;
        ~Joiner() { f(); }
    } joiner{finish_downloads};

    // ---- upload chunks; blocks are enqueued as their planes arrive
    for (int64_t c = 0; c < nchunks; c++) {
        const int slot = (int)(c & 1);
        const int64_t r0 = c * rpc, nr = std::min(rpc, rows - r0);
        if (pin_in) {
            SB_CUDA(cudaMemcpy2DAsync(b0 + (size_t)r0 * dpitch, dpitch, in + (size_t)r0 * in_pitch, in_pitch, rb, (size_t)nr,
                                      cudaMemcpyHostToDevice, res.up));
        } else {
            SB_CUDA(cudaEventSynchronize(up_slot[slot]));
            sbh::parallel_copy_rows(static_cast<char*>(bup[slot]), rb, in + (size_t)r0 * in_pitch, in_pitch, rb, (size_t)nr,
                                    pin_out ? 1 : 2);
            SB_CUDA(cudaMemcpy2DAsync(b0 + (size_t)r0 * dpitch, dpitch, bup[slot], rb, rb, (size_t)nr,
                                      cudaMemcpyHostToDevice, res.up));
            SB_CUDA(cudaEventRecord(up_slot[slot], res.up));
        }
        // the halo / ghost cells live in both buffers (kernels never write them)
        SB_CUDA(cudaMemcpy2DAsync(b1 + (size_t)r0 * dpitch, dpitch, b0 + (size_t)r0 * dpitch, dpitch, rb, (size_t)nr,
                                  cudaMemcpyDeviceToDevice, res.up));
        const int64_t have = r0 + nr;
        if (next_block < nblocks && have >= need_rows(next_block)) {
            cudaEvent_t uploaded;
            if ((rc = res.event(&uploaded)) != SB_OK) return rc;
            SB_CUDA(cudaEventRecord(uploaded, res.up));
            while (next_block < nblocks && have >= need_rows(next_block))
                if ((rc = enqueue_block(next_block++, uploaded)) != SB_OK) return rc;
        }
    }
    P->uploaded = true;
    finish_downloads();
    if (dl_rc != SB_OK) return fail(dl_rc, "streamed download failed: %s", cudaGetErrorString(cudaGetLastError()));
    SB_CUDA(cudaStreamSynchronize(res.down));
    P->cur = final_buf;
    P->zr_lo = 0;
    P->zr_hi = -1;
    SB_CUDA(cudaStreamSynchronize(P->stream));
    SB_CUDA(cudaGetLastError());
    return SB_OK;
}

}  // namespace

extern "C" {

int sb_sweep_host(sb_plan* P, const void* host_in, size_t in_pitch, void* host_out, size_t out_pitch, int64_t steps) {
    if (!P || !host_in || !host_out) return fail(SB_ERR_ARG, "NULL argument");
    if (steps < 0) return fail(SB_ERR_ARG, "steps must be >= 0");
    const size_t rb = (size_t)P->host_row_elems * P->es;
    if (in_pitch == 0) in_pitch = rb;
    if (out_pitch == 0) out_pitch = rb;
    if (in_pitch < rb || out_pitch < rb) return fail(SB_ERR_GRID, "host pitch below the row size %zu", rb);
    SB_CUDA(cudaSetDevice(P->device));
    // the launch sequence run_steps would issue
    std::vector<int> ks;
    if (P->kind == KK_GENERIC) {
        if (steps <= 4096) ks.assign((size_t)steps, 1);      // (longer: the plain path below)
    } else {
        for (int64_t done = 0; done < steps;) {
            const int kk = (steps - done >= P->k) ? P->k : largest_fused_k(P->kind, steps - done, P->k);
            ks.push_back(kk);
            done += kk;
        }
    }
    // Pageable memory: opt-in (SB200_STREAM_SWEEP=1, read per call).  Measured on the C5 box
    // 320-335 vs 347 ms per call with 8 blocks, on C4 (T = 200: 100 launches + their shell
    // kernels per block) 168-202 vs 133 ms -- the host copies (the box crosses the CPU twice)
    // bound the call, not the missing overlap.
    const int nblocks_env = (int)env_double("SB200_STREAM_BLOCKS", 8);
    // With PINNED memory on both sides there are no host copies and the streamed form is the
    // default when the sweep is few launches (SB200_STREAM_SWEEP unset; 0 / 1 force it).
    const int mode = (int)env_double("SB200_STREAM_SWEEP", -1);
    const bool enabled = mode > 0 || (mode < 0 && ks.size() * (size_t)nblocks_env <= 512 &&
                                      sbh::host_is_pinned(host_in) && sbh::host_is_pinned(host_out));

    const int64_t n = P->dims[0];
    const int64_t shift = ks.empty() ? 0 : (int64_t)P->r * (steps - ks.back());
    const int nblocks = (int)std::max<int64_t>(1, std::min<int64_t>(nblocks_env, n / std::max<int64_t>(1, 4 * P->r * (ks.empty() ? 1 : ks[0]))));
    const bool streamed = enabled && P->d == 3 && P->phys_lo && P->phys_hi && !ks.empty() && nblocks >= 2 &&
                          n >= 2 * shift && (size_t)P->host_elems * P->es >= ((size_t)64 << 20) &&
                          P->host_rows % (n + 2 * P->r) == 0;
    if (!streamed) {
        int rc = sbh::enqueue_upload_pitched(P, host_in, in_pitch);
        if (rc != SB_OK) return rc;
        rc = sb_launch(P, steps);
        if (rc != SB_OK) return rc;
        rc = sbh::enqueue_download_pitched(P, host_out, out_pitch);
        if (rc != SB_OK) return rc;
        SB_CUDA(cudaStreamSynchronize(P->stream));
        return SB_OK;
    }
    const bool fma = P->arith == SB_ARITH_FMA;
    const char* in = static_cast<const char*>(host_in);
    char* out = static_cast<char*>(host_out);
    if (P->dtype == SB_F64)
        return fma ? stream_sweep_t<double, true>(P, in, in_pitch, out, out_pitch, ks, nblocks)
                   : stream_sweep_t<double, false>(P, in, in_pitch, out, out_pitch, ks, nblocks);
    return fma ? stream_sweep_t<float, true>(P, in, in_pitch, out, out_pitch, ks, nblocks)
               : stream_sweep_t<float, false>(P, in, in_pitch, out, out_pitch, ks, nblocks);
}

int sb_step_box(sb_plan* P, const int64_t* lo, const int64_t* hi) {
    if (!P || !lo || !hi) return fail(SB_ERR_ARG, "NULL argument");
    if (!P->uploaded) return fail(SB_ERR_STATE, "run before upload");
    if (!(P->phys_lo && P->phys_hi)) return fail(SB_ERR_GRID, "sb_step_box needs a whole-grid plan (no ghost sides)");
    sb::Box3 b;
    for (int a = 0; a < 3; a++) {
        b.base[a] = 0;
        b.ext[a] = 1;
    }
    for (int a = 0; a < P->d; a++) {
        const int ca = 3 - P->d + a;   // canonical axis
        if (lo[a] < 0 || hi[a] > P->dims[a])
            return fail(SB_ERR_GRID, "range (%lld, %lld) outside axis %d of extent %lld", (long long)lo[a],
                        (long long)hi[a], a, (long long)P->dims[a]);
        b.base[ca] = lo[a];
        b.ext[ca] = std::max<int64_t>(0, hi[a] - lo[a]);
    }
    SB_CUDA(cudaSetDevice(P->device));
    const bool fma = P->arith == SB_ARITH_FMA;
    int rc;
    if (P->dtype == SB_F64) {
        auto src = reinterpret_cast<const double*>(P->buf[P->cur]);
        auto dst = reinterpret_cast<double*>(P->buf[P->cur ^ 1]);
        rc = fma ? launch_generic_box<double, true>(P, src, dst, b)
                 : launch_generic_box<double, false>(P, src, dst, b);
    } else {
        auto src = reinterpret_cast<const float*>(P->buf[P->cur]);
        auto dst = reinterpret_cast<float*>(P->buf[P->cur ^ 1]);
        rc = fma ? launch_generic_box<float, true>(P, src, dst, b)
                 : launch_generic_box<float, false>(P, src, dst, b);
    }
    if (rc != SB_OK) return rc;
    P->cur ^= 1;
    P->kernels_launched++;
    P->last_kernel = "generic_step_kernel";
    SB_CUDA(cudaStreamSynchronize(P->stream));
    return SB_OK;
}

int sb_run(sb_plan* P, int64_t steps, sb_timing* t) {
    if (!P) return fail(SB_ERR_ARG, "NULL plan");
    if (!P->uploaded) return fail(SB_ERR_STATE, "run before upload");
    if (steps < 0) return fail(SB_ERR_ARG, "steps must be >= 0");
    if (steps > max_slab_steps(P))
        return fail(SB_ERR_GRID, "slab plan can advance at most %d steps between exchanges", max_slab_steps(P));
    SB_CUDA(cudaSetDevice(P->device));
    int64_t launches = 0;
    int k_used = 1;
    const int64_t kernels_before = P->kernels_launched;
    SB_CUDA(cudaEventRecord(P->ev[0], P->stream));
    int rc = run_graphed(P, steps, &launches, &k_used);
    if (rc != SB_OK) return rc;
    SB_CUDA(cudaEventRecord(P->ev[1], P->stream));
    SB_CUDA(cudaEventSynchronize(P->ev[1]));
    SB_CUDA(cudaGetLastError());
    if (P->d_trace && getenv("SB200_TRACE")) {  // debug: last launch's per-chunk trace
        std::vector<unsigned long long> h((size_t)4 * P->trace_n);
        SB_CUDA(cudaMemcpy(h.data(), P->d_trace, h.size() * 8, cudaMemcpyDeviceToHost));
        if (FILE* f = fopen(getenv("SB200_TRACE"), "wb")) {
            fwrite(h.data(), 8, h.size(), f);
            fclose(f);
        }
    }
    if (t) {
        float ms = 0.f;
        SB_CUDA(cudaEventElapsedTime(&ms, P->ev[0], P->ev[1]));
        t->device_ms = ms;
        t->kernel_ms = ms;
        t->launches = P->kernels_launched - kernels_before;
        int64_t pts = 1;
        for (int a = 0; a < P->d; a++) pts *= P->dims[a];
        t->point_updates = pts * steps;
        t->k_used = k_used;
        t->reserved = 0;
        std::snprintf(t->kernel_name, sizeof(t->kernel_name), "%s", kernel_name(P));
    }
    return SB_OK;
}

int sb_set_stream(sb_plan* P, void* stream) {
    if (!P) return fail(SB_ERR_ARG, "NULL plan");
    P->stream = stream ? reinterpret_cast<cudaStream_t>(stream) : P->own_stream;
    return SB_OK;
}

int sb_device_view(const sb_plan* P, int which, void** base, int64_t* origin, int64_t strides[3]) {
    if (!P || !base || !origin || !strides) return fail(SB_ERR_ARG, "NULL argument");
    if (which != 0 && which != 1) return fail(SB_ERR_ARG, "which must be 0 (current) or 1 (other)");
    *base = P->buf[which == 0 ? P->cur : P->cur ^ 1];
    *origin = P->g.origin;
    strides[0] = strides[1] = strides[2] = 0;
    if (P->d == 1) {
        strides[0] = 1;
    } else if (P->d == 2) {
        strides[0] = P->g.sy;
        strides[1] = 1;
    } else {
        strides[0] = P->g.sz;
        strides[1] = P->g.sy;
        strides[2] = 1;
    }
    return SB_OK;
}

int sb_kernel_count(const sb_plan* P, int64_t* count) {
    if (!P || !count) return fail(SB_ERR_ARG, "NULL argument");
    *count = P->kernels_launched;
    return SB_OK;
}

int sb_plan_k(const sb_plan* P, int32_t* k) {
    if (!P || !k) return fail(SB_ERR_ARG, "NULL argument");
    *k = P->k;
    return SB_OK;
}

}  // extern "C"
