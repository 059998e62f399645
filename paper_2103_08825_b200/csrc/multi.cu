// Single-process multi-GPU sweep: one grid in, one grid out, split into
// slowest-axis slabs over several devices of one node (SURVEY §5, §8(b)/(e):
// the grid-in/grid-out drop-in with `ngpu`).
//
// The reference has no distributed execution (its only parallelism is the
// tile thread pool, tiling.py:372-417); this is the B200 runtime around the
// slab plans of sb200.cu:
//   * slab i owns global interior planes [start_i, end_i) (balanced split),
//     with G = r*k ghost planes on every side facing another slab, so a fused
//     launch of k steps leaves exactly the slab valid (overlapped ghost-zone
//     recompute, no exchange inside a launch);
//   * 2D/3D, per interval of k steps and per slab, all asynchronous:
//       main stream  : edge planes [0, G) and [n-G, n) (range launches into
//                      the other buffer) -> event E_i -> interior [G, n-G)
//                      (completes the step)
//       copy stream  : waits E_i and the neighbours' E (their previous step has
//                      stopped reading the ghost planes about to be
//                      overwritten), then peer-copies the new edge planes into
//                      the neighbours' ghost planes over NVLink
//                      (cudaMemcpyPeerAsync; peer access enabled when the
//                      devices allow it) -> event X_i
//     the next interval's launches of slab i wait on X_{i-1} and X_{i+1};
//     the copies overlap the interior launches;
//   * 1D: the r*k-point exchange runs after each whole launch (latency only).
// Per-point arithmetic is independent of the decomposition, so the result is
// bit-identical to one device (EXACT) -- tested, including several slabs on
// one device (the same code path: peer copies within a device are plain
// device-to-device copies).
#include <cstdio>
#include <cstring>
#include <vector>

#include "plan.hpp"

struct sb_multi {
    int d = 0, r = 0, k = 1, ngpu = 0;
    size_t es = 8;
    int64_t dims[3] = {1, 1, 1};
    int64_t host_plane = 0;          // elements of one global host-box plane (axis 0)
    std::vector<sb_plan*> plans;
    std::vector<int64_t> start, end;
    std::vector<int> dev;
    std::vector<cudaStream_t> copy;  // per slab, on the slab's device
    std::vector<cudaEvent_t> edge_ev, xfer_ev, t0, t1;
    std::vector<char> stage;         // host staging of one local box (download)
    bool pending_xfer = false;       // the last interval's copies feed the next launches
};

namespace {
using sbh::fail;

int64_t plane_stride(const sb_plan* P) { return P->d == 1 ? 1 : (P->d == 2 ? P->g.sy : P->g.sz); }

// Device address of local interior plane p (may be negative: ghost planes) of buffer b.
char* plane_ptr(const sb_plan* P, int b, int64_t p) {
    const int64_t st = plane_stride(P);
    const int64_t first = P->d == 1 ? P->g.origin + p : (P->g.origin / st + p) * st;
    return reinterpret_cast<char*>(P->buf[b]) + first * (int64_t)P->es;
}

void destroy(sb_multi* M) {
    if (!M) return;
    for (size_t i = 0; i < M->plans.size(); i++) {
        if (M->plans[i]) {
            cudaSetDevice(M->dev[i]);
            if (i < M->copy.size() && M->copy[i]) cudaStreamDestroy(M->copy[i]);
            for (auto* v : {&M->edge_ev, &M->xfer_ev, &M->t0, &M->t1})
                if (i < v->size() && (*v)[i]) cudaEventDestroy((*v)[i]);
            sb_plan_destroy(M->plans[i]);
        }
    }
    delete M;
}

// Enqueue the ghost exchange after the edge planes of every slab are in buffer
// `b` of each plan (the buffer the current interval writes).
int enqueue_exchange(sb_multi* M, int b) {
    const int g = M->ngpu;
    for (int i = 0; i < g; i++) {
        sb_plan* P = M->plans[i];
        SB_CUDA(cudaSetDevice(M->dev[i]));
        for (int j = i - 1; j <= i + 1; j++)
            if (j >= 0 && j < g) SB_CUDA(cudaStreamWaitEvent(M->copy[i], M->edge_ev[j], 0));
        const int64_t G = (int64_t)M->r * M->k;
        const size_t bytes = (size_t)(G * plane_stride(P)) * P->es;
        if (i > 0) {   // my low edge [0, G) -> slab i-1's high ghosts [n, n+G)
            sb_plan* Q = M->plans[i - 1];
            SB_CUDA(cudaMemcpyPeerAsync(plane_ptr(Q, b, Q->dims[0]), M->dev[i - 1], plane_ptr(P, b, 0), M->dev[i],
                                        bytes, M->copy[i]));
        }
        if (i < g - 1) {   // my high edge [n-G, n) -> slab i+1's low ghosts [-G, 0)
            sb_plan* Q = M->plans[i + 1];
            SB_CUDA(cudaMemcpyPeerAsync(plane_ptr(Q, b, -G), M->dev[i + 1], plane_ptr(P, b, P->dims[0] - G), M->dev[i],
                                        bytes, M->copy[i]));
        }
        SB_CUDA(cudaEventRecord(M->xfer_ev[i], M->copy[i]));
    }
    M->pending_xfer = true;
    return SB_OK;
}

int wait_incoming(sb_multi* M, int i) {
    if (!M->pending_xfer) return SB_OK;
    for (int j = i - 1; j <= i + 1; j += 2)
        if (j >= 0 && j < M->ngpu) SB_CUDA(cudaStreamWaitEvent(M->plans[i]->stream, M->xfer_ev[j], 0));
    return SB_OK;
}

}  // namespace

using sbh::fail;
extern "C" {

int sb_multi_create(sb_multi** out, const sb_problem* prob, int32_t ngpu, const int32_t* devices) {
    if (!out || !prob) return sbh::fail(SB_ERR_ARG, "NULL argument");
    *out = nullptr;
    if (ngpu < 1) return sbh::fail(SB_ERR_ARG, "ngpu must be >= 1");
    int32_t k = 0;
    int rc = sb_problem_k(prob, &k);
    if (rc != SB_OK) return rc;
    const int64_t n0 = prob->dims[0];
    const int64_t G = (int64_t)prob->r * k;
    if (ngpu > 1 && n0 / ngpu < G)
        return sbh::fail(SB_ERR_GRID, "slabs of %lld planes are thinner than the ghost depth %lld",
                         (long long)(n0 / ngpu), (long long)G);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) ndev = 0;
    sb_multi* M = new (std::nothrow) sb_multi();
    if (!M) return sbh::fail(SB_ERR_NOMEM, "host allocation failed");
    M->d = prob->d;
    M->r = prob->r;
    M->k = k;
    M->ngpu = ngpu;
    M->es = prob->dtype == SB_F64 ? 8 : 4;
    for (int a = 0; a < 3; a++) M->dims[a] = a < prob->d ? prob->dims[a] : 1;
    M->host_plane = 1;
    for (int a = 1; a < prob->d; a++) M->host_plane *= prob->dims[a] + 2 * prob->r;
    const int64_t base = n0 / ngpu, extra = n0 % ngpu;
    int64_t pos = 0;
    size_t max_local = 0;
    for (int i = 0; i < ngpu; i++) {
        const int64_t sz = base + (i < extra ? 1 : 0);
        M->start.push_back(pos);
        M->end.push_back(pos + sz);
        pos += sz;
        const int dv = devices ? devices[i] : i;
        if (dv < 0 || dv >= ndev) {
            destroy(M);
            return sbh::fail(SB_ERR_ARG, "device %d out of range (%d visible)", dv, ndev);
        }
        M->dev.push_back(dv);
    }
    for (int i = 0; i < ngpu; i++) {
        sb_problem sp = *prob;
        sp.k = k;
        sp.device = M->dev[i];
        sp.dims[0] = M->end[i] - M->start[i];
        sp.ghost_lo = i > 0 ? (int32_t)G : 0;
        sp.ghost_hi = i < ngpu - 1 ? (int32_t)G : 0;
        sb_plan* P = nullptr;
        rc = sb_plan_create(&P, &sp);
        if (rc != SB_OK) {
            destroy(M);
            return rc;
        }
        M->plans.push_back(P);
        max_local = std::max(max_local, (size_t)P->host_elems * M->es);
        cudaStream_t cs = nullptr;
        cudaEvent_t e[4] = {};
        if (cudaSetDevice(M->dev[i]) != cudaSuccess || cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&e[0], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&e[1], cudaEventDisableTiming) != cudaSuccess || cudaEventCreate(&e[2]) != cudaSuccess ||
            cudaEventCreate(&e[3]) != cudaSuccess) {
            destroy(M);
            return sbh::fail(SB_ERR_CUDA, "stream/event creation failed on device %d", M->dev[i]);
        }
        M->copy.push_back(cs);
        M->edge_ev.push_back(e[0]);
        M->xfer_ev.push_back(e[1]);
        M->t0.push_back(e[2]);
        M->t1.push_back(e[3]);
    }
    // peer access between neighbouring devices (NVLink); a failure only means the
    // copies are staged by the driver
    for (int i = 0; i + 1 < ngpu; i++) {
        const int a = M->dev[i], b = M->dev[i + 1];
        if (a == b) continue;
        int ok = 0;
        if (cudaDeviceCanAccessPeer(&ok, a, b) == cudaSuccess && ok) {
            cudaSetDevice(a);
            cudaDeviceEnablePeerAccess(b, 0);
            cudaSetDevice(b);
            cudaDeviceEnablePeerAccess(a, 0);
            cudaGetLastError();   // "already enabled" is fine
        }
    }
    M->stage.resize(max_local);
    *out = M;
    return SB_OK;
}

void sb_multi_destroy(sb_multi* M) { destroy(M); }

int sb_multi_info(const sb_multi* M, int32_t* ngpu, int32_t* k) {
    if (!M) return sbh::fail(SB_ERR_ARG, "NULL argument");
    if (ngpu) *ngpu = M->ngpu;
    if (k) *k = M->k;
    return SB_OK;
}

int sb_multi_slab(const sb_multi* M, int32_t i, int64_t* start, int64_t* end, int32_t* device) {
    if (!M || i < 0 || i >= M->ngpu) return sbh::fail(SB_ERR_ARG, "bad slab index");
    if (start) *start = M->start[i];
    if (end) *end = M->end[i];
    if (device) *device = M->dev[i];
    return SB_OK;
}

// Global halo-inclusive host box -> every slab (its interior, halo and ghost
// planes are contiguous planes of the global box).
int sb_multi_upload(sb_multi* M, const void* host, size_t bytes) {
    if (!M || !host) return sbh::fail(SB_ERR_ARG, "NULL argument");
    const int64_t planes = M->dims[0] + 2 * M->r;
    const int64_t total = (M->d == 1 ? M->dims[0] + 2 * M->r : planes * M->host_plane);
    if (bytes != (size_t)total * M->es)
        return sbh::fail(SB_ERR_GRID, "host box has %zu bytes, expected %lld", bytes, (long long)(total * (int64_t)M->es));
    const char* h = reinterpret_cast<const char*>(host);
    for (int i = 0; i < M->ngpu; i++) {
        sb_plan* P = M->plans[i];
        const int64_t first = M->start[i] - P->hlo + M->r;   // global box plane of local plane -hlo
        const int rc = sb_upload(P, h + (size_t)(first * M->host_plane) * M->es, (size_t)P->host_elems * M->es);
        if (rc != SB_OK) return rc;
    }
    M->pending_xfer = false;
    return SB_OK;
}

int sb_multi_download(sb_multi* M, void* host, size_t bytes) {
    if (!M || !host) return sbh::fail(SB_ERR_ARG, "NULL argument");
    const int64_t planes = M->dims[0] + 2 * M->r;
    const int64_t total = (M->d == 1 ? M->dims[0] + 2 * M->r : planes * M->host_plane);
    if (bytes != (size_t)total * M->es)
        return sbh::fail(SB_ERR_GRID, "host box has %zu bytes, expected %lld", bytes, (long long)(total * (int64_t)M->es));
    char* h = reinterpret_cast<char*>(host);
    for (int i = 0; i < M->ngpu; i++) {
        sb_plan* P = M->plans[i];
        int rc = sb_download(P, M->stage.data(), (size_t)P->host_elems * M->es);
        if (rc != SB_OK) return rc;
        // interior planes, plus the physical halo planes of the end slabs
        const int64_t lo = (i == 0 ? -M->r : 0), hi = M->end[i] - M->start[i] + (i == M->ngpu - 1 ? M->r : 0);
        const size_t pb = (size_t)M->host_plane * M->es;
        std::memcpy(h + (size_t)(M->start[i] + lo + M->r) * pb, M->stage.data() + (size_t)(lo + P->hlo) * pb,
                    (size_t)(hi - lo) * pb);
    }
    return SB_OK;
}

// Advance every slab `steps` time steps (k per interval; the tail at a smaller
// depth), exchanging ghosts between intervals.  Synchronous; *timing gets the
// max over devices of each device's event time.
int sb_multi_run(sb_multi* M, int64_t steps, sb_timing* t) {
    if (!M) return sbh::fail(SB_ERR_ARG, "NULL argument");
    if (steps < 0) return sbh::fail(SB_ERR_ARG, "steps must be >= 0");
    const int g = M->ngpu;
    const int64_t kernels0 = [&] {
        int64_t s = 0;
        for (auto* P : M->plans) s += P->kernels_launched;
        return s;
    }();
    for (int i = 0; i < g; i++) {
        SB_CUDA(cudaSetDevice(M->dev[i]));
        SB_CUDA(cudaEventRecord(M->t0[i], M->plans[i]->stream));
    }
    const int64_t G = (int64_t)M->r * M->k;
    int64_t done = 0;
    while (done < steps) {
        int kk = (int)std::min<int64_t>(M->k, steps - done);
        if (M->d != 3) {   // 1D/2D fused depths are powers of two (2D separable: 16, 32)
            int p = 1;
            while (p * 2 <= kk) p *= 2;
            kk = p;
        }
        // the first interval after an upload also needs the ghosts of the uploaded state:
        // sb_upload copied the global box including every slab's ghost planes, so none
        if (M->d == 1 || g == 1) {
            for (int i = 0; i < g; i++) {
                int rc = wait_incoming(M, i);
                if (rc != SB_OK) return rc;
                rc = sb_launch(M->plans[i], kk);
                if (rc != SB_OK) return rc;
                SB_CUDA(cudaEventRecord(M->edge_ev[i], M->plans[i]->stream));
            }
            if (g > 1) {
                const int rc = enqueue_exchange(M, M->plans[0]->cur);   // new values: current buffers
                if (rc != SB_OK) return rc;
            }
        } else {
            for (int i = 0; i < g; i++) {
                sb_plan* P = M->plans[i];
                int rc = wait_incoming(M, i);
                if (rc != SB_OK) return rc;
                const int64_t n = P->dims[0];
                int64_t e_lo = i > 0 ? G : 0, e_hi = i < g - 1 ? n - G : n;
                if (e_lo >= e_hi) {   // thin slab: the edges cover it, no separate interior
                    rc = sb_launch_range(P, kk, 0, n, 0);
                } else {
                    if (e_lo > 0) rc = sb_launch_range(P, kk, 0, e_lo, 0);
                    if (rc == SB_OK && e_hi < n) rc = sb_launch_range(P, kk, e_hi, n, 0);
                }
                if (rc != SB_OK) return rc;
                SB_CUDA(cudaSetDevice(M->dev[i]));
                SB_CUDA(cudaEventRecord(M->edge_ev[i], P->stream));
            }
            int rc = enqueue_exchange(M, M->plans[0]->cur ^ 1);   // edges were written to the other buffers
            if (rc != SB_OK) return rc;
            for (int i = 0; i < g; i++) {
                sb_plan* P = M->plans[i];
                const int64_t n = P->dims[0];
                const int64_t lo = i > 0 ? G : 0, hi = i < g - 1 ? n - G : n;
                rc = lo >= hi ? sb_launch_range(P, kk, n, n, 1) : sb_launch_range(P, kk, lo, hi, 1);
                if (rc != SB_OK) return rc;
            }
        }
        done += kk;
    }
    for (int i = 0; i < g; i++) {
        SB_CUDA(cudaSetDevice(M->dev[i]));
        const int rc = wait_incoming(M, i);   // the last copies land before the run returns
        if (rc != SB_OK) return rc;
        SB_CUDA(cudaEventRecord(M->t1[i], M->plans[i]->stream));
    }
    M->pending_xfer = false;
    double ms_max = 0;
    for (int i = 0; i < g; i++) {
        SB_CUDA(cudaSetDevice(M->dev[i]));
        SB_CUDA(cudaEventSynchronize(M->t1[i]));
        float ms = 0.f;
        SB_CUDA(cudaEventElapsedTime(&ms, M->t0[i], M->t1[i]));
        ms_max = std::max(ms_max, (double)ms);
        SB_CUDA(cudaGetLastError());
    }
    if (t) {
        int64_t pts = 1;
        for (int a = 0; a < M->d; a++) pts *= M->dims[a];
        int64_t kernels = 0;
        for (auto* P : M->plans) kernels += P->kernels_launched;
        t->device_ms = ms_max;
        t->kernel_ms = ms_max;
        t->launches = kernels - kernels0;
        t->point_updates = pts * steps;
        t->k_used = M->k;
        t->reserved = 0;
        const char* nm = M->plans[0]->last_kernel ? M->plans[0]->last_kernel : "generic_step_kernel";
        std::snprintf(t->kernel_name, sizeof(t->kernel_name), "%s", nm);
    }
    return SB_OK;
}

}  // extern "C"
