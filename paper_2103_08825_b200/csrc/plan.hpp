// Host-side plan state shared by the C-ABI unit (sb200.cu) and the kernel
// launch units (launch1d.cu, launch2d.cu, launch3d.cu), compiled separately.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "../../include/sb200.h"
#include "common.cuh"

namespace sbh {

int fail(int code, const char* fmt, ...);
double env_double(const char* name, double dflt);   // development tuning knobs

#define SB_CUDA(call)                                                                     \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(SB_ERR_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));     \
    } while (0)

inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

constexpr int64_t kRightPad1D = 4096 + 1024;  // >= last-chunk overrun (< 32*Q) + lead + RK + Q
constexpr int kMaxS1D = 4096;

enum KernelKind { KK_GENERIC = 1, KK_FUSED1D = 2, KK_FUSED3D = 3, KK_FUSED2D = 4 };

struct Sched1D {
    int K = 0;
    int blocks = 0;
    int nchunks = 0;   // interior chunks
    int nedge = 0;     // boundary chunks (edge kernel)
    void* d_chunks = nullptr;   // sb::Chunk1D[nchunks + nedge]
    int64_t comp_lo = 0, comp_hi = 0;   // composed-stencil range (K < 0 entries)
    std::vector<double> cw;             // composed weights
};


struct Chunk1DHost {
    int64_t start;
    int32_t S;
    int32_t pad;
};

}  // namespace sbh

// A captured sweep: the launch sequence of `steps` steps starting from
// buffer `cur0`, replayed with one cudaGraphLaunch (sb200.cu run_graphed).
struct SweepGraph {
    int64_t steps = 0;
    int cur0 = 0, cur1 = 0;
    int hits = 0;
    cudaGraphExec_t exec = nullptr;
    bool failed = false;
    int64_t kernels = 0, launches = 0;
    int k_used = 1;
    const char* last_kernel = nullptr;
};

struct sb_plan {
    int d = 0, r = 0, shape = 0, nw = 0, dtype = 0, arith = 0, kreq = 0, kernel_req = 0;
    int device = 0;
    std::vector<int32_t> offsets;
    std::vector<double> weights;
    int64_t dims[3] = {1, 1, 1};  // interior, slowest first (first d used)
    int64_t hlo = 0, hhi = 0;     // axis-0 halo/ghost depth on each side
    bool phys_lo = true, phys_hi = true;
    size_t es = 8;
    sb::Geom g{};                 // canonical 3D geometry of the device buffers
    int64_t px = 0;
    size_t buf_elems = 0;
    void* buf[2] = {nullptr, nullptr};
    int cur = 0;
    bool uploaded = false;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t side_stream = nullptr;            // boundary work forked from `stream`
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int64_t* d_lin = nullptr;
    void* d_w = nullptr;
    unsigned int* d_counter = nullptr;  // work queue of the persistent kernels
    std::vector<sbh::Sched1D> sched1d;
    std::vector<SweepGraph> graphs;       // captured sweeps (see run_graphed)
    std::vector<cudaEvent_t> rep_ev;      // sb_launch_repeat: event before each sweep (+1 after)
    int rep_n = 0;                        // sweeps recorded by the last sb_launch_repeat
    CUtensorMap tmap[8][2];                // TMA descriptors [geometry][buffer] (3D; 2, 3: composed; 4-6: box3d)
    bool tmap_ok[8] = {false, false, false, false, false, false, false, false};
    void* tmp = nullptr;                   // scratch grid of the separable composed 2D path
    void* stage = nullptr;                 // reference-storage staging rows (sb_upload_storage)
    size_t stage_bytes = 0;
    int64_t stage_row_elems = 0;
    unsigned long long* d_trace = nullptr;  // debug trace (SB200_TRACE)
    int trace_n = 0;
    int kind = sbh::KK_GENERIC;
    int64_t kernels_launched = 0;   // every kernel launch (sb_kernel_count)
    const char* last_kernel = nullptr;   // main kernel of the last launch (sb_timing.kernel_name)
    int k = 1;
    // output range on the slowest axis of the next launch ([zr_lo, zr_hi); zr_hi < 0:
    // the whole interior) -- sb_launch_range, for exchange/compute overlap in slabs
    int64_t zr_lo = 0, zr_hi = -1;
    int num_sms = 148;
    // host-box geometry
    int64_t host_rows = 0, host_row_elems = 0, host_elems = 0;
    int64_t host_dst_offset = 0;  // device element offset of host element 0
};


// Kernel-family launch entry points (one launch of k fused levels from
// buf[src_idx] into buf[src_idx ^ 1]); each dispatches on dtype/arith.
namespace sbh {
int launch_fused1d(sb_plan* P, int src_idx, int k);
int launch_fused2d(sb_plan* P, int src_idx, int k);
int launch_fused3d(sb_plan* P, int src_idx, int k);
int make_tensor_maps(sb_plan* P, int geo, int box_h);
int finish_upload(sb_plan* P);   // buf[0] uploaded: mirror halo/ghost into buf[1], make buf[0] current
// hostxfer.cu: transfers for pageable host memory through pinned bounce buffers
bool host_is_pinned(const void* p);
int h2d_pageable(void* dst, const void* src, size_t bytes, int device, cudaStream_t st);
int h2d_pageable_rows(void* dst, const void* host, size_t host_pitch, size_t row_bytes, size_t rows, int device,
                      cudaStream_t st);
int d2h_pageable_rows(void* host, size_t host_pitch, const void* src, size_t src_pitch, size_t row_bytes, size_t rows,
                      int device, cudaStream_t st);
void parallel_copy_rows(char* dst, size_t dp, const char* src, size_t sp, size_t row_bytes, size_t rows, int share = 1);
int xfer_acquire(int device, void* up[2], void* down[2], size_t* chunk_bytes);
void xfer_release();
bool sep2d_ok(const sb_plan* P, int k);   // launch2d.cu: separable composed 2D path serves depth k
inline int64_t range_lo(const sb_plan* P) { return P->zr_hi >= 0 ? P->zr_lo : 0; }
inline int64_t range_hi(const sb_plan* P) { return P->zr_hi >= 0 ? P->zr_hi : P->dims[0]; }

// The composed 1D path (compose1d.cuh) serves depth k when the arithmetic is
// FMA, R*k <= 64 taps each side, the halo is a whole number of 16 B vectors
// and the line is long enough for the boundary windows.  `min_k` is 16 by
// default (the level-by-level kernel wins below); depths 32 and 64 exist only
// on this path.
inline bool compose1d_ok(const sb_plan* P, int k, int min_k) {
    const int vec = P->dtype == SB_F64 ? 2 : 4;
    return P->d == 1 && P->arith == SB_ARITH_FMA && k >= min_k && P->r * k <= 64 &&
           (P->r * k) % vec == 0 && P->dims[0] >= (int64_t)12288 * 8 / (int64_t)P->es;
}
}  // namespace sbh
