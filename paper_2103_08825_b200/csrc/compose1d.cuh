// K1c -- 1D composed-stencil sweep (FMA mode): K time steps of a
// constant-coefficient (2R+1)-point stencil as ONE (2RK+1)-tap stencil.
//
// Away from physical boundaries K Jacobi steps are the K-fold convolution
// power of the weights (computed on the host in extended precision and
// rounded once), so a launch of depth K costs 2RK+1 FMAs per point instead of
// K(2R+1) -- for C2 (R=2, K=16) 65 instead of 80 -- and, unlike the
// level-by-level pipeline (fused1d.cuh), needs no redundant lead-in work.
// Values whose dependency cone touches a physical halo within K levels
// (distance < R*K from a physical boundary) are produced by the exact
// level-by-level edge kernel instead (fused1d_edge_kernel), so the Dirichlet
// semantics are unchanged.  Used only in FMA arithmetic mode (results within
// the fp64 bar, not bit-identical); EXACT mode keeps the level-by-level path.
//
// Work: uniform tiles of 32*B outputs, claimed by persistent warps from an
// atomic counter.  A warp stages its tile's inputs (32*B + 2RK points) into a
// padded shared buffer with cp.async (one tile ahead), then lane l produces
// outputs l*B..l*B+B-1 with B independent accumulators (ILP B) and writes
// them as coalesced 16 B vectors.
#pragma once
#include "common.cuh"
#include "fused1d.cuh"

namespace sb {

#ifndef SB_C1_COALESCED_STORES
#define SB_C1_COALESCED_STORES 1
#endif
#ifndef SB_C1_B
#define SB_C1_B 8
#endif
constexpr int C1_B = SB_C1_B;     // outputs per lane per tile
constexpr int C1_WARPS = 4;
constexpr int C1_MAXTAPS = 129;  // R*K <= 64

template <typename T>
struct Compose1DParams {
    const T* src;          // interior position 0
    T* dst;
    int64_t lo, hi;        // composed output range [lo, hi)
    int64_t ntiles;
    int32_t total_warps;
    unsigned int* counter; // [2] next tile, [3] retired warps
    int taps;              // 2*R*K + 1
    T c[C1_MAXTAPS];       // composed weights, offset -RK..RK
};

// Shared layout: 16 B chunk c lives at chunk c + c/4 (one pad chunk every
// 64 B) so lane l's window starting at chunk 4l*B/8... reads conflict-free.
template <typename T>
__device__ __forceinline__ int c1_pad(int i) {   // element index -> padded element index
    constexpr int VEC = Vec16<T>::n;
    const int chunk = i / VEC;
    return i + (chunk / 4) * VEC;
}

// Exact level-by-level boundary windows for the composed path: one warp per
// physical side advances the K steps over the window holding the dependency
// cone of the E = RK outputs next to the boundary, with the Dirichlet halo
// fixed at every level (HaloEdges, timejam.py:53-71) and the same
// canonical-order arithmetic as every other kernel.  The window lives in
// registers (lane l holds PER consecutive positions, neighbours arrive by
// shuffles), so a level costs one shuffle round and 2R+1 dependent FMAs --
// the window is on the critical path of short sweeps (C1: 64 levels).
template <typename T, int R>
struct EdgeWindowParams {
    const T* src;      // interior position 0
    T* dst;
    int64_t n;
    int side[2];       // per block: 0 = low side, 1 = high side
    T w[2 * R + 1];
};

template <typename T, int R, int K, bool FMA>
__device__ __forceinline__ void edge_window_body(const EdgeWindowParams<T, R> P, int b, int lane) {
    constexpr int E = R * K;                        // outputs per side
    constexpr int SPAN = 2 * E + R;                 // outputs + dependency cone + halo
    constexpr int PER = (SPAN + 31) / 32 > R ? (SPAN + 31) / 32 : R;
    const bool lo = P.side[b] == 0;
    // low side: window [-R, 2E); high side: [n - 2E, n + R)
    const int64_t first = lo ? -(int64_t)R : P.n - 2 * E;
    T v[PER];
    unsigned fixed = 0;                             // halo positions never change
#pragma unroll
    for (int j = 0; j < PER; j++) {
        const int64_t pos = first + lane * PER + j;
        v[j] = (pos >= -R && pos < P.n + R) ? P.src[pos] : T(0);
        fixed |= (unsigned)(pos < 0 || pos >= P.n) << j;
    }
#pragma unroll 1
    for (int step = 0; step < K; step++) {
        // values beyond the window's two ends are garbage; it spreads R per
        // level, i.e. at most RK positions deep -- never into the outputs
        T left[R], right[R];
#pragma unroll
        for (int q = 0; q < R; q++) {
            left[q] = __shfl_up_sync(0xffffffffu, v[PER - R + q], 1);
            right[q] = __shfl_down_sync(0xffffffffu, v[q], 1);
        }
        T nv[PER];
#pragma unroll
        for (int j = 0; j < PER; j++) {
            T acc = T(0);
#pragma unroll
            for (int t = 0; t <= 2 * R; t++) {
                const int i = j - R + t;
                const T x = i < 0 ? left[R + i] : (i >= PER ? right[i - PER] : v[i]);
                acc = t == 0 ? acc_first<T, FMA>(P.w[0], x) : acc_term<T, FMA>(acc, P.w[t], x);
            }
            nv[j] = ((fixed >> j) & 1) ? v[j] : acc;
        }
#pragma unroll
        for (int j = 0; j < PER; j++) v[j] = nv[j];
    }
    const int out0 = lo ? R : E;                    // window index of the first output
#pragma unroll
    for (int j = 0; j < PER; j++) {
        const int i = lane * PER + j - out0;
        const int64_t pos = first + lane * PER + j;
        if (i >= 0 && i < E && pos >= 0 && pos < P.n) P.dst[pos] = v[j];
    }
}

template <typename T, int R, int K, bool FMA>
__global__ void __launch_bounds__(32)
edge_window_kernel(const EdgeWindowParams<T, R> P) {
    edge_window_body<T, R, K, FMA>(P, blockIdx.x, threadIdx.x);
}

// R > 0: the first `nedge` CTAs run the boundary windows (warp 0 each, exact
// level by level) instead of composed tiles -- one launch per sweep step, no
// side-stream fork/join; scheduled first, so they overlap the composed tiles.
template <typename T, int HALF, int R = 0>   // HALF = R*K
__global__ void __launch_bounds__(C1_WARPS * 32)
compose1d_kernel(const Compose1DParams<T> P, const EdgeWindowParams<T, (R > 0 ? R : 1)> EP = {}, int nedge = 0) {
    // Programmatic dependent launch: this grid may be scheduled while the previous
    // launch on the stream (the previous sweep step, which wrote our input) drains;
    // wait here for it to complete before touching its output or the tile queue.
    // (A no-op when launched without the attribute.)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if constexpr (R > 0) {
        if ((int)blockIdx.x < nedge) {
            if (threadIdx.x < 32) edge_window_body<T, R, HALF / R, true>(EP, blockIdx.x, threadIdx.x);
            return;
        }
    }
    const int bid = (int)blockIdx.x - (R > 0 ? nedge : 0);
    constexpr int VEC = Vec16<T>::n;
    constexpr int TILE = 32 * C1_B;
    constexpr int SPAN = TILE + 2 * HALF;                 // inputs per tile
    constexpr int CHUNKS = SPAN / VEC;                    // 16 B chunks per tile
    constexpr int PADDED = SPAN + (CHUNKS / 4 + 1) * VEC; // padded elements per buffer
    constexpr int TAPS = 2 * HALF + 1;
    static_assert(SPAN % VEC == 0 && (C1_B + TAPS - 1) % VEC == 0, "tile span must be 16 B aligned");
    extern __shared__ __align__(16) unsigned char smem_c1[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    T* buf = reinterpret_cast<T*>(smem_c1) + warp * 2 * PADDED;   // two buffers per warp

    // A warp's first two tiles are static (global warp id, + total warps);
    // later ones come from the atomic queue (offset by 2 * total warps).
    // Queue claims are pipelined: the atomic for the tile after next is issued
    // before the current tile's FMAs and its result is read after them (no
    // claim at all when the static tiles cover the line, e.g. C1).
    // (volatile asm keeps the compiler from sinking the atomic next to its use)
    const int64_t gw = (int64_t)bid * C1_WARPS + warp;
    const int64_t tw = P.total_warps;
    const bool dynamic = P.ntiles > 2 * tw;
    auto claim_issue = [&]() -> unsigned {
        unsigned id = 0;
        if (dynamic && lane == 0)
            asm volatile("atom.global.add.u32 %0, [%1], 1;" : "=r"(id) : "l"(&P.counter[2]) : "memory");
        return id;
    };
    auto claim_finish = [&](unsigned id) -> int64_t {
        return dynamic ? (int64_t)__shfl_sync(0xffffffffu, id, 0) + 2 * tw : P.ntiles;
    };
    auto stage = [&](int64_t tile, T* dstbuf) {
        if (tile < P.ntiles) {
            const int64_t first = P.lo + tile * TILE - HALF;   // 16 B aligned
            for (int c = lane; c < CHUNKS; c += 32)
                cp_async16(dstbuf + c1_pad<T>(c * VEC), P.src + first + c * VEC, true);
        }
        cp_async_commit();                                 // uniform group counting
    };

    int64_t tile = gw;
    int64_t next = gw + tw;
    int cur = 0;
    stage(tile, buf);
    stage(next, buf + PADDED);
    while (tile < P.ntiles) {
        const unsigned after_raw = claim_issue();         // in flight during the FMAs
        cp_async_wait<1>();
        __syncwarp();
        const T* s = buf + cur * PADDED;
        // lane window base; with C1_B/VEC a multiple of 4 chunks the padding of
        // lane * C1_B + jj splits into a lane part and a compile-time jj part,
        // so every window load is the base plus an immediate offset
        constexpr bool SPLIT = (C1_B / VEC) % 4 == 0;
        const T* sl = s + (SPLIT ? c1_pad<T>(lane * C1_B) : 0);
        T acc[C1_B];
        using V = typename Vec16<T>::type;
#pragma unroll
        for (int jj = 0; jj < C1_B + TAPS - 1; jj += VEC) {
            const int off = SPLIT ? jj + (jj / (4 * VEC)) * VEC : c1_pad<T>(lane * C1_B + jj);
            const V xv = *reinterpret_cast<const V*>(sl + off);   // 16 B, conflict-free
#pragma unroll
            for (int e = 0; e < VEC; e++) {
                const int j = jj + e;
                const T x = reinterpret_cast<const T*>(&xv)[e];
#pragma unroll
                for (int o = 0; o < C1_B; o++) {
                    const int t = j - o;                 // tap index of x for output o
                    if (t >= 0 && t < TAPS) acc[o] = (t == 0) ? x * P.c[0] : __fma_rn(P.c[t], x, acc[o]);
                }
            }
        }
        const int64_t q0 = P.lo + tile * TILE + lane * C1_B;
        const int64_t t0 = P.lo + tile * TILE;
        if (SB_C1_COALESCED_STORES && t0 + TILE <= P.hi) {
            // whole tile: outputs through the tile's (consumed) staging buffer, so each
            // store instruction writes a contiguous 512 B segment (whole sectors)
            T* sb = const_cast<T*>(s);
            __syncwarp();
#pragma unroll
            for (int v = 0; v < C1_B / VEC; v++) {
                V pack;
#pragma unroll
                for (int e = 0; e < VEC; e++) reinterpret_cast<T*>(&pack)[e] = acc[v * VEC + e];
                *reinterpret_cast<V*>(sb + c1_pad<T>(lane * C1_B + v * VEC)) = pack;
            }
            __syncwarp();
#pragma unroll
            for (int c = lane; c < TILE / VEC; c += 32)
                *reinterpret_cast<V*>(P.dst + t0 + c * VEC) = *reinterpret_cast<const V*>(sb + c1_pad<T>(c * VEC));
        } else if (q0 + C1_B <= P.hi) {
#pragma unroll
            for (int v = 0; v < C1_B / VEC; v++) {
                V pack;
#pragma unroll
                for (int e = 0; e < VEC; e++) reinterpret_cast<T*>(&pack)[e] = acc[v * VEC + e];
                *reinterpret_cast<V*>(P.dst + q0 + v * VEC) = pack;
            }
        } else {
#pragma unroll
            for (int o = 0; o < C1_B; o++)
                if (q0 + o < P.hi) P.dst[q0 + o] = acc[o];
        }
        __syncwarp();                                    // buffer `cur` free before it is restaged
        const int64_t after = claim_finish(after_raw);
        stage(after, buf + cur * PADDED);
        tile = next;
        next = after;
        cur ^= 1;
    }
    cp_async_wait<0>();
    if (dynamic && lane == 0) {
        const unsigned retired = atomicAdd(&P.counter[3], 1u);
        if (retired == (unsigned)P.total_warps - 1) {
            atomicExch(&P.counter[2], 0u);
            atomicExch(&P.counter[3], 0u);
        }
    }
}

template <typename T, int HALF>
constexpr int compose1d_smem_bytes() {
    constexpr int VEC = Vec16<T>::n;
    constexpr int SPAN = 32 * C1_B + 2 * HALF;
    constexpr int PADDED = SPAN + (SPAN / VEC / 4 + 1) * VEC;
    return C1_WARPS * 2 * PADDED * (int)sizeof(T);
}

}  // namespace sb
