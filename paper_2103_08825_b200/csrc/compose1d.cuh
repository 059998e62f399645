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

constexpr int C1_B = 8;          // outputs per lane per tile
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

template <typename T, int HALF>   // HALF = R*K
__global__ void __launch_bounds__(C1_WARPS * 32)
compose1d_kernel(const Compose1DParams<T> P) {
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

    // Claims are pipelined: the atomic for the tile after next is issued
    // before the current tile's FMAs and its result is read after them.
    // (volatile asm keeps the compiler from sinking the atomic next to its use)
    auto claim_issue = [&]() -> unsigned {
        unsigned id = 0;
        if (lane == 0)
            asm volatile("atom.global.add.u32 %0, [%1], 1;" : "=r"(id) : "l"(&P.counter[2]) : "memory");
        return id;
    };
    auto claim_finish = [&](unsigned id) -> int64_t {
        return (int64_t)__shfl_sync(0xffffffffu, id, 0);
    };
    auto stage = [&](int64_t tile, T* dstbuf) {
        if (tile < P.ntiles) {
            const int64_t first = P.lo + tile * TILE - HALF;   // 16 B aligned
            for (int c = lane; c < CHUNKS; c += 32)
                cp_async16(dstbuf + c1_pad<T>(c * VEC), P.src + first + c * VEC, true);
        }
        cp_async_commit();                                 // uniform group counting
    };

    int64_t tile = claim_finish(claim_issue());
    int64_t next = claim_finish(claim_issue());
    int cur = 0;
    stage(tile, buf);
    stage(next, buf + PADDED);
    while (tile < P.ntiles) {
        const unsigned after_raw = claim_issue();         // in flight during the FMAs
        cp_async_wait<1>();
        __syncwarp();
        const T* s = buf + cur * PADDED;
        T acc[C1_B];
        using V = typename Vec16<T>::type;
#pragma unroll
        for (int jj = 0; jj < C1_B + TAPS - 1; jj += VEC) {
            const V xv = *reinterpret_cast<const V*>(s + c1_pad<T>(lane * C1_B + jj));   // 16 B, conflict-free
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
        if (q0 + C1_B <= P.hi) {
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
    if (lane == 0) {
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
