// K2p -- the halo-free form of the fused 2D sweep (fused2d.cuh), fp64.
//
// fused2d_kernel carries, per level and row, the tests that make a strip
// correct next to the Dirichlet halo (physical y rows, x-halo columns, ragged
// last strip, rows outside the allocation).  On a 16384^2 grid 98% of the
// (strip, y-range) items touch none of that, and a DFMA occupies the issue
// port for two cycles (DESIGN 6.3), so every other instruction costs FP64
// throughput.  The host marks the items whose whole dependency cone is
// interior (launch2d.cu split_plain_2d); split2d_kernel runs those through
// plain2d_item and the rest -- listed first, so they start with the launch --
// through fused2d_item, in ONE launch (a second kernel on a side stream only
// overlaps if it wins the race for the SMs against the persistent grid:
// measured 1.43-1.69 ms per launch instead of 0.9 when it lost).  Same
// arithmetic, same canonical (dy, dx) order per output: bit-identical to
// fused2d_kernel in both arithmetic modes (scalar_step, kernels.py:103-108 /
// 120-134).
//
// Differences from fused2d_item:
//  * no per-level halo / allocation / store-mask tests: a level is the warp
//    shuffles (levels >= 2) or four shared loads (level 1) plus the push;
//  * staging by whole 32 B sectors: instruction c of a row copies columns
//    [64c, 64c + 64) with lane L on 16 B chunk L, so a warp instruction reads
//    16 full sectors (fused2d_item's lane-owned 32 B chunks touch half of 32
//    sectors per instruction; measured L2 traffic per C3b launch 11.1 -> 10.8
//    GB, so the coalescer already merged most of that); the two strip-edge
//    halo columns are one 16 B chunk each (lanes 0, 1);
//  * level 1 reads its x-neighbours from the shared row, not by shuffles
//    (the strip-edge lanes need no select);
//  * ring of 9 rows, prefetch distance 8; the row loop is unrolled x3 (the
//    pending-row roles rotate by renaming), so ring slots are a per-3-rows
//    base plus compile-time offsets;
//  * code size ~1/3 (fused2d<double, box, 4> is 38 KB of SASS, above the
//    32 KB instruction cache: 11% "no instruction" stalls).
#pragma once
#include "fused2d.cuh"

namespace sb {

constexpr int P2_RING = 9;     // staged rows per warp
constexpr int P2_DIST = 8;     // prefetch distance (rows)
// Shared row, in 16 B chunks: strip chunk q (columns 2q, 2q + 1 of the computed strip) at
// position q + q / 8 -- one pad chunk per 8, so the 8 lanes of a 128-bit load phase (lane
// L on chunks 2L, 2L + 1) fall on 8 different bank groups, where the dense layout gave
// 2-way conflicts on every phase -- then the left / right strip-edge pairs at 72, 73 and
// the dump chunk of the lanes that stage no edge at 74.
constexpr int P2_ROWW = 150;   // doubles per shared row (75 chunks)
constexpr int P2_ROWB = P2_ROWW * 8;
__host__ __device__ constexpr int p2_pos(int q) { return q + (q >> 3); }

__device__ __forceinline__ double2 p2_lds128(unsigned a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ double p2_lds64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
// keep a per-lane constant in its register (ptxas otherwise rematerialises the lane
// arithmetic inside the row loop: +7 instructions per row step)
__device__ __forceinline__ void p2_pin(unsigned& x) { asm volatile("" : "+r"(x)); }
__device__ __forceinline__ void p2_pin(int64_t& x) { asm volatile("" : "+l"(x)); }

// SKEW: level l of row step t consumes the level-(l-1) row completed in step t - 1
// (levels run top down inside a step, so the completed row is read before level
// l-1 restarts that register set): the K pushes of a step are independent --
// every shuffle is issued up front and its latency hidden by the other levels'
// DFMAs (without it 24% of the stall samples are DFMAs waiting on SHFL / LDS
// results; C3b k=4 1049 -> 1102 GStencil/s).  No extra state; an item runs K - 1
// more warm-up steps.
template <bool BOX, int K, bool FMA, bool SEP, bool SKEW>
__device__ __forceinline__ void plain2d_item(const Fused2DParams<double>& P, const Item2D it, double* ring,
                                             const int lane) {
    using T = double;
    using TL = F2Tile<T, K>;
    static_assert(F2_VX == 4, "plain2d: 4 columns per lane");
    const unsigned ring_s = static_cast<unsigned>(__cvta_generic_to_shared(ring));
    // staging: lane L copies chunks L and 32 + L (p2_pos(32 + L) = p2_pos(L) + 36)
    unsigned wr_s = ring_s + 16u * (unsigned)p2_pos(lane);
    // strip-edge pairs: lane 0 columns [-2, 0), lane 1 columns [128, 130); the other lanes
    // issue the same instruction with source size 0 (zero fill) into the dump chunk
    unsigned we_s = ring_s + 16u * (lane == 0 ? 72u : lane == 1 ? 73u : 74u);
    const unsigned esize = lane < 2 ? 16u : 0u;
    unsigned rd = ring_s + 16u * (unsigned)p2_pos(2 * lane);          // own columns of slot 0 (chunks 2L, 2L + 1)
    // x-neighbours at level 1: column -1 (upper half of chunk 2L - 1, or of the left edge
    // pair) and column 4 (lower half of chunk 2L + 2, or of the right edge pair)
    const int nl = lane == 0 ? 2 * 72 + 1 : 2 * p2_pos(2 * lane - 1) + 1;
    const int nr = lane == 31 ? 2 * 73 : 2 * p2_pos(2 * lane + 2);
    unsigned rdl = ring_s + 8u * (unsigned)nl, rdr = ring_s + 8u * (unsigned)nr;
    p2_pin(wr_s);
    p2_pin(we_s);
    p2_pin(rd);
    p2_pin(rdl);
    p2_pin(rdr);
    const bool stores = lane >= TL::HL / F2_VX && lane < 32 - TL::HL / F2_VX;
    const int eoff = lane == 0 ? -2 : lane == 1 ? F2_CW - 2 : 0;      // edge pair relative to the lane's chunk
    {
        const int xc = TL::X0 + it.tix * TL::TXO - TL::HL;   // computed strip origin (16 B aligned)
        const int p_first = it.ys0 - K;
        constexpr int LAG = SKEW ? 3 * K - 1 : 2 * K;   // steps from a level-0 arrival to the level-K row it completes... of ys0
        const int M = (it.ys1 - it.ys0) + LAG;
        const T* gs = P.src + P.origin + (int64_t)p_first * P.sy + xc + 2 * lane;   // row to stage next
        T* outp = P.dst + P.origin + (int64_t)(it.ys0 - LAG) * P.sy + xc + F2_VX * lane;   // level-K row of t = 0

        // one row into the ring slot at byte offset slot_b; unconditional: the host keeps
        // P2_DIST allocated rows below every plain item (split_plain_2d)
        auto stage_from = [&](const T* g, unsigned slot_b) {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(wr_s + slot_b), "l"(g));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(wr_s + slot_b + 576u), "l"(g + 64));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(we_s + slot_b), "l"(g + eoff), "r"(esize));
            cp_async_commit();
        };
#pragma unroll
        for (int t = 0; t < P2_DIST; t++) stage_from(gs + (int64_t)t * P.sy, t * P2_ROWB);
        // The row loop is unrolled x3 and each of its three steps has its own staging and
        // store pointer, advanced by three rows just before its use: a pointer bumped right
        // after the cp.async / store that read it waits on that instruction's operand
        // scoreboard (10% of the stall samples with one running pointer).
        int64_t sy3b = 3 * (int64_t)sizeof(T) * P.sy;    // three rows, in bytes
        p2_pin(sy3b);
        auto bump = [&](auto*& ptr) {
            using Ptr = std::remove_reference_t<decltype(ptr)>;
            ptr = reinterpret_cast<Ptr>(reinterpret_cast<uintptr_t>(ptr) + (uintptr_t)sy3b);
        };
        const T* gsr[3];
        T* outr[3];
#pragma unroll
        for (int q = 0; q < 3; q++) {
            gsr[q] = gs + (int64_t)(P2_DIST + q - 3) * P.sy;
            outr[q] = outp + (int64_t)(q - 3) * P.sy;
        }

        T A[K][3][F2_VX];   // per level: pending-row sets, roles rotating with t (mod 3)
#pragma unroll
        for (int l = 0; l < K; l++)
#pragma unroll
            for (int q = 0; q < 3; q++)
#pragma unroll
                for (int j = 0; j < F2_VX; j++) A[l][q][j] = T(0);

        // ring slot of row t = 3 g + rot: byte base b0 = 3 g ROWB; row t + 8 goes to slot
        // (3 g + rot + 8) mod 9 = 3 ((g + 2) mod 3) + 2 (rot 0), 3 g + rot - 1 (rot 1, 2)
        unsigned b0 = 0, b2 = 6 * P2_ROWB;
        auto row_step = [&](int t, auto rot) {
            constexpr int ROT = decltype(rot)::value;
            constexpr int IC = ROT, IK = (ROT + 1) % 3, IS = (ROT + 2) % 3;
            cp_async_wait<P2_DIST - 1>();
            __syncwarp();
            T u[F2_VX + 2];
            {
                const unsigned sb = b0 + ROT * P2_ROWB;     // slot of row t
                const double2 a = p2_lds128(rd + sb);
                const double2 b = p2_lds128(rd + sb + 16u);
                u[1] = a.x; u[2] = a.y; u[3] = b.x; u[4] = b.y;
                u[0] = p2_lds64(rdl + sb);
                u[5] = p2_lds64(rdr + sb);
            }
            // restage the slot of row t - 1: every lane read it before the __syncwarp above
            bump(gsr[ROT]);
            stage_from(gsr[ROT], ROT == 0 ? b2 + 2 * P2_ROWB : b0 + (ROT - 1) * P2_ROWB);
            if constexpr (SKEW) {
                T out[F2_VX];
#pragma unroll
                for (int l = K; l >= 1; l--) {
                    T v[F2_VX + 2];
                    if (l > 1) {                            // level-(l-1) row completed in the previous step
#pragma unroll
                        for (int j = 0; j < F2_VX; j++) v[j + 1] = A[l - 2][IS][j];
                        v[0] = __shfl_up_sync(0xffffffffu, v[F2_VX], 1);
                        v[F2_VX + 1] = __shfl_down_sync(0xffffffffu, v[1], 1);
                    } else {
#pragma unroll
                        for (int j = 0; j < F2_VX + 2; j++) v[j] = u[j];
                    }
                    f2_push3<T, BOX, FMA, SEP>(v, A[l - 1][IC], A[l - 1][IK], A[l - 1][IS], P.w, P.sa, P.sb);
                    if (l == K) {
#pragma unroll
                        for (int j = 0; j < F2_VX; j++) out[j] = A[K - 1][IC][j];
                    }
                }
#pragma unroll
                for (int j = 0; j < F2_VX; j++) u[j + 1] = out[j];
            } else {
#pragma unroll
                for (int l = 1; l <= K; l++) {
                    if (l > 1) {
                        u[0] = __shfl_up_sync(0xffffffffu, u[F2_VX], 1);
                        u[F2_VX + 1] = __shfl_down_sync(0xffffffffu, u[1], 1);
                    }
                    f2_push3<T, BOX, FMA, SEP>(u, A[l - 1][IC], A[l - 1][IK], A[l - 1][IS], P.w, P.sa, P.sb);
#pragma unroll
                    for (int j = 0; j < F2_VX; j++) u[j + 1] = A[l - 1][IC][j];   // completed row p_first + t - l of level l
                }
            }
            bump(outr[ROT]);
            if (t >= LAG && stores) {                       // level-K row ys0 + t - LAG
                // (global-space stores: the integer pointer bump hides the address space from nvcc)
                asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(outr[ROT]), "d"(u[1]), "d"(u[2]) : "memory");
                asm volatile("st.global.v2.f64 [%0+16], {%1, %2};" ::"l"(outr[ROT]), "d"(u[3]), "d"(u[4]) : "memory");
            }
        };
        for (int t = 0; t < M; t += 3) {
            row_step(t, std::integral_constant<int, 0>());
            if (t + 1 < M) row_step(t + 1, std::integral_constant<int, 1>());
            if (t + 2 < M) row_step(t + 2, std::integral_constant<int, 2>());
            b2 = b0;
            b0 = b0 == 6 * P2_ROWB ? 0u : b0 + 3 * P2_ROWB;
        }
        cp_async_wait<0>();
        __syncwarp();
    }
}

// The 2D launch of depth K: halo items (listed first) and plain items from one queue.
template <bool BOX, int K, bool FMA, bool SEP, int MINB, bool SKEW>
__global__ void __launch_bounds__(F2_WARPS * 32, MINB)
split2d_kernel(const Fused2DParams<double> P) {
    extern __shared__ __align__(16) unsigned char smem_f2[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* ring = reinterpret_cast<double*>(smem_f2) + warp * (F2_DEPTH + K) * F2_ROWW;
    static_assert(P2_RING * P2_ROWW <= (F2_DEPTH + 3) * F2_ROWW, "plain ring fits the general one");
    f2_item_loop(P, lane, [&](const Item2D it, const unsigned item) {
        if (it.plain)
            plain2d_item<BOX, K, FMA, SEP, SKEW>(P, it, ring, lane);
        else
            fused2d_item<double, BOX, K, FMA, SEP>(P, it, ring, lane, item);
    });
}

}  // namespace sb
