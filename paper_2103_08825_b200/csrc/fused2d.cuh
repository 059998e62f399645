// K2 -- fused 2D sweep (r = 1: 9-point box or 5-point star), K time steps
// per HBM round trip: warp-independent y-streaming with temporal blocking.
//
// Replaces the reference's 2D paths -- scalar_step over the whole grid
// (kernels.py:120-134) and the tessellated thread-pool runner
// (tiling.py:372-417, whose tiles synchronise per stage) -- with a scheme
// that needs no block-level synchronisation at all:
//  * one warp owns a strip of 32 x VX computed columns (VX per lane) and
//    streams it along y; a work item is (strip, y range), taken from a
//    host-built guided schedule through one atomic (claims pipelined);
//  * level-0 rows are staged by cp.async into a per-warp shared ring DEPTH
//    rows deep (each lane's VX columns are one 32 B chunk: strips start so
//    that it is 16 B aligned), the strip-edge halo columns by element copies;
//  * x-neighbours of a lane's VX values come from lanes +-1 by warp shuffles;
//    at the strip edges they come from the staged halo columns at level 0 and
//    are garbage above it, so the valid strip shrinks by one column per side
//    per level (overlapped strips: output 32*VX - 2(K-1) columns);
//  * every level keeps two pending partial-sum rows per lane in registers
//    (push form along y): an arriving level-(l-1) row a is folded into rows
//    a+1 (dy=-1, first terms), a (dy=0) and a-1 (dy=+1, completing), so each
//    output sums its terms in canonical (dy, dx) order -- bit-exact in EXACT
//    mode (kernels.py:103-108).
// Boundaries: emitted values outside the interior on a physical side are
// replaced by the Dirichlet halo (global read), beyond the halo shell by 0;
// slab (ghost) sides along y compute normally.
#pragma once
#include <climits>
#include <type_traits>
#include "common.cuh"
#include "fused1d.cuh"   // cp.async helpers, Vec16

namespace sb {

#ifndef SB_F2_VX
#define SB_F2_VX 4
#endif
constexpr int F2_VX = SB_F2_VX;          // columns per lane
constexpr int F2_CW = 32 * F2_VX;        // computed strip width
#ifndef SB_F2_WARPS
#define SB_F2_WARPS 4
#endif
#ifndef SB_F2_DEPTH
#define SB_F2_DEPTH 8
#endif
constexpr int F2_WARPS = SB_F2_WARPS;    // warps per CTA
constexpr int F2_DEPTH = SB_F2_DEPTH;    // staged rows per warp
constexpr int F2_ROWW = F2_CW + 8;       // shared row: 128 columns + edges + pad

struct Item2D {
    int32_t tix;     // strip index
    int32_t ys0;     // output rows [ys0, ys1)
    int32_t ys1;
    int32_t plain;   // 1: the whole dependency cone is interior (plain2d.cuh)
};

template <typename T>
struct Fused2DParams {
    const T* src;
    T* dst;
    int64_t origin, sy;      // element (y, x) at origin + y*sy + x
    int nx, ny;
    int row_lo, row_hi;      // allocated rows [row_lo, row_hi) (halo or ghost included)
    int phys_lo, phys_hi;    // y sides: physical halo (1) or ghost (0)
    int items;
    const Item2D* sched;
    int total_warps;
    unsigned int* counter;   // [0] next item, [1] retired warps
    unsigned long long* trace;   // debug (SB200_TRACE): per item {smid|warp, t0, t1, strip|rows}
    T w[9];                  // w[(dy+1)*3 + (dx+1)]; star uses 5 entries
    T sa[3], sb[3];          // separable path: w[dy][dx] = sa[dy+1] * sb[dx+1]
};

// Strip geometry, lane aligned: the K-1 recomputed columns on each side of a
// strip are rounded up to whole lanes (HL columns), so lanes either own four
// output columns or none -- every storing lane writes whole 16 B vectors and
// no lane takes a partial-store path except on the grid's last strip.  The
// computed strip origin xc = x0 - HL is then 16 B aligned for any x0 that is
// a multiple of VX (output strips start at multiples of TXO).
template <typename T, int K>
struct F2Tile {
    static constexpr int VEC = 16 / (int)sizeof(T);
    static constexpr int HL = F2_VX * ((K - 1 + F2_VX - 1) / F2_VX);
    static constexpr int TXO = F2_CW - 2 * HL;
    static constexpr int X0 = 0;
    static_assert(HL % VEC == 0 && TXO > 0, "strip geometry");
};

template <typename T>   // one element (4 or 8 B), zero-filled when !valid
__device__ __forceinline__ void cp_async_elem(void* smem, const void* gmem, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    if (sizeof(T) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(valid ? 8 : 0));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(valid ? 4 : 0));
}

// Fold an arriving level-(l-1) row a into three pending-row sets: Pm = row
// a-1 (its dy=+1 terms complete it), P0 = row a (dy=0), nx = row a+1 (dy=-1,
// started here).  The caller rotates the roles of the three sets from row to
// row by renaming (the row loop is unrolled x3), so no register moves.
template <typename T, bool BOX, bool FMA, bool SEP = false>
__device__ __forceinline__ void f2_push3(const T (&u)[F2_VX + 2], T (&Pm)[F2_VX], T (&P0)[F2_VX], T (&nx)[F2_VX],
                                         const T* w, const T* sa = nullptr, const T* sb = nullptr) {
    // u[0] = column -1, u[1..VX] = own columns, u[VX+1] = column VX
    if (SEP) {
        // rank-1 box weights w[dy][dx] = sa[dy] * sb[dx] (FMA mode only): one horizontal
        // 3-tap pass, then the vertical push -- 6 instead of 9 FMAs per point and level
        // (same terms, regrouped: within the fp64 bar, not bit-identical)
        T h[F2_VX];
#pragma unroll
        for (int j = 0; j < F2_VX; j++)
            h[j] = acc_term<T, true>(acc_term<T, true>(acc_first<T, true>(sb[0], u[j]), sb[1], u[j + 1]), sb[2], u[j + 2]);
#pragma unroll
        for (int j = 0; j < F2_VX; j++) {
            Pm[j] = acc_term<T, true>(Pm[j], sa[2], h[j]);      // dy=+1: completes a-1
            P0[j] = acc_term<T, true>(P0[j], sa[1], h[j]);      // dy= 0
            nx[j] = acc_first<T, true>(sa[0], h[j]);            // dy=-1
        }
    } else if (BOX) {
#pragma unroll
        for (int q = 0; q < 3; q++) {          // dx = q - 1
#pragma unroll
            for (int j = 0; j < F2_VX; j++) {
                const T x = u[j + q];
                Pm[j] = acc_term<T, FMA>(Pm[j], w[6 + q], x);                        // dy=+1: completes a-1
                P0[j] = acc_term<T, FMA>(P0[j], w[3 + q], x);                        // dy= 0
                nx[j] = q == 0 ? acc_first<T, FMA>(w[0], x) : acc_term<T, FMA>(nx[j], w[q], x);  // dy=-1
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < F2_VX; j++) {
            Pm[j] = acc_term<T, FMA>(Pm[j], w[7], u[j + 1]);      // (1,0)
            P0[j] = acc_term<T, FMA>(P0[j], w[3], u[j]);          // (0,-1)
            nx[j] = acc_first<T, FMA>(w[1], u[j + 1]);            // (-1,0)
        }
#pragma unroll
        for (int j = 0; j < F2_VX; j++) P0[j] = acc_term<T, FMA>(P0[j], w[4], u[j + 1]);   // (0,0)
#pragma unroll
        for (int j = 0; j < F2_VX; j++) P0[j] = acc_term<T, FMA>(P0[j], w[5], u[j + 2]);   // (0,1)
    }
}

// One (strip, y-range) item of the general kernel, run by one warp on its ring of
// F2_DEPTH + K shared rows: prefetch distance F2_DEPTH - 1 plus the K rows already
// consumed (their x-halo columns are the Dirichlet values of the rows completed by
// levels 1..K: no global reload on the edge strips).
// shared row layout: [VEC-1] left edge, [VEC..VEC+CW) strip columns, [VEC+CW] right edge
template <typename T, bool BOX, int K, bool FMA, bool SEP>
__device__ __forceinline__ void fused2d_item(const Fused2DParams<T>& P, const Item2D it, T* ring, const int lane,
                                             const unsigned item) {
    using TL = F2Tile<T, K>;
    constexpr int VEC = 16 / (int)sizeof(T);
    using V = typename Vec16<T>::type;
    constexpr int RING = F2_DEPTH + K;
    {
        unsigned long long tr0 = 0;
        if (P.trace && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr0));
        const int x0 = TL::X0 + it.tix * TL::TXO;       // output strip origin
        const int xc = x0 - TL::HL;                     // computed strip origin (16 B aligned)
        const int ys0 = it.ys0, ys1 = it.ys1;
        const int p_first = ys0 - K;
        const int M = (ys1 - ys0) + 2 * K;

        int col[F2_VX];
        unsigned out_mask = 0, shell_mask = 0, store_mask = 0;
#pragma unroll
        for (int j = 0; j < F2_VX; j++) {
            const int x = xc + F2_VX * lane + j;
            col[j] = x;
            out_mask |= (unsigned)(x < 0 || x >= P.nx) << j;
            shell_mask |= (unsigned)(x >= -1 && x <= P.nx) << j;
            const int cj = x - x0;
            store_mask |= (unsigned)(cj >= 0 && cj < TL::TXO && x >= 0 && x < P.nx) << j;
        }
        const bool warp_out = __any_sync(0xffffffffu, out_mask != 0);   // strip touches the x halo
        // rows outside [ylo, yhi) on a physical side are Dirichlet halo
        const int ylo = P.phys_lo ? 0 : INT_MIN / 2, yhi = P.phys_hi ? P.ny : INT_MAX / 2;
        T* const out_base = P.dst + P.origin + (int64_t)(p_first - K) * P.sy + col[0];   // row of t = 0
        const int ecol = lane == 0 ? xc - 1 : xc + F2_CW;   // strip-edge halo column (lanes 0, 31)
        const bool eload = (lane == 0 || lane == 31) && ecol >= -1 && ecol <= P.nx;

        // per-item staging state: per-lane source pointers advanced one row per call and
        // per-lane chunk predicates (rows outside the allocation are warp-uniform)
        const T* gsrc = P.src + P.origin + (int64_t)p_first * P.sy + xc + F2_VX * lane;
        const T* gedge = P.src + P.origin + (int64_t)p_first * P.sy + ecol;
        unsigned chunk_ok = 0;
#pragma unroll
        for (int c = 0; c < F2_VX / VEC; c++) {
            const int x = xc + F2_VX * lane + c * VEC;  // chunk start (16 B aligned)
            chunk_ok |= (unsigned)(x >= -VEC && x <= P.nx) << c;
        }
        int ys = p_first;                               // row of the next stage() call
        int slot_s = 0;                                 // its ring slot
        const unsigned soff = static_cast<unsigned>(__cvta_generic_to_shared(ring)) +
                              (VEC + F2_VX * lane) * (unsigned)sizeof(T);
        auto stage = [&]() {
            const bool rok = ys < p_first + M && ys >= P.row_lo && ys < P.row_hi;
            const unsigned srow = soff + slot_s * (F2_ROWW * (unsigned)sizeof(T));
#pragma unroll
            for (int c = 0; c < F2_VX / VEC; c++) {
                const bool ok = rok && ((chunk_ok >> c) & 1);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(srow + c * 16),
                             "l"(ok ? gsrc + c * VEC : P.src), "r"(ok ? 16 : 0));
            }
            if (lane == 0 || lane == 31) {
                const bool ok = rok && eload;
                cp_async_elem<T>(ring + slot_s * F2_ROWW + (lane == 0 ? VEC - 1 : VEC + F2_CW), ok ? gedge : P.src, ok);
            }
            cp_async_commit();
            gsrc += P.sy;
            gedge += P.sy;
            ys++;
            slot_s = slot_s + 1 == RING ? 0 : slot_s + 1;
        };
#pragma unroll
        for (int t = 0; t < F2_DEPTH - 1; t++) stage();
        int slot_t = 0;                                 // ring slot of row t

        T A[K][3][F2_VX];   // per level: pending-row sets, roles rotating with t (mod 3)
#pragma unroll
        for (int l = 0; l < K; l++)
#pragma unroll
            for (int q = 0; q < 3; q++)
#pragma unroll
                for (int j = 0; j < F2_VX; j++) A[l][q][j] = T(0);

        auto row_step = [&](int t, auto rot) {
            constexpr int IC = decltype(rot)::value, IK = (IC + 1) % 3, IS = (IC + 2) % 3;
            cp_async_wait<F2_DEPTH - 2>();
            __syncwarp();
            const T* row = ring + slot_t * F2_ROWW;
            T v[F2_VX];
#pragma unroll
            for (int j = 0; j < F2_VX; j++) v[j] = row[VEC + F2_VX * lane + j];
            T edge = lane == 0 ? row[VEC - 1] : row[VEC + F2_CW];
            __syncwarp();                                   // slot t-K-1 fully read before restaging
            stage();                                        // row t + DEPTH - 1
            const int a0 = p_first + t;
            // no level of this row touches a physical y halo and the strip no x halo
            const bool plain = !warp_out && a0 - K >= ylo && a0 - 1 < yhi;
#pragma unroll
            for (int l = 1; l <= K; l++) {
                T u[F2_VX + 2];
                const T left = __shfl_up_sync(0xffffffffu, v[F2_VX - 1], 1);
                const T right = __shfl_down_sync(0xffffffffu, v[0], 1);
                // the strip-edge halo column matters only at level 1; above it the
                // strip's outermost columns are garbage anyway (overlapped strips)
                u[0] = (l == 1 && lane == 0) ? edge : left;
                u[F2_VX + 1] = (l == 1 && lane == 31) ? edge : right;
#pragma unroll
                for (int j = 0; j < F2_VX; j++) u[j + 1] = v[j];
                f2_push3<T, BOX, FMA, SEP>(u, A[l - 1][IC], A[l - 1][IK], A[l - 1][IS], P.w, P.sa, P.sb);
                T (&done)[F2_VX] = A[l - 1][IC];        // completed: row a0 - l of level l
                const int yc = a0 - l;                      // completed level-l row
                const bool y_out = yc < ylo || yc >= yhi;
                if (!plain && y_out) {                      // (warp-uniform) physical y-halo row
                    const bool y_shell = yc >= -1 && yc <= P.ny;
                    const bool y_alloc = yc >= P.row_lo && yc < P.row_hi;
                    const T* rowp = P.src + P.origin + (int64_t)yc * P.sy;
#pragma unroll
                    for (int j = 0; j < F2_VX; j++) {
                        const bool sh = y_alloc && y_shell && ((shell_mask >> j) & 1);
                        done[j] = sh ? rowp[col[j]] : T(0);
                    }
                } else if (warp_out) {                      // x-halo columns of an interior (or ghost) row:
                    // the level-0 value of row yc, still in the ring (zero-filled outside the allocation)
                    const int sl = slot_t - l;
                    const T* r0 = ring + (sl < 0 ? sl + RING : sl) * F2_ROWW + VEC + F2_VX * lane;
#pragma unroll
                    for (int j = 0; j < F2_VX; j++)
                        if ((out_mask >> j) & 1) done[j] = ((shell_mask >> j) & 1) ? r0[j] : T(0);
                }
                if (l < K) {
#pragma unroll
                    for (int j = 0; j < F2_VX; j++) v[j] = done[j];
                } else if (yc >= ys0 && yc < ys1) {
                    T* rowp = out_base + (int64_t)t * P.sy;    // row yc, column col[0]
                    if (store_mask == (1u << F2_VX) - 1) {  // whole 16 B-aligned chunk: vector stores
#pragma unroll
                        for (int c = 0; c < F2_VX / VEC; c++) {
                            V pack;
#pragma unroll
                            for (int e = 0; e < VEC; e++) reinterpret_cast<T*>(&pack)[e] = done[c * VEC + e];
                            *reinterpret_cast<V*>(rowp + c * VEC) = pack;
                        }
                    } else if (store_mask) {                // last strip only: columns past nx
#pragma unroll
                        for (int j = 0; j < F2_VX; j++)
                            if ((store_mask >> j) & 1) rowp[j] = done[j];
                    }
                }
            }
            slot_t = slot_t + 1 == RING ? 0 : slot_t + 1;
        };
        if constexpr (K <= 4) {
            // roles renamed by unrolling x3 (no moves): C3b k=4 1041-1047 vs 1025 GStencil/s
            for (int t = 0; t < M; t += 3) {
                row_step(t, std::integral_constant<int, 0>());
                if (t + 1 < M) row_step(t + 1, std::integral_constant<int, 1>());
                if (t + 2 < M) row_step(t + 2, std::integral_constant<int, 2>());
            }
        } else {
            // k = 8: the x3 body needs 254 registers (769 vs 968 GStencil/s); rotate by moves
            for (int t = 0; t < M; t++) {
                row_step(t, std::integral_constant<int, 0>());
#pragma unroll
                for (int l = 0; l < K; l++)
#pragma unroll
                    for (int j = 0; j < F2_VX; j++) {
                        A[l][0][j] = A[l][1][j];
                        A[l][1][j] = A[l][2][j];
                    }
            }
        }
        cp_async_wait<0>();
        __syncwarp();
        if (P.trace && lane == 0) {
            unsigned long long tr1;
            unsigned smid;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr1));
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            P.trace[4 * item + 0] = ((unsigned long long)smid << 32) | (blockIdx.x * F2_WARPS + (threadIdx.x >> 5));
            P.trace[4 * item + 1] = tr0;
            P.trace[4 * item + 2] = tr1;
            P.trace[4 * item + 3] = ((unsigned long long)it.tix << 40) | (unsigned long long)(it.ys1 - it.ys0);
        }
    }
}

// Persistent warps over the item list: one atomic per claim, issued one item
// ahead; the last warp to retire resets the queue for the next launch.
template <typename T, typename ItemFn>
__device__ __forceinline__ void f2_item_loop(const Fused2DParams<T>& P, const int lane, ItemFn&& run) {
    auto claim_issue = [&]() -> unsigned {
        unsigned id = 0;
        if (lane == 0)
            asm volatile("atom.global.add.u32 %0, [%1], 1;" : "=r"(id) : "l"(&P.counter[0]) : "memory");
        return id;
    };
    unsigned item = __shfl_sync(0xffffffffu, claim_issue(), 0);
    while (item < (unsigned)P.items) {
        const unsigned next_raw = claim_issue();        // resolved after this item
        run(P.sched[item], item);
        item = __shfl_sync(0xffffffffu, next_raw, 0);
    }
    if (lane == 0) {
        const unsigned retired = atomicAdd(&P.counter[1], 1u);
        if (retired == (unsigned)P.total_warps - 1) {
            atomicExch(&P.counter[0], 0u);
            atomicExch(&P.counter[1], 0u);
        }
    }
}

template <typename T, bool BOX, int K, bool FMA, bool SEP = false>
__global__ void __launch_bounds__(F2_WARPS * 32)
fused2d_kernel(const Fused2DParams<T> P) {
    extern __shared__ __align__(16) unsigned char smem_f2[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    T* ring = reinterpret_cast<T*>(smem_f2) + warp * (F2_DEPTH + K) * F2_ROWW;
    f2_item_loop(P, lane, [&](const Item2D it, const unsigned item) {
        fused2d_item<T, BOX, K, FMA, SEP>(P, it, ring, lane, item);
    });
}

template <typename T, int K>
constexpr int fused2d_smem_bytes() { return F2_WARPS * (F2_DEPTH + K) * F2_ROWW * (int)sizeof(T); }

}  // namespace sb
