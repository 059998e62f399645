// K2 -- fused 2D sweep (r = 1: 9-point box or 5-point star), K time steps
// per HBM round trip: warp-independent y-streaming with temporal blocking.
//
// Replaces the reference's 2D paths -- scalar_step over the whole grid
// (kernels.py:120-134) and the tessellated thread-pool runner
// (tiling.py:372-417, whose tiles synchronise per stage) -- with a scheme
// that needs no synchronisation at all:
//  * one warp owns a strip of 32 x VX computed columns (VX per lane) and
//    streams it along y; a work item is (strip, y segment), claimed from an
//    atomic queue by persistent warps;
//  * x-neighbours of a lane's VX values come from lanes +-1 by warp
//    shuffles; at the strip edges they come from the loaded halo columns at
//    level 0 and are garbage above it, so the valid strip shrinks by one
//    column per side per level (overlapped tiles: output 32*VX - 2(K-1));
//  * every level keeps two pending partial-sum rows per lane in registers
//    (push form along y): an arriving level-(l-1) row a is folded into rows
//    a+1 (dy=-1, first terms), a (dy=0) and a-1 (dy=+1, completing), so each
//    output sums its terms in canonical (dy, dx) order -- bit-exact in EXACT
//    mode (kernels.py:103-108);
//  * level-0 rows are loaded straight into registers, DEPTH rows ahead.
// Boundaries: as in the 3D kernel, emitted values outside the interior on a
// physical side are replaced by the Dirichlet halo (global read), values
// beyond the halo shell by 0; slab (ghost) sides along y compute normally.
#pragma once
#include "common.cuh"

namespace sb {

constexpr int F2_VX = 4;                 // columns per lane
constexpr int F2_CW = 32 * F2_VX;        // computed strip width
constexpr int F2_WARPS = 4;              // warps per CTA
constexpr int F2_DEPTH = 4;              // level-0 rows in flight per warp

template <typename T>
struct Fused2DParams {
    const T* src;
    T* dst;
    int64_t origin, sy;      // element (y, x) at origin + y*sy + x
    int nx, ny;
    int row_lo, row_hi;      // loadable rows [row_lo, row_hi) (halo or ghost included)
    int phys_lo, phys_hi;    // y sides: physical halo (1) or ghost (0)
    int tiles_x, nseg, ly, items;
    int total_warps;
    unsigned int* counter;   // [0] next item, [1] retired warps
    T w[9];                  // w[(dy+1)*3 + (dx+1)]; star uses 5 entries
};

template <int K>
struct F2Tile {
    static constexpr int TXO = F2_CW - 2 * (K - 1);
};

template <typename T, bool BOX, bool FMA>
__device__ __forceinline__ void f2_push(const T (&u)[F2_VX + 2], T (&Pm)[F2_VX], T (&P0)[F2_VX], T (&done)[F2_VX],
                                        const T* w) {
    // u[0] = column -1, u[1..VX] = own columns, u[VX+1] = column VX
    T nx[F2_VX];
    if (BOX) {
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
#pragma unroll
    for (int j = 0; j < F2_VX; j++) {
        done[j] = Pm[j];
        Pm[j] = P0[j];
        P0[j] = nx[j];
    }
}

template <typename T, bool BOX, int K, bool FMA>
__global__ void __launch_bounds__(F2_WARPS * 32)
fused2d_kernel(const Fused2DParams<T> P) {
    using TL = F2Tile<K>;
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned item = 0;
        if (lane == 0) item = atomicAdd(&P.counter[0], 1u);
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item >= (unsigned)P.items) break;
        const int tix = item % P.tiles_x, seg = item / P.tiles_x;
        const int x0 = tix * TL::TXO;               // output strip origin
        const int xc = x0 - (K - 1);                // computed strip origin
        const int ys0 = seg * P.ly, ys1 = min(P.ny, ys0 + P.ly);
        const int p_first = ys0 - K;
        const int M = (ys1 - ys0) + 2 * K;

        // per-lane column bookkeeping (fixed for the item)
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
        const int ecol = lane == 0 ? xc - 1 : xc + F2_CW;   // strip-edge halo column (lanes 0, 31)
        const bool eload = (lane == 0 || lane == 31) && ecol >= -1 && ecol <= P.nx;
        bool cload[F2_VX];
#pragma unroll
        for (int j = 0; j < F2_VX; j++) cload[j] = col[j] >= -1 && col[j] <= P.nx;

        // level-0 rows in flight: ring of DEPTH rows of VX values + one edge value
        T ring[F2_DEPTH][F2_VX + 1];
        auto load_row = [&](int t, T (&dstv)[F2_VX + 1]) {
            const int y = p_first + t;
            const bool rok = t < M && y >= P.row_lo && y < P.row_hi;
            const T* rowp = P.src + P.origin + (int64_t)y * P.sy;
#pragma unroll
            for (int j = 0; j < F2_VX; j++) dstv[j] = (rok && cload[j]) ? __ldg(rowp + col[j]) : T(0);
            dstv[F2_VX] = (rok && eload) ? __ldg(rowp + ecol) : T(0);
        };
#pragma unroll
        for (int d = 0; d < F2_DEPTH; d++) load_row(d, ring[d]);

        T Pm[K][F2_VX], P0[K][F2_VX];
#pragma unroll
        for (int l = 0; l < K; l++)
#pragma unroll
            for (int j = 0; j < F2_VX; j++) Pm[l][j] = P0[l][j] = T(0);

        for (int t0 = 0; t0 < M; t0 += F2_DEPTH) {
#pragma unroll
            for (int d = 0; d < F2_DEPTH; d++) {
                const int t = t0 + d;
                if (t >= M) break;
                T cur[F2_VX + 1];
#pragma unroll
                for (int j = 0; j <= F2_VX; j++) cur[j] = ring[d][j];
                load_row(t + F2_DEPTH, ring[d]);              // refill this slot, DEPTH ahead
                const int a0 = p_first + t;
                T v[F2_VX];
#pragma unroll
                for (int j = 0; j < F2_VX; j++) v[j] = cur[j];
                T edge = cur[F2_VX];
#pragma unroll
                for (int l = 1; l <= K; l++) {
                    T u[F2_VX + 2];
                    const T left = __shfl_up_sync(0xffffffffu, v[F2_VX - 1], 1);
                    const T right = __shfl_down_sync(0xffffffffu, v[0], 1);
                    u[0] = lane == 0 ? edge : left;
                    u[F2_VX + 1] = lane == 31 ? edge : right;
#pragma unroll
                    for (int j = 0; j < F2_VX; j++) u[j + 1] = v[j];
                    T done[F2_VX];
                    f2_push<T, BOX, FMA>(u, Pm[l - 1], P0[l - 1], done, P.w);
                    const int yc = a0 - l;                    // completed level-l row
                    const bool y_out = (P.phys_lo && yc < 0) || (P.phys_hi && yc >= P.ny);
                    if (y_out || out_mask) {                  // Dirichlet halo, same at every level
                        const bool y_shell = yc >= -1 && yc <= P.ny;
                        // rows outside the allocation (first completions of a ghost-side
                        // segment) are garbage that never reaches a valid output: no load
                        const bool y_alloc = yc >= P.row_lo && yc < P.row_hi;
                        const T* rowp = P.src + P.origin + (int64_t)yc * P.sy;
#pragma unroll
                        for (int j = 0; j < F2_VX; j++) {
                            if (y_out || ((out_mask >> j) & 1)) {
                                // the y-shell test applies only to physical halo rows; ghost rows
                                // (slab sides) are real grid rows whose x-halo cells are Dirichlet
                                const bool sh = y_alloc && (!y_out || y_shell) && ((shell_mask >> j) & 1);
                                done[j] = sh ? rowp[col[j]] : T(0);
                            }
                        }
                    }
                    if (l < K) {
#pragma unroll
                        for (int j = 0; j < F2_VX; j++) v[j] = done[j];
                        edge = T(0);                          // beyond level 0 the strip edge is garbage
                    } else if (yc >= ys0 && yc < ys1) {
                        T* rowp = P.dst + P.origin + (int64_t)yc * P.sy;
#pragma unroll
                        for (int j = 0; j < F2_VX; j++)
                            if ((store_mask >> j) & 1) rowp[col[j]] = done[j];
                    }
                }
            }
        }
    }
    if (lane == 0) {
        const unsigned retired = atomicAdd(&P.counter[1], 1u);
        if (retired == (unsigned)P.total_warps - 1) {
            atomicExch(&P.counter[0], 0u);
            atomicExch(&P.counter[1], 0u);
        }
    }
}

}  // namespace sb
