// K3/K4 -- fused 3D sweep (r = 1 star 7-point or box 27-point), K time
// steps per HBM round trip: 2.5D streaming along z with temporal blocking.
//
// Replaces the reference's 3D path, which has no blocking at all
// (harness.py:127-136 runs 3D untiled) and sums the canonical offsets with
// numpy passes (kernels.py:103-108).
//
// Structure (one work item = one xy tile x one z segment; persistent CTAs
// claim items from an atomic queue):
//  * level-0 planes arrive by TMA (cp.async.bulk.tensor.3d, mbarrier ring of
//    NS0 slots, out-of-bounds boxes zero-filled) as a PW x PH box: the 64 x 32
//    computed region plus one ring;
//  * every level l = 1..K keeps, per thread, two pending partial-sum planes in
//    registers (push form along z): when the level-(l-1) plane a arrives, its
//    in-plane neighbourhood is read from shared memory ONCE and folded into
//    output planes a+1 (dz=-1, first terms), a (dz=0) and a-1 (dz=+1, last
//    terms -> complete).  Each output therefore still sums its terms in
//    canonical (dz, dy, dx) lexicographic order (bit-exact in EXACT mode);
//  * the completed level-l plane goes to a shared plane read by level l+1
//    in the same step; level K goes to global memory.
//  * 256 threads x (2 x 4) points cover the 64 x 32 computed region at every
//    level; valid data shrinks by one ring per level, so the output tile is
//    (66 - 2K) x (34 - 2K) (overlapped-tile recompute in x and y).
//
// Boundaries: an emitted value at a position outside the interior on a
// physical side is replaced by the Dirichlet halo value (read from global;
// the halo is the same at every level), beyond the halo shell by 0 (never
// used by a valid output).  Slab (ghost) sides along z are computed normally.
#pragma once
#include <cuda.h>

#include "common.cuh"

#ifndef SB_F3_PAIR
#define SB_F3_PAIR 1    // fp32 box FMA mode: paired accumulators, FFMA2 with broadcast input
#endif


namespace sb {

constexpr int F3_CW = 64;        // computed region width (x)
constexpr int F3_PW = 68;        // shared plane width: ring + region + pad (16 B rows)
#ifndef SB_F3_NS0
#define SB_F3_NS0 3     // measured: 3 >= 4 > 2 on every C4/C5 depth (C5 fp32 k=2 +4%, fp64 +1-2%)
#endif
#ifndef SB_F3_DBL
#define SB_F3_DBL 0     // double-buffered level planes: no end-of-plane barrier
#endif
constexpr int F3_NS0 = SB_F3_NS0;   // TMA ring depth (level-0 planes)
constexpr int F3_NB = SB_F3_DBL ? 2 : 1;   // buffers per level plane

// CTA geometry: NTY thread rows of 32 threads, 2 x 4 points per thread, so the
// computed region is 64 x (4*NTY) and the plane box 68 x (4*NTY + 2).
template <int NTY, int RPT = 4>
struct F3Geo {
    static constexpr int THREADS = 32 * NTY;
    static constexpr int CH = RPT * NTY;        // computed region height (y)
    static constexpr int PH = CH + 2;           // shared plane height: ring + region + ring
};

// Plane stride in elements: TMA destinations must be 128 B aligned.
template <typename T, int NTY, int RPT = 4>
struct F3Plane {
    static constexpr int ELEMS = ((F3_PW * F3Geo<NTY, RPT>::PH * (int)sizeof(T) + 127) / 128) * 128 / (int)sizeof(T);
    static constexpr unsigned BOX_BYTES = F3_PW * F3Geo<NTY, RPT>::PH * sizeof(T);
};
template <typename T, int K, int NTY, int RPT = 4>
constexpr int f3_smem_bytes() { return (F3_NS0 + F3_NB * (K - 1)) * F3Plane<T, NTY, RPT>::ELEMS * (int)sizeof(T); }

template <typename T>
struct Fused3DParams {
    const T* src;            // buffer bases (element (z,y,x) at origin + z*sz + y*sy + x)
    T* dst;
    int64_t origin, sz, sy;
    int nx, ny, nz;
    int ax, ry, hz;          // allocation coordinates of interior (0,0,0): col, row, plane
    int hz_hi;               // planes allocated above the interior (halo or ghost)
    int phys_lo, phys_hi;    // z sides: physical halo (1) or ghost (0)
    int ghost_lo, ghost_hi;  // ghost depth on slab sides (0 on physical sides)
    int tiles_x, tiles_y, nseg, lz;
    int z0, z1;              // output planes [z0, z1) of this launch (range launches)
    int items;
    int total_ctas;
    unsigned int* counter;   // [0] next item, [1] retired CTAs
    T w[27];                 // w[(dz+1)*9 + (dy+1)*3 + (dx+1)]; star uses 7 entries
    unsigned long long wp[18];   // fp32 box: weight pairs of f3_push_pair
};

// Output tile geometry.  The TMA box's first column (x0 - K) must be 16 B
// aligned (measured: an unaligned innermost coordinate traps with "illegal
// instruction"), so the tile pitch is a multiple of the 16 B vector and the
// tiles start at X0 <= 0 with X0 == K (mod VEC); columns x < 0 are not stored.
template <typename T, int K, int NTY, int RPT = 4>
struct F3Tile {
    static constexpr int VEC = 16 / (int)sizeof(T);
    static constexpr int TXO = ((F3_CW - 2 * (K - 1)) / VEC) * VEC;   // output tile width
    static constexpr int TYO = F3Geo<NTY, RPT>::CH - 2 * (K - 1);     // output tile height
    static constexpr int X0 = (K % VEC == 0) ? 0 : (K % VEC) - VEC;  // first tile's x origin
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                            int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(smem_dst)),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// Fold one arriving plane into a level's pending sums (push form along z),
// streaming the plane one row (4 values) at a time into the point-rows it
// touches, so only 4 plane values are live.  Term-major order: consecutive
// FMAs in the instruction stream belong to independent points (ILP 2*RPT).  Rows arrive in increasing dy and dx
// ascends within a row, so each accumulator still receives its terms in
// canonical (dy, dx) order within its dz group.
template <typename T, bool BOX, bool FMA, int RPT = 4>
__device__ __forceinline__ void f3_push_rows(const T* plane, int tx, int ty, T (&Pm)[RPT][2], T (&P0)[RPT][2],
                                             T (&done)[RPT][2], const T* w) {
    T nx[RPT][2];
#pragma unroll
    for (int r = 0; r < RPT + 2; r++) {
        T u[4];
        const T* row = plane + (RPT * ty + r) * F3_PW + 2 * tx;
        if (sizeof(T) == 8) {
            const double2 a = *reinterpret_cast<const double2*>(row);
            const double2 b = *reinterpret_cast<const double2*>(row + 2);
            u[0] = (T)a.x; u[1] = (T)a.y; u[2] = (T)b.x; u[3] = (T)b.y;
        } else {
            const float2 a = *reinterpret_cast<const float2*>(row);
            const float2 b = *reinterpret_cast<const float2*>(row + 2);
            u[0] = (T)a.x; u[1] = (T)a.y; u[2] = (T)b.x; u[3] = (T)b.y;
        }
#pragma unroll
        for (int i = 0; i < RPT; i++) {
            const int dy = r - i - 1;                   // this row's dy for point-row i
            if (dy < -1 || dy > 1) continue;
#pragma unroll
            for (int dx = -1; dx <= 1; dx++) {
                const int q = (dy + 1) * 3 + (dx + 1);
#pragma unroll
                for (int j = 0; j < 2; j++) {
                    const T x = u[j + 1 + dx];
                    if (BOX) {
                        Pm[i][j] = acc_term<T, FMA>(Pm[i][j], w[18 + q], x);   // dz=+1: completes a-1
                        P0[i][j] = acc_term<T, FMA>(P0[i][j], w[9 + q], x);    // dz= 0
                        nx[i][j] = q == 0 ? acc_first<T, FMA>(w[0], x)         // dz=-1: starts a+1
                                          : acc_term<T, FMA>(nx[i][j], w[q], x);
                    } else {
                        if (q == 4) {
                            Pm[i][j] = acc_term<T, FMA>(Pm[i][j], w[22], x);   // (1,0,0)
                            nx[i][j] = acc_first<T, FMA>(w[4], x);             // (-1,0,0)
                        }
                        if (q == 1 || q == 3 || q == 4 || q == 5 || q == 7)    // (0,dy,dx) of the star
                            P0[i][j] = acc_term<T, FMA>(P0[i][j], w[9 + q], x);
                    }
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < RPT; i++)
#pragma unroll
        for (int j = 0; j < 2; j++) {
            done[i][j] = Pm[i][j];
            Pm[i][j] = P0[i][j];
            P0[i][j] = nx[i][j];
        }
}

// ---- fp32 box, FMA mode: paired accumulators (FFMA2 with a broadcast input).
// A thread's two x-adjacent points keep each pending sum as one 64-bit register
// pair (point j=0 low, j=1 high).  An input value x in row column c feeds
// point j=0 with dx = c-1 and point j=1 with dx = c-2, i.e. the SAME x with two
// different weights: one FFMA2 (weight pair from the constant bank, x
// broadcast from a 32-bit register -- no packing moves) updates both points;
// the edge columns c=0 / c=3 feed one point and take a scalar FFMA on that
// half.  18 instead of 27 FMA-pipe instructions per point pair and dz group.
// Each half still receives its terms in canonical (dy, dx) order; the first
// term is an FMA onto +0 (equal to the rounded product up to the sign of zero).
__device__ __forceinline__ unsigned long long f2_fma_bcast(unsigned long long w2, float x, unsigned long long acc) {
    unsigned long long xx, d;
    asm("mov.b64 %0, {%1, %1};" : "=l"(xx) : "f"(x));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(w2), "l"(xx), "l"(acc));
    return d;
}
template <int HALF>
__device__ __forceinline__ unsigned long long f2_fma_half(float w, float x, unsigned long long acc) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc));
    if (HALF == 0) lo = __fmaf_rn(w, x, lo);
    else hi = __fmaf_rn(w, x, hi);
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}

// wp[(b*3 + dy+1)*2 + c-1] = (w[9b + (dy+1)*3 + c], w[9b + (dy+1)*3 + c-1]) for c in {1, 2}
template <int RPT = 4>
__device__ __forceinline__ void f3_push_pair(const float* plane, int tx, int ty, unsigned long long (&Pm)[RPT],
                                             unsigned long long (&P0)[RPT], float (&done)[RPT][2],
                                             const float* w, const unsigned long long* wp) {
    unsigned long long nx[RPT];
#pragma unroll
    for (int i = 0; i < RPT; i++) nx[i] = 0ull;
#pragma unroll
    for (int r = 0; r < RPT + 2; r++) {
        const float* row = plane + (RPT * ty + r) * F3_PW + 2 * tx;
        const float2 a = *reinterpret_cast<const float2*>(row);
        const float2 b = *reinterpret_cast<const float2*>(row + 2);
        const float u[4] = {a.x, a.y, b.x, b.y};   // columns 2tx-1 .. 2tx+2
#pragma unroll
        for (int i = 0; i < RPT; i++) {
            const int dy = r - i - 1;
            if (dy < -1 || dy > 1) continue;
            const int q0 = (dy + 1) * 3;          // (dy, dx=-1)
            // c = 0: point 0, dx = -1
            Pm[i] = f2_fma_half<0>(w[18 + q0], u[0], Pm[i]);
            P0[i] = f2_fma_half<0>(w[9 + q0], u[0], P0[i]);
            nx[i] = f2_fma_half<0>(w[q0], u[0], nx[i]);
            // c = 1, 2: both points (dx = c-1 for point 0, c-2 for point 1)
#pragma unroll
            for (int c = 1; c <= 2; c++) {
                Pm[i] = f2_fma_bcast(wp[(2 * 3 + dy + 1) * 2 + c - 1], u[c], Pm[i]);
                P0[i] = f2_fma_bcast(wp[(1 * 3 + dy + 1) * 2 + c - 1], u[c], P0[i]);
                nx[i] = f2_fma_bcast(wp[(0 * 3 + dy + 1) * 2 + c - 1], u[c], nx[i]);
            }
            // c = 3: point 1, dx = +1
            Pm[i] = f2_fma_half<1>(w[18 + q0 + 2], u[3], Pm[i]);
            P0[i] = f2_fma_half<1>(w[9 + q0 + 2], u[3], P0[i]);
            nx[i] = f2_fma_half<1>(w[q0 + 2], u[3], nx[i]);
        }
    }
#pragma unroll
    for (int i = 0; i < RPT; i++) {
        asm("mov.b64 {%0, %1}, %2;" : "=f"(done[i][0]), "=f"(done[i][1]) : "l"(Pm[i]));
        Pm[i] = P0[i];
        P0[i] = nx[i];
    }
}

template <typename T, bool PAIR, int RPT> struct F3Pend { T v[RPT][2]; };
template <typename T, int RPT> struct F3Pend<T, true, RPT> { unsigned long long v[RPT]; };

// RPT: point rows per thread (each thread owns 2 x RPT points of the region)
template <typename T, bool BOX, int K, bool FMA, int MINB, int NTY, int RPT = 4>
__global__ void __launch_bounds__(F3Geo<NTY, RPT>::THREADS, MINB)
fused3d_kernel(const __grid_constant__ CUtensorMap tmap, const Fused3DParams<T> P) {
    constexpr int PLANE = F3Plane<T, NTY, RPT>::ELEMS;
    constexpr unsigned PLANE_BYTES = F3Plane<T, NTY, RPT>::BOX_BYTES;
    constexpr int NPT = 2 * RPT;                  // points per thread
    using TL = F3Tile<T, K, NTY, RPT>;
    extern __shared__ __align__(1024) unsigned char smem3d[];   // TMA destinations: 128 B aligned
    T* s0 = reinterpret_cast<T*>(smem3d);              // NS0 level-0 slots
    T* sl = s0 + F3_NS0 * PLANE;                       // levels 1..K-1, one plane each
    __shared__ uint64_t bar[F3_NS0];
    __shared__ unsigned s_item;

    const int tid = threadIdx.x;
    const int tx = tid & 31, ty = tid >> 5;
    if (tid == 0) {
        for (int i = 0; i < F3_NS0; i++) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
    }
    __syncthreads();

    unsigned gstep = 0;   // CTA-lifetime step counter: slot = g % NS0, parity = (g / NS0) & 1
    for (;;) {
        if (tid == 0) s_item = atomicAdd(&P.counter[0], 1u);
        __syncthreads();
        const unsigned item = s_item;
        if (item >= (unsigned)P.items) break;
        const int tix = item % P.tiles_x;
        const int tiy = (item / P.tiles_x) % P.tiles_y;
        const int seg = item / (P.tiles_x * P.tiles_y);
        const int x0 = TL::X0 + tix * TL::TXO, y0 = tiy * TL::TYO;   // output tile origin
        const int xc = x0 - (K - 1), yc = y0 - (K - 1);         // computed region origin
        // per-thread masks of its 8 points outside the x/y interior / on the halo shell,
        // and their in-plane offsets (for the Dirichlet values)
        // and the points this thread stores at level K (inside the output tile and the grid)
        unsigned out_mask = 0, shell_mask = 0, store_mask = 0;
#pragma unroll
        for (int q = 0; q < NPT; q++) {
            const int y = yc + RPT * ty + (q >> 1), x = xc + 2 * tx + (q & 1);
            const bool out = x < 0 || x >= P.nx || y < 0 || y >= P.ny;
            const bool shell = x >= -1 && x <= P.nx && y >= -1 && y <= P.ny;
            const int ri = y - y0, cj = x - x0;
            const bool st = ri >= 0 && ri < TL::TYO && cj >= 0 && cj < TL::TXO && !out;
            out_mask |= (unsigned)out << q;
            shell_mask |= (unsigned)shell << q;
            store_mask |= (unsigned)st << q;
        }
        // in-plane element offset of point (0, 0); point q is + (q >> 1) * sy + (q & 1)
        const int64_t hbase = P.origin + (int64_t)(yc + RPT * ty) * P.sy + (xc + 2 * tx);
        auto hoff = [&](int q) -> int64_t { return hbase + (q >> 1) * P.sy + (q & 1); };
        T* const obase = P.dst + hbase;        // + zc * sz per plane
        int zs0 = P.z0 + seg * P.lz, zs1 = min(P.z1, zs0 + P.lz);   // output planes
        // slab sides: the first/last segment also produces nothing below 0 / above nz
        const int p_first = zs0 - K;
        const int M = (zs1 - zs0) + 2 * K;                      // level-0 arrivals

        auto issue = [&](int t) {
            const unsigned g = gstep + t;
            uint64_t* b = &bar[g % F3_NS0];
            mbar_expect_tx(b, PLANE_BYTES);
            tma_load_3d(s0 + (g % F3_NS0) * PLANE, &tmap, b, P.ax + x0 - K, P.ry + y0 - K, P.hz + p_first + t);
        };
        if (tid == 0)
            for (int t = 0; t < F3_NS0 && t < M; t++) issue(t);

        constexpr bool PAIR = sizeof(T) == 4 && FMA && BOX && SB_F3_PAIR;
        F3Pend<T, PAIR, RPT> Pm[K], P0[K];
#pragma unroll
        for (int l = 0; l < K; l++) {
            if constexpr (PAIR) {
#pragma unroll
                for (int i = 0; i < RPT; i++) Pm[l].v[i] = P0[l].v[i] = 0ull;
            } else {
#pragma unroll
                for (int i = 0; i < RPT; i++)
#pragma unroll
                    for (int j = 0; j < 2; j++) Pm[l].v[i][j] = P0[l].v[i][j] = T(0);
            }
        }

        for (int t = 0; t < M; t++) {
            const unsigned g = gstep + t;
            mbar_wait(&bar[g % F3_NS0], (g / F3_NS0) & 1);
            const int a0 = p_first + t;   // level-0 plane that arrived
#pragma unroll
            for (int l = 1; l <= K; l++) {
                const T* in = (l == 1) ? s0 + (g % F3_NS0) * PLANE
                                       : sl + ((l - 2) * F3_NB + (SB_F3_DBL ? (t & 1) : 0)) * PLANE;
                T done[RPT][2];
                if constexpr (PAIR)
                    f3_push_pair<RPT>(reinterpret_cast<const float*>(in), tx, ty, Pm[l - 1].v, P0[l - 1].v,
                                 reinterpret_cast<float(&)[RPT][2]>(done), reinterpret_cast<const float*>(P.w), P.wp);
                else
                    f3_push_rows<T, BOX, FMA, RPT>(in, tx, ty, Pm[l - 1].v, P0[l - 1].v, done, P.w);
                const int zc = a0 - l;    // completed level-l plane
                const bool z_out = (P.phys_lo && zc < 0) || (P.phys_hi && zc >= P.nz);
                if (z_out) {   // uniform: a physical halo plane, every value is Dirichlet
                    const bool z_shell = zc >= -1 && zc <= P.nz;
#pragma unroll
                    for (int q = 0; q < NPT; q++) {
                        T hv = T(0);
                        if (z_shell && ((shell_mask >> q) & 1)) hv = P.src[hoff(q) + (int64_t)zc * P.sz];
                        done[q >> 1][q & 1] = hv;
                    }
                } else if (out_mask) {   // only threads owning points outside the x/y interior
                    // planes below/above the allocation (first completions of a ghost-side
                    // segment) are garbage that never reaches a valid output: no load
                    const bool z_alloc = zc >= -P.hz && zc < P.nz + P.hz_hi;
#pragma unroll
                    for (int q = 0; q < NPT; q++)
                        if ((out_mask >> q) & 1)
                            done[q >> 1][q & 1] =
                                (z_alloc && ((shell_mask >> q) & 1)) ? P.src[hoff(q) + (int64_t)zc * P.sz] : T(0);
                }
                if (l < K) {
                    T* o = sl + ((l - 1) * F3_NB + (SB_F3_DBL ? (t & 1) : 0)) * PLANE;
#pragma unroll
                    for (int i = 0; i < RPT; i++)
#pragma unroll
                        for (int j = 0; j < 2; j++) o[(RPT * ty + i + 1) * F3_PW + 2 * tx + j + 1] = done[i][j];
                } else if (zc >= zs0 && zc < zs1 && store_mask) {
                    T* row = obase + (int64_t)zc * P.sz;
#pragma unroll
                    for (int i = 0; i < RPT; i++) {
#pragma unroll
                        for (int j = 0; j < 2; j++)
                            if ((store_mask >> (2 * i + j)) & 1) row[j] = done[i][j];
                        row += P.sy;
                    }
                }
                if (l < K || K == 1) __syncthreads();
                if (l == 1 && tid == 0 && t + F3_NS0 < M)
                    issue(t + F3_NS0);   // slot consumed by level 1
            }
            if (K > 1 && !SB_F3_DBL) __syncthreads();   // level K read sl[K-2] before the next step rewrites it
        }
        gstep += M;
    }
    if (tid == 0) {
        const unsigned retired = atomicAdd(&P.counter[1], 1u);
        if (retired == (unsigned)P.total_ctas - 1) {
            atomicExch(&P.counter[0], 0u);
            atomicExch(&P.counter[1], 0u);
        }
    }
}

}  // namespace sb
