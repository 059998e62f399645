// K5b -- 3D 27-point box sweep, two time steps per HBM round trip, with
// ring-only recompute (C5: BASELINE configs[4], fp64 and fp32).
//
// Replaces the 3D scalar_step loop (kernels.py:120-134; the reference runs 3D
// untiled, harness.py:127-136; arithmetic kernels.py:103-108).
//
// A 27-point box costs 27 FMAs per update whatever the blocking (no
// composition helps: two steps of it are a 125-point box), so at k = 2 the
// sweep is FP64-pipe bound and every redundant level-1 point is lost
// throughput.  The level-by-level kernel K3 (fused3d.cuh) computes a fixed
// 64 x 16 region at both levels and keeps the (66-2K) x (34-2K)-style shrunken
// tile: 24% of its DFMAs were redundant on C5 (overlap + x-tile quantisation).
// Here the OUTPUT tile is exactly 64 x TY (TY = 4 x warps; 768 = 12 x 64 =
// 24 x 32, so no quantisation on C5) and level 1 computes exactly the output
// tile grown by its 1-point ring:
//   * every thread owns 2 x 4 points at both levels (level 1 shifted one
//     column left so every shared-memory access is a 16 B (fp64) / 8 B (fp32)
//     aligned vector: level-1 main columns [x0-1, x0+63), level 2 [x0, x0+64));
//   * the rest of the level-1 ring -- rows y0-1 and y0+TY over the main
//     columns, and columns x0+63, x0+64 over rows y0-1 .. y0+TY -- is a set of
//     "ring jobs" of 2 x-adjacent points per lane, one job per warp for the
//     first few warps, pushed with the same code (1 point row instead of 4);
//   => level-1 work = (64 + 2) x (TY + 2) points for 64 x TY outputs:
//      6% redundant DFMAs at TY = 32 (9% at TY = 16) instead of 24%.
// Everything else is the 2.5D z-stream of K3: level-0 planes arrive by TMA
// (68 x (TY+4) boxes fp64, 72 x (TY+4) fp32, mbarrier ring, OOB zero fill);
// each level keeps two pending partial-sum planes per point in registers
// (push form along z: an arriving plane's in-plane neighbourhood is read once
// from shared memory and folded into outputs a+1, a, a-1); the completed
// level-1 plane goes to a double-buffered shared plane (one barrier per
// arriving plane), level 2 to global memory with vector stores.
// Canonical (dz, dy, dx) order per output is kept (EXACT mode bit-identical).
//
// fp32, FMA mode: the two x-adjacent points of a lane keep every pending sum
// as one 64-bit register pair and take their terms as ONE packed FFMA2 with
// the weight broadcast to both halves and the two inputs (u[c+dx], u[c+1+dx])
// as a register pair -- (u-1,u0) and (u1,u2) straight from two 8 B shared
// loads, (u0,u1) assembled by two moves -- 27 FFMA2 per point pair and plane,
// half the FMA-pipe issue slots of scalar FFMA.
//
// Boundaries: level-1 values at positions outside the interior on a physical
// side are replaced by the Dirichlet halo value (read from global; the halo is
// the same at every level), beyond the halo shell by 0 (never used by a valid
// output).  Slab (ghost) sides along z are computed like interior planes.
#pragma once
#include <cuda.h>

#include <type_traits>

#include "common.cuh"
#include "fused3d.cuh"   // TMA / mbarrier helpers

namespace sb {

#ifndef SB_B3_NS0
#define SB_B3_NS0 3
#endif
constexpr int B3_NS0 = SB_B3_NS0;   // TMA ring depth (level-0 planes)
// fp32 pair path: the dx = 0 term of a point pair as two scalar FFMAs on the
// halves of the accumulator pair (1) or as one FFMA2 on an assembled /
// shifted-copy input pair (0)
#ifndef SB_B3_MIDSCALAR
#define SB_B3_MIDSCALAR 1
#endif
constexpr bool B3_MIDSCALAR = SB_B3_MIDSCALAR != 0;

template <typename T, int NW>
struct B3Geo {
    static constexpr int THREADS = 32 * NW;
    static constexpr int TY = 4 * NW;                        // output tile height
    static constexpr int XOFF = sizeof(T) == 8 ? 2 : 4;      // box starts at x0 - XOFF (16 B aligned)
    static constexpr int PW = 64 + 2 * XOFF;                 // box / plane width: 68 fp64, 72 fp32
    static constexpr int PH = TY + 4;                        // box height: rows y0-2 .. y0+TY+1
    static constexpr int ELEMS = ((PW * PH * (int)sizeof(T) + 127) / 128) * 128 / (int)sizeof(T);
    static constexpr unsigned BOX_BYTES = PW * PH * sizeof(T);
    static constexpr int NJOBS = 2 + (TY + 2 + 31) / 32;     // ring jobs: 2 rows + column pairs
    // level-0 slots + two level-1 planes (+ two shifted copies for the fp32 pair path)
    static constexpr int SMEM = (B3_NS0 + (sizeof(T) == 4 && !B3_MIDSCALAR ? 4 : 2)) * ELEMS * (int)sizeof(T);
};

constexpr int B3_MAX_SEG = 47;

template <typename T>
struct Box3DParams {
    const T* src;
    T* dst;
    int64_t origin, sz, sy;
    int nx, ny, nz;
    int ax, ry, hz, hz_hi;   // allocation coordinates of interior (0,0,0); planes above
    int phys_lo, phys_hi;
    int tiles_x, tiles_y, nseg, items, total_ctas;
    // z segments of this launch's output planes: segment s = [zb[s], zb[s+1]), the same for
    // every xy tile; lengths decrease (guided schedule: the last items are short)
    int zb[B3_MAX_SEG + 1];
    unsigned int* counter;   // [0] next item, [1] retired CTAs
    T w[27];                 // w[(dz+1)*9 + (dy+1)*3 + (dx+1)]
    unsigned long long wpp[27];   // fp32: (w, w) pairs for the packed FFMA2 push
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Pending sums of RPT point rows x 2 columns: fp64/fp32 scalars, or (fp32
// FMA mode) one 64-bit register pair per point row (column 0 low, 1 high).
template <typename T, bool PAIR, int RPT> struct B3Acc {
    T v[RPT][2];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < RPT; i++) v[i][0] = v[i][1] = T(0);
    }
    __device__ __forceinline__ T get(int i, int j) const { return v[i][j]; }
    __device__ __forceinline__ void set(int i, int j, T x) { v[i][j] = x; }
};
template <typename T, int RPT> struct B3Acc<T, true, RPT> {
    unsigned long long v[RPT];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < RPT; i++) v[i] = 0ull;
    }
    __device__ __forceinline__ T get(int i, int j) const {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v[i]));
        return (T)(j ? hi : lo);
    }
    __device__ __forceinline__ void set(int i, int j, T x) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v[i]));
        if (j) hi = (float)x; else lo = (float)x;
        asm("mov.b64 %0, {%1, %2};" : "=l"(v[i]) : "f"(lo), "f"(hi));
    }
};

// Fold one arriving plane a into three pending-sum sets (push form along z):
// C = output a-1 (its dz=+1 terms complete it), K = output a (dz=0), S =
// output a+1 (dz=-1, started here).  `p` points at the (row y-1, column x-1)
// neighbour of the lane's first point; rows are PW apart.  Rows arrive in
// increasing dy and dx ascends within a row, so every accumulator receives
// its terms in canonical (dz, dy, dx) order.  The caller rotates the roles
// of the three sets from plane to plane (no register moves).
template <typename T, bool FMA, int RPT, int PW>
__device__ __forceinline__ void b3_push(const T* p, B3Acc<T, false, RPT>& C, B3Acc<T, false, RPT>& K,
                                        B3Acc<T, false, RPT>& S, const T* w) {
#pragma unroll
    for (int r = 0; r < RPT + 2; r++) {
        T u[4];
        if constexpr (sizeof(T) == 8) {
            const double2 a = *reinterpret_cast<const double2*>(p + r * PW);
            const double2 b = *reinterpret_cast<const double2*>(p + r * PW + 2);
            u[0] = a.x; u[1] = a.y; u[2] = b.x; u[3] = b.y;
        } else {
            const float2 a = *reinterpret_cast<const float2*>(p + r * PW);
            const float2 b = *reinterpret_cast<const float2*>(p + r * PW + 2);
            u[0] = a.x; u[1] = a.y; u[2] = b.x; u[3] = b.y;
        }
#pragma unroll
        for (int i = 0; i < RPT; i++) {
            const int dy = r - i - 1;
            if (dy < -1 || dy > 1) continue;
#pragma unroll
            for (int dx = -1; dx <= 1; dx++) {
                const int q = (dy + 1) * 3 + (dx + 1);
#pragma unroll
                for (int j = 0; j < 2; j++) {
                    const T x = u[j + 1 + dx];
                    C.v[i][j] = acc_term<T, FMA>(C.v[i][j], w[18 + q], x);
                    K.v[i][j] = acc_term<T, FMA>(K.v[i][j], w[9 + q], x);
                    S.v[i][j] = q == 0 ? acc_first<T, FMA>(w[0], x) : acc_term<T, FMA>(S.v[i][j], w[q], x);
                }
            }
        }
    }
}

// fp32 FMA mode: packed pairs.  Each term of both points is ONE FFMA2 with
// the weight broadcast (w, w) and the input pair (u[dx], u[dx+1]) relative to
// the lane's first column.  (u-1, u0) and (u1, u2) are aligned 8 B loads;
// (u0, u1) comes from `pm` (a copy of the plane shifted by one column, when
// the producer wrote one) or is assembled from the other two.
__device__ __forceinline__ unsigned long long b3_ffma2(unsigned long long w2, unsigned long long x2,
                                                       unsigned long long acc) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(w2), "l"(x2), "l"(acc));
    return d;
}

// acc.lo += w * u0, acc.hi += w * u1: the dx = 0 term of a point pair, whose
// inputs (u0, u1) straddle the two aligned 8 B loads.  As ONE FFMA2 the input
// pair has to be assembled in a fresh aligned register pair, and ptxas rebuilds
// it for every use (two moves per FFMA2: ~100 MOV / IMAD.MOV per warp and plane
// beside 243 FFMA2 in the C5 kernel); two scalar FFMAs on the halves of the
// accumulator pair take the same two FMA-pipe cycles and no moves.
__device__ __forceinline__ unsigned long long b3_fma_mid(unsigned long long acc, float w, float u0, float u1) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc));
    lo = fmaf(w, u0, lo);
    hi = fmaf(w, u1, hi);
    unsigned long long d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
    return d;
}

template <int RPT, int PW>
__device__ __forceinline__ void b3_push_pair_mid(const float* p, B3Acc<float, true, RPT>& C, B3Acc<float, true, RPT>& K,
                                                 B3Acc<float, true, RPT>& S, const unsigned long long* wpp,
                                                 const float* w) {
#pragma unroll
    for (int r = 0; r < RPT + 2; r++) {
        const unsigned long long a = *reinterpret_cast<const unsigned long long*>(p + r * PW);       // (u-1, u0)
        const unsigned long long b = *reinterpret_cast<const unsigned long long*>(p + r * PW + 2);   // (u1, u2)
        float um, u0, u1, u2;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(um), "=f"(u0) : "l"(a));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(u1), "=f"(u2) : "l"(b));
        (void)um;
        (void)u2;
#pragma unroll
        for (int i = 0; i < RPT; i++) {
            const int dy = r - i - 1;
            if (dy < -1 || dy > 1) continue;
            const int q = (dy + 1) * 3;
            C.v[i] = b3_ffma2(wpp[18 + q], a, C.v[i]);
            K.v[i] = b3_ffma2(wpp[9 + q], a, K.v[i]);
            S.v[i] = b3_ffma2(wpp[q], a, q == 0 ? 0ull : S.v[i]);
            C.v[i] = b3_fma_mid(C.v[i], w[18 + q + 1], u0, u1);
            K.v[i] = b3_fma_mid(K.v[i], w[9 + q + 1], u0, u1);
            S.v[i] = b3_fma_mid(S.v[i], w[q + 1], u0, u1);
            C.v[i] = b3_ffma2(wpp[18 + q + 2], b, C.v[i]);
            K.v[i] = b3_ffma2(wpp[9 + q + 2], b, K.v[i]);
            S.v[i] = b3_ffma2(wpp[q + 2], b, S.v[i]);
        }
    }
}

template <int RPT, int PW, bool SHIFTED>
__device__ __forceinline__ void b3_push_pair(const float* p, const float* pm, B3Acc<float, true, RPT>& C,
                                             B3Acc<float, true, RPT>& K, B3Acc<float, true, RPT>& S,
                                             const unsigned long long* wpp) {
#pragma unroll
    for (int r = 0; r < RPT + 2; r++) {
        const unsigned long long a = *reinterpret_cast<const unsigned long long*>(p + r * PW);       // (u-1, u0)
        const unsigned long long b = *reinterpret_cast<const unsigned long long*>(p + r * PW + 2);   // (u1, u2)
        unsigned long long m;                                                                       // (u0, u1)
        if constexpr (SHIFTED) {
            m = *reinterpret_cast<const unsigned long long*>(pm + r * PW);
        } else {
            asm("{\n\t.reg .b32 al, ah, bl, bh;\n\t"
                "mov.b64 {al, ah}, %1;\n\t"
                "mov.b64 {bl, bh}, %2;\n\t"
                "mov.b64 %0, {ah, bl};\n\t}"
                : "=l"(m) : "l"(a), "l"(b));
        }
#pragma unroll
        for (int i = 0; i < RPT; i++) {
            const int dy = r - i - 1;
            if (dy < -1 || dy > 1) continue;
#pragma unroll
            for (int dx = -1; dx <= 1; dx++) {
                const int q = (dy + 1) * 3 + (dx + 1);
                const unsigned long long x2 = dx < 0 ? a : (dx == 0 ? m : b);
                C.v[i] = b3_ffma2(wpp[18 + q], x2, C.v[i]);
                K.v[i] = b3_ffma2(wpp[9 + q], x2, K.v[i]);
                S.v[i] = b3_ffma2(wpp[q], x2, q == 0 ? 0ull : S.v[i]);
            }
        }
    }
}

template <typename T, bool PAIR, bool FMA, int RPT, int PW, bool SHIFTED = false>
__device__ __forceinline__ void b3_fold(const T* p, const T* pm, B3Acc<T, PAIR, RPT>& C, B3Acc<T, PAIR, RPT>& K,
                                        B3Acc<T, PAIR, RPT>& S, const Box3DParams<T>& P) {
    if constexpr (PAIR && B3_MIDSCALAR)
        b3_push_pair_mid<RPT, PW>(reinterpret_cast<const float*>(p), C, K, S, P.wpp,
                                  reinterpret_cast<const float*>(P.w));
    else if constexpr (PAIR)
        b3_push_pair<RPT, PW, SHIFTED>(reinterpret_cast<const float*>(p), reinterpret_cast<const float*>(pm), C, K,
                                       S, P.wpp);
    else
        b3_push<T, FMA, RPT, PW>(p, C, K, S, P.w);
}

// Store the two x-adjacent values of point row i (aligned: 16 B fp64, 8 B fp32).
template <typename T, bool PAIR, int RPT>
__device__ __forceinline__ void b3_st2(T* p, const B3Acc<T, PAIR, RPT>& A, int i) {
    if constexpr (PAIR) *reinterpret_cast<unsigned long long*>(p) = A.v[i];
    else if constexpr (sizeof(T) == 8) *reinterpret_cast<double2*>(p) = make_double2(A.v[i][0], A.v[i][1]);
    else *reinterpret_cast<float2*>(p) = make_float2(A.v[i][0], A.v[i][1]);
}

template <typename T, bool FMA, int NW, int MINB, bool U3>
__global__ void __launch_bounds__(32 * NW, MINB)
box3d_kernel(const __grid_constant__ CUtensorMap tmap, const Box3DParams<T> P) {
    using G = B3Geo<T, NW>;
    constexpr int PW = G::PW, TY = G::TY, PLANE = G::ELEMS;
    constexpr bool PAIR = sizeof(T) == 4 && FMA;
    // fp32 pairs: level-1 planes also get a copy shifted right by one column,
    // so level 2 loads all three input pairs aligned
    constexpr bool SHIFTED = PAIR && !B3_MIDSCALAR;
    constexpr bool UNROLL3 = U3;
    extern __shared__ __align__(1024) unsigned char smem_b3[];
    T* s0 = reinterpret_cast<T*>(smem_b3);      // B3_NS0 level-0 slots
    T* s1 = s0 + B3_NS0 * PLANE;                 // two level-1 planes (+ two shifted copies)
    __shared__ uint64_t bar[B3_NS0];
    __shared__ unsigned s_item;

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int i = 0; i < B3_NS0; i++) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
    }
    __syncthreads();

    // ring job of this warp (warp-uniform kind; lane activity per job):
    //   job 0: level-1 row y0-1,  columns x0-1+2*lane (+1)
    //   job 1: level-1 row y0+TY, same columns
    //   job 2+: columns x0+63, x0+64 of level-1 row y0-1 + lane + 32*(job-2)
    // Jobs rotate with the CTA index so that the warps without one (NJOBS < NW)
    // fall on different SM sub-partitions in co-resident CTAs.
    const int jw = (warp + (int)blockIdx.x) % NW;
    const int job = jw < G::NJOBS ? jw : -1;
    int rj_dy, rj_dx;   // ring-job point (0) offset from (y0, x0)
    if (job == 0) { rj_dy = -1; rj_dx = -1 + 2 * lane; }
    else if (job == 1) { rj_dy = TY; rj_dx = -1 + 2 * lane; }
    else { rj_dy = -1 + lane + 32 * (job - 2); rj_dx = 63; }
    const bool has_job = job >= 0;
    const bool rj_on = has_job && (job < 2 || rj_dy <= TY);

    // TMA ring position of the next arrival (CTA lifetime): slot and mbarrier parity
    int gslot = 0;
    unsigned gphase = 0;
    for (;;) {
        if (tid == 0) s_item = atomicAdd(&P.counter[0], 1u);
        __syncthreads();
        const unsigned item = s_item;
        if (item >= (unsigned)P.items) break;
        const int tix = item % P.tiles_x;
        const int tiy = (item / P.tiles_x) % P.tiles_y;
        const int seg = item / (P.tiles_x * P.tiles_y);
        const int x0 = tix * 64, y0 = tiy * TY;

        // level-1 points: main (x0-1+2*lane+j, y0+4*warp+i), ring job (x0+rj_dx+j, y0+rj_dy)
        // masks: outside the x/y interior, and on the halo shell (Dirichlet value there)
        unsigned m_out = 0, m_shell = 0;
#pragma unroll
        for (int q = 0; q < 10; q++) {
            const bool main = q < 8;
            const int y = main ? y0 + 4 * warp + (q >> 1) : y0 + rj_dy;
            const int x = main ? x0 - 1 + 2 * lane + (q & 1) : x0 + rj_dx + (q & 1);
            const bool out = x < 0 || x >= P.nx || y < 0 || y >= P.ny;
            const bool shell = x >= -1 && x <= P.nx && y >= -1 && y <= P.ny;
            m_out |= (unsigned)out << q;
            m_shell |= (unsigned)shell << q;
        }
        if (!rj_on) {
            m_out &= 0xffu;
            m_shell &= 0xffu;
        }
        const int zs0 = P.zb[seg], zs1 = P.zb[seg + 1];
        const int p_first = zs0 - 2;
        const int M = (zs1 - zs0) + 4;                          // level-0 arrivals

        auto issue = [&](int t, int slot) {   // arrival t into ring slot `slot`
            uint64_t* b = &bar[slot];
            mbar_expect_tx(b, G::BOX_BYTES);
            tma_load_3d(s0 + slot * PLANE, &tmap, b, P.ax + x0 - G::XOFF, P.ry + y0 - 2, P.hz + p_first + t);
        };
        if (tid == 0)
            for (int t = 0; t < B3_NS0 && t < M; t++) issue(t, (gslot + t) % B3_NS0);
        int slot = gslot;
        unsigned phase = gphase;

        // level-2 stores: the lane's 2 x 4 outputs of plane zs0 (the pointer advances one
        // plane per stored plane); mode 2 = all four rows as aligned vectors, 1 = partial
        // (tiles on the domain edge), 0 = nothing to store
        const int xs = x0 + 2 * lane;
        const int nrow = min(4, P.ny - (y0 + 4 * warp));
        const int st_mode = (xs + 1 < P.nx && nrow == 4) ? 2 : ((xs < P.nx && nrow > 0) ? 1 : 0);
        T* orow = P.dst + P.origin + (int64_t)zs0 * P.sz + (int64_t)(y0 + 4 * warp) * P.sy + xs;

        B3Acc<T, PAIR, 4> A[3], B[3];     // level 1 / level 2 pending sums, main points (roles rotate)
        B3Acc<T, PAIR, 1> R[3];           // level 1, ring job
#pragma unroll
        for (int i = 0; i < 3; i++) {
            A[i].zero();
            B[i].zero();
            R[i].zero();
        }

        // Dirichlet values of level-1 points outside the x/y interior (rare: tiles on the
        // domain edge) or of a whole physical halo plane
        auto fix_l1 = [&](B3Acc<T, PAIR, 4>& Cm, B3Acc<T, PAIR, 1>& Cr, int zc) {
            const bool z_out = (P.phys_lo && zc < 0) || (P.phys_hi && zc >= P.nz);
            if (!z_out && !m_out) return;
            const bool z_shell = zc >= -1 && zc <= P.nz;
            // planes below/above the allocation (first completions of a ghost-side
            // segment) are garbage that never reaches a valid output: no load
            const bool z_alloc = zc >= -P.hz && zc < P.nz + P.hz_hi;
            const unsigned need = z_out ? 0x3ffu : m_out;
            const bool load_ok = z_out ? z_shell : z_alloc;
            const int64_t hb_main = P.origin + (int64_t)zc * P.sz + (int64_t)(y0 + 4 * warp) * P.sy + (x0 - 1 + 2 * lane);
            const int64_t hb_ring = P.origin + (int64_t)zc * P.sz + (int64_t)(y0 + rj_dy) * P.sy + (x0 + rj_dx);
#pragma unroll
            for (int q = 0; q < 10; q++)
                if ((need >> q) & 1) {
                    const T hv = (load_ok && ((m_shell >> q) & 1))
                                     ? P.src[(q < 8 ? hb_main + (q >> 1) * P.sy : hb_ring) + (q & 1)]
                                     : T(0);
                    if (q < 8) Cm.set(q >> 1, q & 1, hv);
                    else Cr.set(0, q & 1, hv);
                }
        };

        // one arriving plane; ROT selects which accumulator set completes (ROT), continues
        // (ROT+1) and starts (ROT+2) -- constant after unrolling, so no register moves
        // ---- level 1 for arrival t: completes level-1 plane a0-1 into buffer `l1`
        auto level1 = [&](int t, auto rot, T* l1) {
            constexpr int ROT = decltype(rot)::value;
            constexpr int IC = ROT, IK = (ROT + 1) % 3, IS = (ROT + 2) % 3;
            mbar_wait(&bar[slot], phase);
            const int a0 = p_first + t;   // level-0 plane that arrived
            const T* in0 = s0 + slot * PLANE;
            // main: rows y-1 .. y+4 of the box (box row 0 = y0-2), columns x-1 .. (box col 0 = x0-XOFF)
            b3_fold<T, PAIR, FMA, 4, PW>(in0 + (4 * warp + 1) * PW + (2 * lane - 2 + G::XOFF), nullptr, A[IC], A[IK],
                                         A[IS], P);
            if (has_job)
                b3_fold<T, PAIR, FMA, 1, PW>(in0 + (rj_dy + 1) * PW + (rj_dx - 1 + G::XOFF), nullptr, R[IC], R[IK],
                                             R[IS], P);
            fix_l1(A[IC], R[IC], a0 - 1);
            return std::integral_constant<int, IC>();
        };
        auto store_l1 = [&](auto ic, T* l1) {
            constexpr int IC = decltype(ic)::value;
            // level-1 plane: row 0 = y0-1, column 0 = x0-1 (shifted copy: column 0 = x0-2)
#pragma unroll
            for (int i = 0; i < 4; i++) b3_st2(l1 + (4 * warp + i + 1) * PW + 2 * lane, A[IC], i);
            if (rj_on) b3_st2(l1 + (rj_dy + 1) * PW + (rj_dx + 1), R[IC], 0);
            if constexpr (SHIFTED) {
                T* l1s = l1 + 2 * PLANE;
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    l1s[(4 * warp + i + 1) * PW + 2 * lane + 1] = A[IC].get(i, 0);
                    l1s[(4 * warp + i + 1) * PW + 2 * lane + 2] = A[IC].get(i, 1);
                }
                if (rj_on) {
                    l1s[(rj_dy + 1) * PW + (rj_dx + 2)] = R[IC].get(0, 0);
                    l1s[(rj_dy + 1) * PW + (rj_dx + 3)] = R[IC].get(0, 1);
                }
            }
        };
        // ---- level 2 for arrival t: reads level-1 plane a0-1 from `l1`, completes a0-2
        auto level2 = [&](int t, auto rot, const T* l1) {
            constexpr int ROT = decltype(rot)::value;
            constexpr int IC = ROT, IK = (ROT + 1) % 3, IS = (ROT + 2) % 3;
            // (the level-1 planes of arrivals 0 and 1 lie below every output's cone: no fold;
            // the sets they would have started complete at t = 2, 3, before the first store)
            if (t >= 2)
                b3_fold<T, PAIR, FMA, 4, PW, SHIFTED>(l1 + (4 * warp) * PW + 2 * lane, l1 + 2 * PLANE + (4 * warp) * PW +
                                                      2 * lane + 2, B[IC], B[IK], B[IS], P);
            // output plane zc = zs0 + (t - 4): inside [zs0, zs1) exactly for 4 <= t < M
            if (t >= 4) {
                if (st_mode == 2) {
                    T* r1 = orow + P.sy;
                    T* r2 = r1 + P.sy;
                    b3_st2(orow, B[IC], 0);
                    b3_st2(r1, B[IC], 1);
                    b3_st2(r2, B[IC], 2);
                    b3_st2(r2 + P.sy, B[IC], 3);
                } else if (st_mode == 1) {      // domain-edge tiles: short rows / odd last column
                    if (xs + 1 < P.nx) {
#pragma unroll
                        for (int i = 0; i < 4; i++)
                            if (i < nrow) b3_st2(orow + i * P.sy, B[IC], i);
                    } else {
#pragma unroll
                        for (int i = 0; i < 4; i++)
                            if (i < nrow) orow[i * P.sy] = B[IC].get(i, 0);
                    }
                }
                orow += P.sz;
            }
        };
        auto next_slot = [&]() {
            if (++slot == B3_NS0) {
                slot = 0;
                phase ^= 1u;
            }
        };
        // one arrival, both levels, one CTA barrier between them (level-1 buffers
        // alternate, so no trailing barrier)
        auto plane = [&](int t, auto rot) {
            T* l1 = s1 + (t & 1) * PLANE;
            auto ic = level1(t, rot, l1);
            store_l1(ic, l1);
            __syncthreads();   // level-1 plane complete; level-0 slot consumed
            if (tid == 0 && t + B3_NS0 < M) issue(t + B3_NS0, slot);
            next_slot();
            level2(t, rot, l1);
        };

        if constexpr (UNROLL3) {
            // accumulator roles rotate by renaming: no register moves (fp32: they would
            // compete with the FFMA2s for the FMA pipe)
            for (int t = 0; t < M; t += 3) {
                plane(t, std::integral_constant<int, 0>());
                if (t + 1 < M) plane(t + 1, std::integral_constant<int, 1>());
                if (t + 2 < M) plane(t + 2, std::integral_constant<int, 2>());
            }
        } else {
            // one copy of the plane code (instruction-cache footprint: the 3x unrolled fp64
            // loop measured 9% no-instruction stalls); roles rotate by moves, which run on
            // the FMA pipe, idle in fp64
            for (int t = 0; t < M; t++) {
                plane(t, std::integral_constant<int, 0>());
                A[0] = A[1]; A[1] = A[2];
                B[0] = B[1]; B[1] = B[2];
                R[0] = R[1]; R[1] = R[2];
            }
        }
        gslot = slot;   // (the barrier at the top of the item loop orders the next item's writes)
        gphase = phase;
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
