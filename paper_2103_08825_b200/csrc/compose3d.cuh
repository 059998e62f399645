// K4c -- composed two-step 3D star sweep (FMA mode): two Jacobi steps of the
// 7-point star per HBM round trip as ONE pass of its 25-point square (the
// radius-2 "diamond" |dz|+|dy|+|dx| <= 2), instead of two dependent levels.
//
// Away from a physical boundary two steps of a constant-coefficient stencil
// equal one step of its self-convolution (weights composed on the host in
// extended precision, rounded once), so the fused pass needs no level planes,
// no inter-level barriers and no overlapped-tile recompute: it is a k=1-style
// 2.5D stream (TMA plane ring, push-form partial sums along z) with radius 2.
// 25 FMAs per point per pass = 12.5 per update (7 for the level-by-level
// path), far under the FP64 roofline at the HBM bound of k=2.
//
// Points whose two-step cone touches the Dirichlet halo (the interior's outer
// layer on every physical side) are not compositions -- the halo is held
// fixed at the intermediate step -- so the main kernel skips them and
// compose3d_shell_kernel recomputes them level by level (7 first-level values
// from the input, halo values where the neighbour is halo, then the second
// step), concurrently on the side stream.  Slab (ghost) sides along z are
// interior-like: the ghost depth is r*k = 2 planes, as for the fused kernel.
//
// Replaces the 3D scalar_step loop (kernels.py:120-134; the reference runs 3D
// untiled, harness.py:127-136).  EXACT mode (bit-identity) never uses it.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "fused3d.cuh"   // TMA / mbarrier helpers

namespace sb {

constexpr int C3_CW = 64;   // region width (x): 32 lanes x 2 points
constexpr int C3_PW = 68;   // shared plane width: 2 + 64 + 2 (rows 16 B multiples)
#ifndef SB_C3_NS
#define SB_C3_NS 4      // measured: 4 > 3 on C4 (697 vs 680 GStencil/s)
#endif
constexpr int C3_NS = SB_C3_NS;   // TMA ring depth

template <int NTY>
struct C3Geo {
    static constexpr int THREADS = 32 * NTY;
    static constexpr int CH = 4 * NTY;     // region height
    static constexpr int PH = CH + 4;      // plane height: 2-ring
};

template <typename T, int NTY>
struct C3Plane {
    static constexpr int ELEMS = ((C3_PW * C3Geo<NTY>::PH * (int)sizeof(T) + 127) / 128) * 128 / (int)sizeof(T);
    static constexpr unsigned BOX_BYTES = C3_PW * C3Geo<NTY>::PH * sizeof(T);
};
template <typename T, int NTY>
constexpr int c3_smem_bytes() { return C3_NS * C3Plane<T, NTY>::ELEMS * (int)sizeof(T); }

// Composed weight of offset (dz, dy, dx) in the 5 x 5 x 5 cube (zero off the diamond).
__host__ __device__ constexpr int c3_widx(int dz, int dy, int dx) { return (dz + 2) * 25 + (dy + 2) * 5 + (dx + 2); }

constexpr int C3_MAX_SEG = 47;

template <typename T>
struct Compose3DParams {
    const T* src;
    T* dst;
    int64_t origin, sz, sy;
    int nx, ny, nz;
    int ax, ry, hz, hz_hi;   // allocation coordinates of interior (0,0,0); planes above
    int phys_lo, phys_hi;
    int x0_first;            // x origin of the first tile (<= 0; TMA box starts 16 B aligned)
    int tiles_x, tiles_y, nseg, lz, items, total_ctas;
    int z0, z1;              // output planes [z0, z1) of this launch (range launches)
    int zb[C3_MAX_SEG + 1];  // z segment s = [zb[s], zb[s+1]): equal lengths, then a guided tail (launch3d.cu)
    unsigned int* counter;
    T w[125];                // composed weights w[c3_widx(dz, dy, dx)], |dz|+|dy|+|dx| <= 2
    T wx[2][125];            // exact two-step weights of the x = 0 / x = nx-1 face points
};

// Fold one arriving plane a into the four pending outputs A[0] = a-2 (its
// dz=+2 term completes it), A[1] = a-1, A[2] = a, A[3] = a+1, and start a+2.
// Rows arrive with increasing dy, dx ascends within a row: every output sums
// its terms in canonical (dz, dy, dx) order.
template <typename T>
__device__ __forceinline__ void c3_push(const T* plane, int tx, int ty, T (&A)[4][4][2], T (&done)[4][2],
                                        const T* w) {
    T nx[4][2];
#pragma unroll
    for (int r = 0; r < 8; r++) {
        T u[6];   // region columns 2tx-2 .. 2tx+3 of plane row 4ty+r (region row 4ty-2+r)
        const T* row = plane + (4 * ty + r) * C3_PW + 2 * tx;
#pragma unroll
        for (int h = 0; h < 3; h++) {
            if (sizeof(T) == 8) {
                const double2 v = *reinterpret_cast<const double2*>(row + 2 * h);
                u[2 * h] = (T)v.x;
                u[2 * h + 1] = (T)v.y;
            } else {
                const float2 v = *reinterpret_cast<const float2*>(row + 2 * h);
                u[2 * h] = (T)v.x;
                u[2 * h + 1] = (T)v.y;
            }
        }
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int dy = r - 2 - i;
            if (dy < -2 || dy > 2) continue;
            const int ady = dy < 0 ? -dy : dy;
#pragma unroll
            for (int dx = -2; dx <= 2; dx++) {
                const int adx = dx < 0 ? -dx : dx;
                if (ady + adx > 2) continue;
#pragma unroll
                for (int j = 0; j < 2; j++) {
                    const T x = u[j + 2 + dx];
                    if (ady + adx == 0) {
                        A[0][i][j] = acc_term<T, true>(A[0][i][j], w[c3_widx(2, 0, 0)], x);   // dz=+2: completes a-2
                        nx[i][j] = acc_first<T, true>(w[c3_widx(-2, 0, 0)], x);               // dz=-2: starts a+2
                    }
                    if (ady + adx <= 1) A[1][i][j] = acc_term<T, true>(A[1][i][j], w[c3_widx(1, dy, dx)], x);
                    A[2][i][j] = acc_term<T, true>(A[2][i][j], w[c3_widx(0, dy, dx)], x);
                    if (ady + adx <= 1) A[3][i][j] = acc_term<T, true>(A[3][i][j], w[c3_widx(-1, dy, dx)], x);
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 2; j++) {
            done[i][j] = A[0][i][j];
            A[0][i][j] = A[1][i][j];
            A[1][i][j] = A[2][i][j];
            A[2][i][j] = A[3][i][j];
            A[3][i][j] = nx[i][j];
        }
}

template <typename T, int NTY, int MINB>
__global__ void __launch_bounds__(C3Geo<NTY>::THREADS, MINB)
compose3d_kernel(const __grid_constant__ CUtensorMap tmap, const Compose3DParams<T> P) {
    constexpr int PLANE = C3Plane<T, NTY>::ELEMS;
    constexpr unsigned PLANE_BYTES = C3Plane<T, NTY>::BOX_BYTES;
    constexpr int CH = C3Geo<NTY>::CH;
    extern __shared__ __align__(1024) unsigned char smem_c3[];
    T* s0 = reinterpret_cast<T*>(smem_c3);
    __shared__ uint64_t bar[C3_NS];
    __shared__ unsigned s_item;

    const int tid = threadIdx.x;
    const int tx = tid & 31, ty = tid >> 5;
    if (tid == 0) {
        for (int i = 0; i < C3_NS; i++) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
    }
    __syncthreads();

    unsigned gstep = 0;
    for (;;) {
        if (tid == 0) s_item = atomicAdd(&P.counter[0], 1u);
        __syncthreads();
        const unsigned item = s_item;
        if (item >= (unsigned)P.items) break;
        const int tix = item % P.tiles_x;
        const int tiy = (item / P.tiles_x) % P.tiles_y;
        const int seg = item / (P.tiles_x * P.tiles_y);
        const int x0 = P.x0_first + tix * C3_CW, y0 = tiy * CH;
        // stored points: inside the interior and not on the x/y shell (shell kernel)
        // x-face points (x = 0 or nx-1, y off the y shell) are stored too, corrected
        // below; the y and z shells belong to compose3d_shell_kernel
        unsigned store_mask = 0;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int y = y0 + 4 * ty + (q >> 1), x = x0 + 2 * tx + (q & 1);
            store_mask |= (unsigned)(x >= 0 && x < P.nx && y >= 1 && y < P.ny - 1) << q;
        }
        // x faces in this tile (CTA-uniform): side 0 holds x = 0, side 1 x = nx-1
        const bool face0 = x0 <= 0, face1 = x0 + C3_CW > P.nx - 1;
        const int own0 = (0 - x0) >> 1, own1 = (P.nx - 1 - x0) >> 1;    // owner lanes
        const int oj0 = (0 - x0) & 1, oj1 = (P.nx - 1 - x0) & 1;         // owner point column
        // helper lanes 0-3 (side 0) and 4-7 (side 1) each evaluate one row's x-face point
        const int hs = tx >> 2, hrow = tx & 3;
        const bool helper = tx < 8 && (hs == 0 ? face0 : face1);
        const int hpc = (hs == 0 ? 0 : P.nx - 1) - x0 + 2;                // plane column of the point
        const T* const wf = P.wx[hs];
        T* const obase = P.dst + P.origin + (int64_t)(y0 + 4 * ty) * P.sy + (x0 + 2 * tx);
        const int zs0 = P.zb[seg], zs1 = P.zb[seg + 1];
        const int zlo = P.phys_lo ? 1 : 0, zhi = P.phys_hi ? P.nz - 1 : P.nz;   // z shell excluded
        const int p_first = zs0 - 2;
        const int M = (zs1 - zs0) + 4;

        auto issue = [&](int t) {
            const unsigned g = gstep + t;
            uint64_t* b = &bar[g % C3_NS];
            mbar_expect_tx(b, PLANE_BYTES);
            tma_load_3d(s0 + (g % C3_NS) * PLANE, &tmap, b, P.ax + x0 - 2, P.ry + y0 - 2, P.hz + p_first + t);
        };
        if (tid == 0)
            for (int t = 0; t < C3_NS && t < M; t++) issue(t);

        // helper lanes: the x-face point's own 25-tap push (weights wx[side]), pending
        // outputs a-2 .. a+1 as in c3_push
        T H0 = T(0), H1 = T(0), H2 = T(0), H3 = T(0);
        T A[4][4][2];
#pragma unroll
        for (int s = 0; s < 4; s++)
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 2; j++) A[s][i][j] = T(0);

        for (int t = 0; t < M; t++) {
            const unsigned g = gstep + t;
            mbar_wait(&bar[g % C3_NS], (g / C3_NS) & 1);
            T done[4][2];
            const T* pl = s0 + (g % C3_NS) * PLANE;
            c3_push<T>(pl, tx, ty, A, done, P.w);
            if (face0 || face1) {
                // x-face points are not compositions (one neighbour is the held halo): their
                // exact two-step value is a 25-tap sum too, with the folded weights wx[side]
                // (no subtraction, so NaN / Inf propagate as in the level-by-level sweep)
                T hd = T(0);
                if (helper) {
                    const T* pp = pl + (4 * ty + hrow + 2) * C3_PW + hpc;   // the point in plane a
                    T nxt = T(0);
#pragma unroll
                    for (int dy = -2; dy <= 2; dy++)
#pragma unroll
                        for (int dx = -2; dx <= 2; dx++) {
                            const int m = (dy < 0 ? -dy : dy) + (dx < 0 ? -dx : dx);
                            if (m > 2) continue;
                            const T v = pp[dy * C3_PW + dx];
                            if (m == 0) {
                                H0 = acc_term<T, true>(H0, wf[c3_widx(2, 0, 0)], v);
                                nxt = acc_first<T, true>(wf[c3_widx(-2, 0, 0)], v);
                            }
                            if (m <= 1) H1 = acc_term<T, true>(H1, wf[c3_widx(1, dy, dx)], v);
                            H2 = acc_term<T, true>(H2, wf[c3_widx(0, dy, dx)], v);
                            if (m <= 1) H3 = acc_term<T, true>(H3, wf[c3_widx(-1, dy, dx)], v);
                        }
                    hd = H0;
                    H0 = H1;
                    H1 = H2;
                    H2 = H3;
                    H3 = nxt;
                }
#pragma unroll
                for (int sd = 0; sd < 2; sd++) {
                    if (!(sd == 0 ? face0 : face1)) continue;
                    const int own = sd == 0 ? own0 : own1, oj = sd == 0 ? oj0 : oj1;
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        const T e = __shfl_sync(0xffffffffu, hd, sd * 4 + i);
#pragma unroll
                        for (int j = 0; j < 2; j++)
                            if (tx == own && j == oj) done[i][j] = e;
                    }
                }
            }
            const int zc = p_first + t - 2;       // completed output plane
            if (zc >= zs0 && zc < zs1 && zc >= zlo && zc < zhi && store_mask) {
                T* row = obase + (int64_t)zc * P.sz;
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    if (((store_mask >> (2 * i)) & 3) == 3 && sizeof(T) == 8) {
                        *reinterpret_cast<double2*>(row) = make_double2((double)done[i][0], (double)done[i][1]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 2; j++)
                            if ((store_mask >> (2 * i + j)) & 1) row[j] = done[i][j];
                    }
                    row += P.sy;
                }
            }
            __syncthreads();   // slot g % NS consumed by every thread
            if (tid == 0 && t + C3_NS < M) issue(t + C3_NS);
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

// ---- the physical shell: two exact levels of the 7-point star (FMA mode)

template <typename T>
struct Shell3DParams {
    const T* src;
    T* dst;
    int64_t origin, sz, sy;
    int nx, ny, nz;
    int phys_lo, phys_hi;
    int hz, hz_hi;           // planes allocated below / above the interior
    int z0, z1;              // output planes [z0, z1) of this launch
    int zf_lo, zf_hi;        // physical z faces inside [z0, z1) (0 / 1 each)
    int64_t nzf, nyf, nxf;   // points in the z-face, y-face and x-face segments
    T w[7];                  // star weights, canonical order
};

template <typename T>
__global__ void __launch_bounds__(256) compose3d_shell_kernel(const Shell3DParams<T> P) {
    const int64_t total = P.nzf + P.nyf + P.nxf;
    const int zlo = max(P.z0, P.phys_lo ? 1 : 0), zhi = min(P.z1, P.phys_hi ? P.nz - 1 : P.nz);
    const int64_t nzi = zhi - zlo > 0 ? zhi - zlo : 0;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        int z, y, x;
        int64_t e = idx;
        if (e < P.nzf) {                       // z faces (physical sides only)
            const int64_t per = (int64_t)P.nx * P.ny;
            const int f = (int)(e / per);
            e -= f * per;
            z = (f == 0 && P.zf_lo) ? 0 : P.nz - 1;
            y = (int)(e / P.nx);
            x = (int)(e % P.nx);
        } else if ((e -= P.nzf) < P.nyf) {     // y faces, z in [zlo, zhi)
            const int64_t per = nzi * P.nx;
            const int f = (int)(e / per);
            e -= f * per;
            y = f == 0 ? 0 : P.ny - 1;
            z = zlo + (int)(e / P.nx);
            x = (int)(e % P.nx);
        } else {                               // x faces, y in [1, ny-1), z in [zlo, zhi)
            e -= P.nyf;
            const int64_t per = nzi * (P.ny - 2);
            const int f = (int)(e / per);
            e -= f * per;
            x = f == 0 ? 0 : P.nx - 1;
            z = zlo + (int)(e / (P.ny - 2));
            y = 1 + (int)(e % (P.ny - 2));
        }
        const T* c = P.src + P.origin + (int64_t)z * P.sz + (int64_t)y * P.sy + x;
        // the 25 input values of the two-step cone, all loads issued up front;
        // positions beyond the halo (outside the allocation in y or z) are only
        // ever needed by halo neighbours, which take their own value instead
        T v[5][5][5];
#pragma unroll
        for (int dz = -2; dz <= 2; dz++)
#pragma unroll
            for (int dy = -2; dy <= 2; dy++)
#pragma unroll
                for (int dx = -2; dx <= 2; dx++) {
                    const int m = (dz < 0 ? -dz : dz) + (dy < 0 ? -dy : dy) + (dx < 0 ? -dx : dx);
                    if (m > 2) continue;
                    const bool ok = z + dz >= -P.hz && z + dz < P.nz + P.hz_hi && y + dy >= -1 && y + dy <= P.ny;
                    v[dz + 2][dy + 2][dx + 2] = ok ? c[(int64_t)dz * P.sz + (int64_t)dy * P.sy + dx] : T(0);
                }
        // first-level value at neighbour offset (oz, oy, ox): the halo value on a
        // physical side, else the 7-point step of the input (canonical order)
        auto level1 = [&](int oz, int oy, int ox) -> T {
            const int qz = z + oz, qy = y + oy, qx = x + ox;
            const bool halo = qx < 0 || qx >= P.nx || qy < 0 || qy >= P.ny || (P.phys_lo && qz < 0) ||
                              (P.phys_hi && qz >= P.nz);
            const int bz = oz + 2, by = oy + 2, bx = ox + 2;
            T s = acc_first<T, true>(P.w[0], v[bz - 1][by][bx]);
            s = acc_term<T, true>(s, P.w[1], v[bz][by - 1][bx]);
            s = acc_term<T, true>(s, P.w[2], v[bz][by][bx - 1]);
            s = acc_term<T, true>(s, P.w[3], v[bz][by][bx]);
            s = acc_term<T, true>(s, P.w[4], v[bz][by][bx + 1]);
            s = acc_term<T, true>(s, P.w[5], v[bz][by + 1][bx]);
            s = acc_term<T, true>(s, P.w[6], v[bz + 1][by][bx]);
            return halo ? v[bz][by][bx] : s;
        };
        T out = acc_first<T, true>(P.w[0], level1(-1, 0, 0));
        out = acc_term<T, true>(out, P.w[1], level1(0, -1, 0));
        out = acc_term<T, true>(out, P.w[2], level1(0, 0, -1));
        out = acc_term<T, true>(out, P.w[3], level1(0, 0, 0));
        out = acc_term<T, true>(out, P.w[4], level1(0, 0, 1));
        out = acc_term<T, true>(out, P.w[5], level1(0, 1, 0));
        out = acc_term<T, true>(out, P.w[6], level1(1, 0, 0));
        P.dst[P.origin + (int64_t)z * P.sz + (int64_t)y * P.sy + x] = out;
    }
}

}  // namespace sb
