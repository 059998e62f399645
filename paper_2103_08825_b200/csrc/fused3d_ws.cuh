// K3/K4 (k = 2) -- warp-specialised level pipeline for the 3D sweep.
//
// Same arithmetic and geometry as fused3d_kernel (push form along z, 64 x 32
// computed region, TMA-fed level-0 planes, canonical (dz, dy, dx) order per
// output), but the two fused levels run on two 8-warp groups of one CTA at
// the same time instead of one after the other behind CTA-wide barriers:
//
//   group 1 (warps 0-7):  TMA plane a  -> level-1 plane a-1 -> S1[a % 2]
//   group 2 (warps 8-15): S1[(a-1) % 2] -> level-2 plane a-2 -> global
//
// Hand-offs are mbarriers only (no __syncthreads inside an item): s0full /
// s0empty guard the TMA ring, s1full / s1empty the double-buffered level-1
// plane.  While one group is in its shared-memory read/emit phase the other
// keeps the FP64 pipe busy -- the lock-step phases of the barrier version were
// its main loss (profiles/r01_ncu_prof_3d_*).
#pragma once
#include "fused3d.cuh"

namespace sb {

constexpr int WS_GROUP = 256;                 // threads per level group
constexpr int WS_THREADS = 2 * WS_GROUP;

template <typename T>
constexpr int ws_smem_bytes() { return (F3_NS0 + 2) * F3Plane<T, 8>::ELEMS * (int)sizeof(T); }

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <typename T, bool BOX, bool FMA>
__global__ void __launch_bounds__(WS_THREADS, 1)
fused3d_ws_kernel(const __grid_constant__ CUtensorMap tmap, const Fused3DParams<T> P) {
    constexpr int K = 2;
    constexpr int NTY = 8;
    constexpr int PLANE = F3Plane<T, NTY>::ELEMS;
    constexpr unsigned PLANE_BYTES = F3Plane<T, NTY>::BOX_BYTES;
    using TL = F3Tile<T, K, NTY>;
    extern __shared__ __align__(1024) unsigned char smem3ws[];
    T* s0 = reinterpret_cast<T*>(smem3ws);    // NS0 TMA slots
    T* s1 = s0 + F3_NS0 * PLANE;              // two level-1 planes
    __shared__ uint64_t s0full[F3_NS0], s0empty[F3_NS0], s1full[2], s1empty[2];
    __shared__ unsigned s_item;

    const int tid = threadIdx.x;
    const int group = tid / WS_GROUP;          // 0: level 1, 1: level 2
    const int gt = tid % WS_GROUP;
    const int tx = gt & 31, ty = gt >> 5;
    if (tid == 0) {
        for (int i = 0; i < F3_NS0; i++) {
            mbar_init(&s0full[i], 1);
            mbar_init(&s0empty[i], WS_GROUP);
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(&s1full[i], WS_GROUP);
            mbar_init(&s1empty[i], WS_GROUP);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
    }
    __syncthreads();

    unsigned gstep = 0;   // CTA-lifetime step counter (both groups count alike)
    for (;;) {
        if (tid == 0) s_item = atomicAdd(&P.counter[0], 1u);
        __syncthreads();                      // item boundary: both groups done with the last one
        const unsigned item = s_item;
        if (item >= (unsigned)P.items) break;
        const int tix = item % P.tiles_x;
        const int tiy = (item / P.tiles_x) % P.tiles_y;
        const int seg = item / (P.tiles_x * P.tiles_y);
        const int x0 = TL::X0 + tix * TL::TXO, y0 = tiy * TL::TYO;
        const int xc = x0 - (K - 1), yc = y0 - (K - 1);
        const int zs0 = P.z0 + seg * P.lz, zs1 = min(P.z1, zs0 + P.lz);
        const int p_first = zs0 - K;
        const int M = (zs1 - zs0) + 2 * K;

        unsigned out_mask = 0, shell_mask = 0;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int y = yc + 4 * ty + (q >> 1), x = xc + 2 * tx + (q & 1);
            out_mask |= (unsigned)(x < 0 || x >= P.nx || y < 0 || y >= P.ny) << q;
            shell_mask |= (unsigned)(x >= -1 && x <= P.nx && y >= -1 && y <= P.ny) << q;
        }
        // in-plane offset of point q, computed only on the (rare) boundary path
        auto hoff = [&](int q) -> int64_t {
            return P.origin + (int64_t)(yc + 4 * ty + (q >> 1)) * P.sy + (xc + 2 * tx + (q & 1));
        };
        auto halo_fix = [&](T (&done)[4][2], int zc) {
            const bool z_out = (P.phys_lo && zc < 0) || (P.phys_hi && zc >= P.nz);
            if (z_out) {
                const bool z_shell = zc >= -1 && zc <= P.nz;
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    T hv = T(0);
                    if (z_shell && ((shell_mask >> q) & 1)) hv = P.src[hoff(q) + (int64_t)zc * P.sz];
                    done[q >> 1][q & 1] = hv;
                }
            } else if (out_mask) {
                const bool z_alloc = zc >= -P.hz && zc < P.nz + P.hz_hi;
#pragma unroll
                for (int q = 0; q < 8; q++)
                    if ((out_mask >> q) & 1)
                        done[q >> 1][q & 1] =
                            (z_alloc && ((shell_mask >> q) & 1)) ? P.src[hoff(q) + (int64_t)zc * P.sz] : T(0);
            }
        };
        auto issue = [&](int t) {
            const unsigned g = gstep + t;
            uint64_t* b = &s0full[g % F3_NS0];
            mbar_expect_tx(b, PLANE_BYTES);
            tma_load_3d(s0 + (g % F3_NS0) * PLANE, &tmap, b, P.ax + x0 - K, P.ry + y0 - K, P.hz + p_first + t);
        };

        T Pm[4][2], P0[4][2];
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int j = 0; j < 2; j++) Pm[i][j] = P0[i][j] = T(0);

        if (group == 0) {
            // ------------------------------------------------ level 1 (+ TMA producer)
            if (gt == 0)
                for (int t = 0; t < F3_NS0 && t < M; t++) issue(t);
            for (int t = 0; t < M; t++) {
                const unsigned g = gstep + t;
                mbar_wait(&s0full[g % F3_NS0], (g / F3_NS0) & 1);
                T done[4][2];
                f3_push_rows<T, BOX, FMA>(s0 + (g % F3_NS0) * PLANE, tx, ty, Pm, P0, done, P.w);
                mbar_arrive(&s0empty[g % F3_NS0]);
                // refill the slot consumed one step ago (all of its readers have long arrived)
                if (gt == 0 && t >= 1 && t - 1 + F3_NS0 < M) {
                    const unsigned gp = g - 1;
                    mbar_wait(&s0empty[gp % F3_NS0], (gp / F3_NS0) & 1);
                    issue(t - 1 + F3_NS0);
                }
                halo_fix(done, p_first + t - 1);
                mbar_wait(&s1empty[g % 2], ((g / 2) & 1) ^ 1);
                T* o = s1 + (g % 2) * PLANE;
#pragma unroll
                for (int i = 0; i < 4; i++)
#pragma unroll
                    for (int j = 0; j < 2; j++) o[(4 * ty + i + 1) * F3_PW + 2 * tx + j + 1] = done[i][j];
                mbar_arrive(&s1full[g % 2]);
            }
        } else {
            // ------------------------------------------------ level 2 -> global
            for (int t = 0; t < M; t++) {
                const unsigned g = gstep + t;
                mbar_wait(&s1full[g % 2], (g / 2) & 1);
                T done[4][2];
                f3_push_rows<T, BOX, FMA>(s1 + (g % 2) * PLANE, tx, ty, Pm, P0, done, P.w);
                mbar_arrive(&s1empty[g % 2]);
                const int zc = p_first + t - 2;
                halo_fix(done, zc);
                if (zc >= zs0 && zc < zs1) {
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        const int ri = 4 * ty + i - (K - 1);
                        const int y = y0 + ri;
                        if (ri < 0 || ri >= TL::TYO || y >= P.ny) continue;
#pragma unroll
                        for (int j = 0; j < 2; j++) {
                            const int cj = 2 * tx + j - (K - 1);
                            const int x = x0 + cj;
                            if (cj >= 0 && cj < TL::TXO && x >= 0 && x < P.nx)
                                P.dst[P.origin + (int64_t)zc * P.sz + (int64_t)y * P.sy + x] = done[i][j];
                        }
                    }
                }
            }
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
