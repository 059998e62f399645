// K2c -- composed separable 2D sweep (FMA mode, rank-1 box weights
// w[dy][dx] = a[dy] * b[dx], e.g. C3a's 1/9): K steps per HBM round trip as
// TWO one-dimensional composed passes.
//
// Away from the Dirichlet halo, K steps of a separable stencil are one step
// of the separable stencil a^{*K} (x) b^{*K} (K-fold convolution powers,
// composed on the host in long double, rounded once), so a launch costs
// 2 (2K+1) FMAs per point -- 4.06 per update at K = 32, against 6 for the
// separable level-by-level push and 9 for the plain one:
//   * sep_vpass_kernel: tmp = a^{*K} along y (columns; each thread streams its
//     column, B outputs per thread from 2K+B loads, coalesced across the warp);
//   * sep_hpass_kernel: out = b^{*K} along x on tmp (rows; warp tiles staged in
//     padded shared memory, 8 outputs per lane), for the points at distance
//     >= K from every physical side.
// The band of points closer than K to a physical side (their two-step... K-step
// cone reaches the held halo) is computed exactly, level by level, by
// sep_band_kernel: each CTA evolves a (band + cone) region K levels in shared
// memory with the halo cells held fixed and writes the band part -- on a side
// stream, concurrently with the passes (disjoint outputs, both read only src).
//
// Replaces the level-by-level 2D path (kernels.py:120-134 / tiling.py:372-417)
// for this stencil class in FMA mode; EXACT mode never uses it.
#pragma once
#include "common.cuh"
#include "compose1d.cuh"   // c1_pad, cp_async helpers

namespace sb {

#ifndef SB_SEP_VB
#define SB_SEP_VB 16
#endif
#ifndef SB_SEP_HB
#define SB_SEP_HB 8
#endif
constexpr int SEP_VB = SB_SEP_VB;  // output rows per thread in the vertical pass
constexpr int SEP_VT = 128;        // threads per vertical-pass CTA (columns)
constexpr int SEP_HB = SB_SEP_HB;  // outputs per lane in the horizontal pass
constexpr int SEP_HW = 4;          // warps per horizontal-pass CTA
constexpr int SEP_BW = 64;         // band chunk width (outputs along the band)
constexpr int SEP_BT = 512;        // band CTA threads

template <typename T>
struct SepParams {
    const T* src;        // interior (0, 0) of the current buffer
    T* dst;              // interior (0, 0) of the other buffer
    T* tmp;              // interior (0, 0) of the scratch buffer (same pitch)
    int64_t sy;          // row pitch (elements)
    int nx, ny;
    T c[65];             // composed 1D weights (2K+1), offset -K..K (vertical: a^{*K}; horizontal: b^{*K})
    int y0, y1;          // output rows [y0, y1) of the passes (K from a physical side)
    int row_hi;          // rows < row_hi are allocated (input guard of the staged pass)
};

// tmp[y][x] = sum_m a^{*K}[m] src[y+m][x], rows y in [K, ny-K), all columns.
// WG (whole grid, both y sides physical): the pass rows are [K, ny - K) as
// compile-time expressions; otherwise [P.y0, P.y1) (slab ghosts / ranges).
template <typename T, int K, bool WG>
__global__ void __launch_bounds__(SEP_VT) sep_vpass_kernel(const SepParams<T> P) {
    const int Y0 = WG ? K : P.y0, Y1 = WG ? P.ny - K : P.y1;
    const int x = blockIdx.x * SEP_VT + threadIdx.x;
    const int y0 = Y0 + blockIdx.y * SEP_VB;
    if (x >= P.nx || y0 >= Y1) return;
    const T* s = P.src + (int64_t)(y0 - K) * P.sy + x;
    T acc[SEP_VB];
#pragma unroll
    for (int m = 0; m < 2 * K + SEP_VB; m++) {
        const T v = s[(int64_t)m * P.sy];
#pragma unroll
        for (int o = 0; o < SEP_VB; o++) {
            const int t = m - o;                   // tap of v for output row y0 + o
            if (t >= 0 && t <= 2 * K) acc[o] = t == 0 ? v * P.c[0] : __fma_rn(P.c[t], v, acc[o]);
        }
    }
    T* d = P.tmp + (int64_t)y0 * P.sy + x;
#pragma unroll
    for (int o = 0; o < SEP_VB; o++)
        if (y0 + o < Y1) d[(int64_t)o * P.sy] = acc[o];
}

// Shared-memory staged form of the vertical pass: a CTA of SEP_VW warps owns 32
// columns x (SEP_VW * SEP_VB) output rows and loads its 2K + SEP_VW*SEP_VB input
// rows once (coalesced 256 B row segments), so L2 traffic per output is
// (2K + VW*VB) / (VW*VB) elements instead of (2K + VB) / VB.
constexpr int SEP_VW = 8;
template <typename T, int K>
constexpr int sep_vpass_smem_bytes() { return (2 * K + SEP_VW * SEP_VB) * 32 * (int)sizeof(T); }

template <typename T, int K, bool WG>
__global__ void __launch_bounds__(SEP_VW * 32) sep_vpass_smem_kernel(const SepParams<T> P) {
    extern __shared__ __align__(16) unsigned char smem_v[];
    T* col = reinterpret_cast<T*>(smem_v);            // [row][32]
    constexpr int ROWS = 2 * K + SEP_VW * SEP_VB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int x = blockIdx.x * 32 + lane;
    const int yb = (WG ? K : P.y0) + blockIdx.y * (SEP_VW * SEP_VB);  // first output row of the CTA
    const int y_end = WG ? P.ny - K : P.y1;
    const int row_hi = WG ? P.ny + 1 : P.row_hi;
    for (int r = warp; r < ROWS; r += SEP_VW) {
        const int y = yb - K + r;                       // input row; past the allocation: unused
        col[r * 32 + lane] = (x < P.nx && y < row_hi) ? P.src[(int64_t)y * P.sy + x] : T(0);
    }
    __syncthreads();
    const int y0 = yb + warp * SEP_VB;
    if (x >= P.nx || y0 >= y_end) return;
    const T* s = col + warp * SEP_VB * 32 + lane;
    T acc[SEP_VB];
#pragma unroll
    for (int m = 0; m < 2 * K + SEP_VB; m++) {
        const T v = s[m * 32];
#pragma unroll
        for (int o = 0; o < SEP_VB; o++) {
            const int t = m - o;
            if (t >= 0 && t <= 2 * K) acc[o] = t == 0 ? v * P.c[0] : __fma_rn(P.c[t], v, acc[o]);
        }
    }
    T* d = P.tmp + (int64_t)y0 * P.sy + x;
#pragma unroll
    for (int o = 0; o < SEP_VB; o++)
        if (y0 + o < y_end) d[(int64_t)o * P.sy] = acc[o];
}

// dst[y][x] = sum_m b^{*K}[m] tmp[y][x+m], rows [K, ny-K), columns [K, nx-K).
template <typename T, int K, bool WG>
__global__ void __launch_bounds__(SEP_HW * 32) sep_hpass_kernel(const SepParams<T> P) {
    constexpr int VEC = Vec16<T>::n;
    constexpr int TILE = 32 * SEP_HB;
    constexpr int SPAN = TILE + 2 * K;                          // inputs per warp tile
    constexpr int CHUNKS = SPAN / VEC;
    constexpr int PADDED = SPAN + (CHUNKS / 4 + 1) * VEC;
    constexpr int TAPS = 2 * K + 1;
    static_assert(SPAN % VEC == 0 && (SEP_HB + TAPS - 1) % VEC == 0, "tile span must be 16 B aligned");
    __shared__ __align__(16) T sm[SEP_HW][PADDED];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int y = (WG ? K : P.y0) + blockIdx.y;
    const int x0 = K + (blockIdx.x * SEP_HW + warp) * TILE;     // first output of the tile
    if (x0 >= P.nx - K || (!WG && y >= P.y1)) return;           // (warp-uniform)
    const T* row = P.tmp + (int64_t)y * P.sy;
    T* buf = sm[warp];
    // inputs x0-K .. x0+TILE+K; columns past nx-1 are never used by a stored output
    for (int c = lane; c < CHUNKS; c += 32) {
        const int xs = x0 - K + c * VEC;
        const bool ok = xs + VEC <= P.nx;
        using V = typename Vec16<T>::type;
        V v;
        if (ok) {
            v = *reinterpret_cast<const V*>(row + xs);
        } else {
#pragma unroll
            for (int e = 0; e < VEC; e++) reinterpret_cast<T*>(&v)[e] = xs + e < P.nx ? row[xs + e] : T(0);
        }
        *reinterpret_cast<V*>(buf + c1_pad<T>(c * VEC)) = v;
    }
    __syncwarp();
    T acc[SEP_HB];
    using V = typename Vec16<T>::type;
    // lane window base + compile-time offsets when SEP_HB/VEC is a multiple of 4
    // chunks (see compose1d_kernel)
    constexpr bool SPLIT = (SEP_HB / VEC) % 4 == 0;
    const T* bl = buf + (SPLIT ? c1_pad<T>(lane * SEP_HB) : 0);
#pragma unroll
    for (int jj = 0; jj < SEP_HB + TAPS - 1; jj += VEC) {
        const int off = SPLIT ? jj + (jj / (4 * VEC)) * VEC : c1_pad<T>(lane * SEP_HB + jj);
        const V xv = *reinterpret_cast<const V*>(bl + off);
#pragma unroll
        for (int e = 0; e < VEC; e++) {
            const int j = jj + e;
            const T x = reinterpret_cast<const T*>(&xv)[e];
#pragma unroll
            for (int o = 0; o < SEP_HB; o++) {
                const int t = j - o;
                if (t >= 0 && t < TAPS) acc[o] = t == 0 ? x * P.c[0] : __fma_rn(P.c[t], x, acc[o]);
            }
        }
    }
    // outputs through the (now free) staging buffer: each store instruction then
    // writes a contiguous 32 x 16 B row segment (whole sectors) instead of 32
    // lane-strided pieces
    __syncwarp();
#pragma unroll
    for (int v = 0; v < SEP_HB / VEC; v++) {
        V pack;
#pragma unroll
        for (int e = 0; e < VEC; e++) reinterpret_cast<T*>(&pack)[e] = acc[v * VEC + e];
        *reinterpret_cast<V*>(buf + c1_pad<T>(lane * SEP_HB + v * VEC)) = pack;
    }
    __syncwarp();
    T* d = P.dst + (int64_t)y * P.sy + x0;
    const int nout = P.nx - K - x0;                               // outputs of this tile inside the range
#pragma unroll
    for (int c = lane; c < TILE / VEC; c += 32) {
        const V pack = *reinterpret_cast<const V*>(buf + c1_pad<T>(c * VEC));
        if ((c + 1) * VEC <= nout) {
            *reinterpret_cast<V*>(d + c * VEC) = pack;
        } else {
#pragma unroll
            for (int e = 0; e < VEC; e++)
                if (c * VEC + e < nout) d[c * VEC + e] = reinterpret_cast<const T*>(&pack)[e];
        }
    }
}

// One band region: outputs [oy0, oy0+oh) x [ox0, ox0+ow) (interior coordinates),
// evolved from the region [oy0-K-1, oy0+oh+K+1) x [ox0-K-1, ox0+ow+K+1).
struct BandItem {
    int32_t oy0, ox0, oh, ow;
};

template <typename T>
struct SepBandParams {
    const T* src;        // interior (0, 0) of the current buffer
    T* dst;
    int64_t sy;
    int nx, ny;
    int row_lo, row_hi;  // allocated rows [row_lo, row_hi) (halo or ghost planes included)
    int fix_lo, fix_hi;  // physical halo rows held fixed (-1 / ny), or out of range on ghost sides
    const BandItem* items;
    int nitems;
    T w[9];              // box weights w[(dy+1)*3 + dx+1]
};

// Exact K-level evolution of each band region in shared memory (two buffers):
// cells on the physical halo ring keep their value at every level, cells
// outside the allocation are 0, the region's own outer ring (not physical) is
// never updated -- its staleness spreads one cell per level, K levels never
// reach the outputs (K+1 away).  Canonical (dy, dx) FMA order per point.
template <typename T, int K, bool WG>
__global__ void __launch_bounds__(SEP_BT) sep_band_kernel(const SepBandParams<T> P) {
    // WG: rows -1 and ny are the physical halo (allocated, held fixed)
    const int row_lo = WG ? -1 : P.row_lo, row_hi = WG ? P.ny + 1 : P.row_hi;
    const int fix_lo = WG ? -1 : P.fix_lo, fix_hi = WG ? P.ny : P.fix_hi;
    extern __shared__ __align__(16) unsigned char smem_band[];
    T* A = reinterpret_cast<T*>(smem_band);
    const BandItem it = P.items[blockIdx.x];
    const int ry0 = it.oy0 - K - 1, rx0 = it.ox0 - K - 1;
    const int RH = it.oh + 2 * K + 2, RW = it.ow + 2 * K + 2;
    T* B = A + RH * RW;
    // load: allocation = interior plus the 1-cell halo ring
    for (int i = threadIdx.x; i < RH * RW; i += SEP_BT) {
        const int y = ry0 + i / RW, x = rx0 + i % RW;
        const bool alloc = y >= row_lo && y < row_hi && x >= -1 && x <= P.nx;
        const T v = alloc ? P.src[(int64_t)y * P.sy + x] : T(0);
        A[i] = v;
        B[i] = v;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // updatable cells: inside the interior and not on the region's outer ring
    // rows: allocated and not a held physical halo row (ghost rows update like interior)
    const int ly_lo = max(1, max(row_lo, fix_lo + 1) - ry0);
    const int ly_hi = min(RH - 1, min(row_hi, fix_hi) - ry0);
    const int lx_lo = max(1, -rx0), lx_hi = min(RW - 1, P.nx - rx0);
    // work units: (32-column group, SEG-row segment); a lane walks its column down
    // the segment with a 3 x 3 register window (3 shared loads per cell, not 9)
    // level l+1 is only needed within K-l-1 cells of the output rectangle (the
    // cone shrinks by one cell per level): cells farther out are not updated
    constexpr int SEG = 8;
    for (int l = 0; l < K; l++) {
        const int sh = l + 1;
        const int y_lo = max(ly_lo, 1 + sh), y_hi = min(ly_hi, RH - 1 - sh);
        const int x_lo = max(lx_lo, 1 + sh), x_hi = min(lx_hi, RW - 1 - sh);
        const int ncg = (x_hi - x_lo + 31) / 32, nseg = (y_hi - y_lo + SEG - 1) / SEG;
        for (int u = warp; u < ncg * nseg; u += SEP_BT / 32) {
            const int lx = x_lo + (u % ncg) * 32 + lane;
            const int r0 = y_lo + (u / ncg) * SEG, r1 = min(y_hi, r0 + SEG);
            if (lx < x_hi) {
                const T* c = A + (r0 - 1) * RW + lx;
                T a0 = c[-1], a1 = c[0], a2 = c[1];
                c += RW;
                T b0 = c[-1], b1 = c[0], b2 = c[1];
                for (int ly = r0; ly < r1; ly++) {
                    c += RW;
                    const T d0 = c[-1], d1 = c[0], d2 = c[1];
                    T s = a0 * P.w[0];
                    s = __fma_rn(P.w[1], a1, s);
                    s = __fma_rn(P.w[2], a2, s);
                    s = __fma_rn(P.w[3], b0, s);
                    s = __fma_rn(P.w[4], b1, s);
                    s = __fma_rn(P.w[5], b2, s);
                    s = __fma_rn(P.w[6], d0, s);
                    s = __fma_rn(P.w[7], d1, s);
                    s = __fma_rn(P.w[8], d2, s);
                    B[ly * RW + lx] = s;
                    a0 = b0, a1 = b1, a2 = b2;
                    b0 = d0, b1 = d1, b2 = d2;
                }
            }
        }
        __syncthreads();
        T* t = A;
        A = B;
        B = t;
    }
    for (int i = threadIdx.x; i < it.oh * it.ow; i += SEP_BT) {
        const int oy = it.oy0 + i / it.ow, ox = it.ox0 + i % it.ow;
        if (oy < 0 || oy >= P.ny || ox < 0 || ox >= P.nx) continue;
        P.dst[(int64_t)oy * P.sy + ox] = A[(oy - ry0) * RW + (ox - rx0)];
    }
}

template <typename T, int K>
constexpr int sep_band_smem_bytes(int oh, int ow) {
    return 2 * (oh + 2 * K + 2) * (ow + 2 * K + 2) * (int)sizeof(T);
}

}  // namespace sb
