// Unit-axis layout conversions between NATURAL rows and the reference's
// BLOCK_TRANSPOSE / DLT storage rows (stencilbench/transpose.py:266-357,
// index map core.py:206-229), on the device.
//
// A row of reference storage is [hu halo | unit_np padded region | hu halo];
// only the padded region is permuted:
//   BLOCK_TRANSPOSE: natural o = b*vl^2 + p*vl + q (p, q < vl) sits at
//                    b*vl^2 + q*vl + p (every vl x vl block transposed);
//   DLT:             natural q*sub + c (sub = unit_np / vl) sits at c*vl + q.
// Halo cells (natural index < 0 or >= unit_np) are the identity.
//
// The permutation is a pure byte shuffle (HBM-bound, no arithmetic), so both
// sides of every transfer are coalesced: a CTA stages one contiguous storage
// tile of LT_S elements in shared memory and the natural side is read or
// written as contiguous runs (BLOCK_TRANSPOSE: the same LT_S-element range,
// DLT: vl runs of LT_S/vl elements, one per sub-stream).
#pragma once
#include <cstdint>

namespace sb {

constexpr int LT_S = 1024;        // storage elements per tile (multiple of vl^2 for vl in {4, 8})
constexpr int LT_THREADS = 256;

enum { LT_NATURAL = 0, LT_BLOCK_TRANSPOSE = 1, LT_DLT = 2 };

template <typename T>
struct LayoutXfer {
    const T* src;            // storage -> natural: storage rows; natural -> storage: natural rows
    T* dst;
    int64_t rows;
    int64_t nat_stride;      // natural-side row stride (elements)
    int64_t sto_stride;      // storage-side row stride
    int64_t nat0;            // natural side: element offset of natural index 0 in row 0
    int64_t sto0;            // storage side: element offset of the padded region (hu) in row 0
    int64_t i_lo, i_hi;      // natural indices moved (may reach into the halo: identity there)
    int64_t unit_np;
    int64_t sub;             // unit_np / vl (DLT sub-stream length)
    int64_t tiles;           // ceil(unit_np / LT_S)
    int layout, vl;
    int to_storage;          // 0: storage -> natural (gather), 1: natural -> storage (scatter)
};

// Natural index and in-tile storage offset of the e-th element of storage tile t
// (elements enumerated in natural order, so consecutive e are consecutive
// natural indices within a run).  Returns false past the region's end.
__device__ __forceinline__ bool lt_map(int layout, int vl, int64_t unit_np, int64_t sub, int64_t t, int e,
                                       int64_t& i, int& ls) {
    const int64_t s0 = t * LT_S;
    if (layout == LT_BLOCK_TRANSPOSE) {
        const int vv = vl * vl;
        const int o = e % vv;
        ls = (e - o) + (o % vl) * vl + o / vl;
        i = s0 + e;
        return i < unit_np;
    }
    // DLT: the tile holds sub-stream columns c in [s0/vl, s0/vl + LT_S/vl)
    const int tc = LT_S / vl;
    const int q = e / tc, cl = e % tc;
    const int64_t c = s0 / vl + cl;
    ls = cl * vl + q;
    i = (int64_t)q * sub + c;
    return c < sub;
}

template <typename T>
__global__ void __launch_bounds__(LT_THREADS) layout_xfer_kernel(const LayoutXfer<T> a) {
    __shared__ T tile[LT_S];
    const int tid = threadIdx.x;
    for (int64_t row = blockIdx.y; row < a.rows; row += gridDim.y) {
        const T* srow;
        T* drow;
        if (a.to_storage) {
            srow = a.src + a.nat0 + row * a.nat_stride;
            drow = a.dst + a.sto0 + row * a.sto_stride;
        } else {
            srow = a.src + a.sto0 + row * a.sto_stride;
            drow = a.dst + a.nat0 + row * a.nat_stride;
        }
        if (blockIdx.x == a.tiles) {
            // halo cells: identity map, natural index outside [0, unit_np)
            for (int64_t i = a.i_lo + tid; i < (a.i_hi < 0 ? a.i_hi : (int64_t)0); i += LT_THREADS) drow[i] = srow[i];
            for (int64_t i = (a.i_lo > a.unit_np ? a.i_lo : a.unit_np) + tid; i < a.i_hi; i += LT_THREADS) drow[i] = srow[i];
            continue;
        }
        const int64_t t = blockIdx.x;
        const int64_t s0 = t * LT_S;
        if (a.layout == LT_NATURAL) {   // identity (plain copy of the region range)
            for (int e = tid; e < LT_S; e += LT_THREADS) {
                const int64_t i = s0 + e;
                if (i < a.unit_np && i >= a.i_lo && i < a.i_hi) drow[i] = srow[i];
            }
            continue;
        }
        const int nvalid = (int)(a.unit_np - s0 < LT_S ? a.unit_np - s0 : LT_S);
        if (!a.to_storage) {
            // storage tile -> smem (coalesced), natural runs out (coalesced)
            for (int e = tid; e < nvalid; e += LT_THREADS) tile[e] = srow[s0 + e];
            __syncthreads();
            for (int e = tid; e < LT_S; e += LT_THREADS) {
                int64_t i;
                int ls;
                if (lt_map(a.layout, a.vl, a.unit_np, a.sub, t, e, i, ls) && i >= a.i_lo && i < a.i_hi)
                    drow[i] = tile[ls];
            }
        } else {
            // natural runs in (coalesced), storage tile out (coalesced); storage cells whose
            // natural index lies outside [i_lo, i_hi) keep their value
            for (int e = tid; e < LT_S; e += LT_THREADS) {
                int64_t i;
                int ls;
                if (lt_map(a.layout, a.vl, a.unit_np, a.sub, t, e, i, ls))
                    tile[ls] = (i >= a.i_lo && i < a.i_hi) ? srow[i] : drow[s0 + ls];
            }
            __syncthreads();
            for (int e = tid; e < nvalid; e += LT_THREADS) drow[s0 + e] = tile[e];
        }
        __syncthreads();
    }
}

}  // namespace sb
