// K5 -- generic single-step sweep: any d (1..3), any order r, star or box,
// any weights, fp64/fp32, EXACT or FMA.  One time step per launch.
//
// This is the correctness anchor and the fallback for stencil classes that
// have no fused kernel.  It restates scalar_step (stencilbench/kernels.py:
// 120-134): out-of-place, halo read-only, per point the canonical-order sum
// of kernels.py:103-108.  Weights and linearised offsets live in a small
// device table staged to shared memory once per CTA.
#pragma once
#include "common.cuh"

namespace sb {

constexpr int kGenericThreads = 256;
constexpr int kGenericMaxW = 1024;

// Interior sub-box computed by one launch: positions base[a] .. base[a] +
// ext[a] - 1 on each canonical axis (z, y, x).  The full sweep uses the whole
// interior (on a slab axis extended into the ghost planes); sb_step_box
// passes the reference's `ranges` (kernels.py:88-108).
struct Box3 {
    int64_t base[3];
    int64_t ext[3];
};

template <typename T, bool FMA>
__global__ void __launch_bounds__(kGenericThreads)
generic_step_kernel(const T* __restrict__ src, T* __restrict__ dst, Geom g, Box3 b, int nw,
                    const int64_t* __restrict__ lin, const T* __restrict__ w) {
    __shared__ int64_t s_lin[kGenericMaxW];
    __shared__ T s_w[kGenericMaxW];
    for (int i = threadIdx.x; i < nw; i += blockDim.x) {
        s_lin[i] = lin[i];
        s_w[i] = w[i];
    }
    __syncthreads();

    const int64_t rows = b.ext[0] * b.ext[1];
    const int64_t x = b.base[2] + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= b.base[2] + b.ext[2]) return;
    for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
        const int64_t z = b.base[0] + row / b.ext[1];
        const int64_t y = b.base[1] + row % b.ext[1];
        const int64_t p = g.origin + z * g.sz + y * g.sy + x;
        T acc = acc_first<T, FMA>(s_w[0], src[p + s_lin[0]]);
        for (int i = 1; i < nw; i++) acc = acc_term<T, FMA>(acc, s_w[i], src[p + s_lin[i]]);
        dst[p] = acc;
    }
}

}  // namespace sb
