// Launch unit of the fused 2D kernel (K2): strip/segment work items.
#include <cstdio>
#include <cstdlib>

#include "plan.hpp"
#include "fused2d.cuh"

namespace sbh {
namespace {

// ---------------------------------------------------------------- 2D

template <typename T, bool BOX, int K, bool FMA>
int launch_fused2d_k(sb_plan* P, const T* src, T* dst) {
    using TL = sb::F2Tile<K>;
    auto kern = sb::fused2d_kernel<T, BOX, K, FMA>;
    int occ = 0;
    SB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, sb::F2_WARPS * 32, 0));
    occ = std::max(occ, 1);
    sb::Fused2DParams<T> prm;
    prm.src = src;
    prm.dst = dst;
    prm.origin = P->g.origin;
    prm.sy = P->g.sy;
    prm.ny = (int)P->dims[0];
    prm.nx = (int)P->dims[1];
    prm.row_lo = -(int)P->hlo;
    prm.row_hi = (int)(P->dims[0] + P->hhi);
    prm.phys_lo = P->phys_lo;
    prm.phys_hi = P->phys_hi;
    prm.tiles_x = (int)((P->dims[1] + TL::TXO - 1) / TL::TXO);
    const int warps_max = P->num_sms * occ * sb::F2_WARPS;
    const double per = env_double("SB200_2D_ITEMS_PER_WARP", 3.0);
    int nseg = (int)std::max<int64_t>(1, std::min<int64_t>(P->dims[0], (int64_t)(per * warps_max / prm.tiles_x + 0.5)));
    // keep segments long against the 2K-row warm-up
    nseg = (int)std::min<int64_t>(nseg, std::max<int64_t>(1, P->dims[0] / (16 * K)));
    prm.ly = (int)((P->dims[0] + nseg - 1) / nseg);
    prm.nseg = (int)((P->dims[0] + prm.ly - 1) / prm.ly);
    prm.items = prm.tiles_x * prm.nseg;
    const int blocks = std::min(P->num_sms * occ, (prm.items + sb::F2_WARPS - 1) / sb::F2_WARPS);
    prm.total_warps = blocks * sb::F2_WARPS;
    prm.counter = P->d_counter;
    for (int i = 0; i < 9; i++) prm.w[i] = T(0);
    for (int i = 0; i < P->nw; i++) {
        const int* o = &P->offsets[2 * i];
        prm.w[(o[0] + 1) * 3 + (o[1] + 1)] = (T)P->weights[i];
    }
    kern<<<(unsigned)blocks, sb::F2_WARPS * 32, 0, P->stream>>>(prm);
    SB_CUDA(cudaGetLastError());
    return SB_OK;
}

template <typename T, bool BOX, bool FMA>
int launch_fused2d_b(sb_plan* P, const T* src, T* dst, int k) {
    switch (k) {
        case 1: return launch_fused2d_k<T, BOX, 1, FMA>(P, src, dst);
        case 2: return launch_fused2d_k<T, BOX, 2, FMA>(P, src, dst);
        case 4: return launch_fused2d_k<T, BOX, 4, FMA>(P, src, dst);
        case 8: return launch_fused2d_k<T, BOX, 8, FMA>(P, src, dst);
        default: return fail(SB_ERR_ARG, "unsupported 2D fused depth %d", k);
    }
}

template <typename T, bool FMA>
int launch_fused2d_t(sb_plan* P, const T* src, T* dst, int k) {
    if (P->shape == SB_BOX) return launch_fused2d_b<T, true, FMA>(P, src, dst, k);
    return launch_fused2d_b<T, false, FMA>(P, src, dst, k);
}


}  // namespace

int launch_fused2d(sb_plan* P, int src_idx, int k) {
    const bool fma = P->arith == SB_ARITH_FMA;
    if (P->dtype == SB_F64) {
        auto src = reinterpret_cast<const double*>(P->buf[src_idx]);
        auto dst = reinterpret_cast<double*>(P->buf[src_idx ^ 1]);
        return fma ? launch_fused2d_t<double, true>(P, src, dst, k) : launch_fused2d_t<double, false>(P, src, dst, k);
    }
    auto src = reinterpret_cast<const float*>(P->buf[src_idx]);
    auto dst = reinterpret_cast<float*>(P->buf[src_idx ^ 1]);
    return fma ? launch_fused2d_t<float, true>(P, src, dst, k) : launch_fused2d_t<float, false>(P, src, dst, k);
}

}  // namespace sbh
