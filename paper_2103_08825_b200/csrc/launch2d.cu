#include <atomic>
// Launch unit of the fused 2D kernel (K2): strip/segment work items.
#include <cstdio>
#include <cstdlib>

#include <climits>
#include <cmath>
#include <type_traits>

#include "plan.hpp"
#include "fused2d.cuh"
#include "plain2d.cuh"
#include "sep2d.cuh"

#ifndef SB_P2_MINB
#define SB_P2_MINB 3      // CTAs per SM of split2d_kernel at K = 3, 4 (4: 128 registers, measured slower)
#endif

namespace sbh {
namespace {

// ---------------------------------------------------------------- 2D

// Guided (strip, y-range) schedule: a first round of long ranges (about
// FRAC of the work spread over all warps), then ranges shrinking with the
// remaining work, never below MIN rows (each item re-computes a 2K-row
// warm-up).  Items are claimed in list order.
std::vector<sb::Item2D> guided_schedule_2d(int tiles_x, int64_t ny, int64_t warps, int K) {
    const double frac = env_double("SB200_2D_FIRST_FRAC", 0.4);
    const int64_t min_rows = std::max<int64_t>((int64_t)env_double("SB200_2D_MIN_ROWS", 24 * K), 8);
    std::vector<sb::Item2D> out;
    std::vector<int64_t> pos(tiles_x, 0);   // per-strip cursor
    const int64_t total = (int64_t)tiles_x * ny;
    // about one item per warp per round, never more items than warps (a first-round
    // item left over for a late claim is a long tail: traced on C3)
    const int64_t per_strip = std::max<int64_t>(1, warps / tiles_x);
    int64_t done = 0;
    bool first = true;
    while (done < total) {
        // one round = about one item per warp: per_strip consecutive items on every strip
        const int64_t rem = total - done;
        int64_t len = first ? (int64_t)(frac * (double)total / (double)warps) : rem / (2 * warps);
        len = std::max<int64_t>(len, min_rows);
        first = false;
        for (int64_t rep = 0; rep < per_strip; rep++) {
            for (int t = 0; t < tiles_x; t++) {
                if (pos[t] >= ny) continue;
                const int64_t l = std::min<int64_t>(len, ny - pos[t]);
                sb::Item2D it;
                it.tix = t;
                it.ys0 = (int32_t)pos[t];
                it.ys1 = (int32_t)(pos[t] + l);
                it.plain = 0;
                out.push_back(it);
                pos[t] += l;
                done += l;
            }
        }
    }
    return out;
}

// Rank-1 box weights w[dy][dx] = a[dy] * b[dx] (e.g. C3a's uniform 1/9): the
// separable push (6 FMAs per point and level instead of 9), FMA mode only.
bool separable_weights(const sb_plan* P, double a[3], double b[3]) {
    static const int enabled = (int)env_double("SB200_2D_SEPARABLE", 1);
    if (!enabled || P->shape != SB_BOX || P->arith != SB_ARITH_FMA || P->nw != 9) return false;
    double w[3][3] = {};
    double wmax = 0;
    for (int i = 0; i < 9; i++) {
        const int* o = &P->offsets[2 * i];
        w[o[0] + 1][o[1] + 1] = P->weights[i];
        wmax = std::max(wmax, std::fabs(P->weights[i]));
    }
    if (w[1][1] == 0) return false;
    for (int i = 0; i < 3; i++) {
        a[i] = w[i][1];
        b[i] = w[1][i] / w[1][1];
    }
    // exactly rank 1 in double (a near-separable table would run a slightly
    // different operator whose error grows with T): otherwise the 9-term path
    (void)wmax;
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++)
            if (a[i] * b[j] != w[i][j]) return false;
    return true;
}

// Split a guided schedule into the items whose whole K-level dependency cone is
// interior (plain2d_kernel) and the rest (fused2d_kernel): strips that touch an x
// halo column, and the K - 1 rows next to a physical y side of every other strip.
template <int K>
void split_plain_2d(const sb_plan* P, const std::vector<sb::Item2D>& items, std::vector<sb::Item2D>& plain,
                    std::vector<sb::Item2D>& edge) {
    using TL = sb::F2Tile<double, K>;
    const int64_t nx = P->dims[1], ny = P->dims[0];
    const int64_t row_lo = -P->hlo, row_hi = ny + P->hhi;
    // output rows whose level-1..K cone stays inside computed rows and whose level-0 rows are allocated
    const int64_t plo = std::max<int64_t>(P->phys_lo ? K - 1 : INT_MIN / 2, row_lo + K);
    // (plain2d_kernel prefetches P2_DIST rows past an item without testing: they must be allocated)
    const int64_t phi = std::min<int64_t>(P->phys_hi ? ny - (K - 1) : INT_MAX / 2, row_hi - 2 * K - sb::P2_DIST);   // (+ K - 1 more level-0 rows in the skewed form)
    static const int min_rows = (int)env_double("SB200_2D_PLAIN_MIN_ROWS", 8);
    for (const auto& it : items) {
        const int64_t xc = (int64_t)TL::X0 + (int64_t)it.tix * TL::TXO - TL::HL;
        const bool xplain = xc >= 0 && xc + sb::F2_CW <= nx;   // every computed column interior, edge columns in [-1, nx]
        const int64_t lo = std::max<int64_t>(it.ys0, plo), hi = std::min<int64_t>(it.ys1, phi);
        if (!xplain || hi - lo < min_rows) {
            edge.push_back(it);
            continue;
        }
        sb::Item2D e = it;
        if (lo > it.ys0) {
            e.ys0 = it.ys0;
            e.ys1 = (int32_t)lo;
            edge.push_back(e);
        }
        if (hi < it.ys1) {
            e.ys0 = (int32_t)hi;
            e.ys1 = it.ys1;
            edge.push_back(e);
        }
        e.ys0 = (int32_t)lo;
        e.ys1 = (int32_t)hi;
        plain.push_back(e);
    }
}

int upload_items(sb_plan* P, const std::vector<sb::Item2D>& items, void** d) {
    *d = nullptr;
    if (items.empty()) return SB_OK;
    SB_CUDA(cudaMalloc(d, sizeof(sb::Item2D) * items.size()));
    // stream-ordered: a pageable cudaMemcpy may return before its DMA lands, and the
    // kernel runs on the (non-blocking) plan stream
    SB_CUDA(cudaMemcpyAsync(*d, items.data(), sizeof(sb::Item2D) * items.size(), cudaMemcpyHostToDevice, P->stream));
    SB_CUDA(cudaStreamSynchronize(P->stream));
    return SB_OK;
}

template <typename T, bool BOX, int K, bool FMA, bool SEP>
int launch_fused2d_k(sb_plan* P, const T* src, T* dst) {
    using TL = sb::F2Tile<T, K>;
    // fp64, K = 4: the halo-free items run the lean path of split2d_kernel (plain2d.cuh);
    // SB200_2D_PLAIN=0: every item on fused2d_kernel.  (K = 2 is HBM-bound and measured
    // slower on the split kernel at 3, 4 and 5 CTAs per SM: C3b 583-597 vs 619 GStencil/s.)
    constexpr bool HAS_PLAIN = std::is_same<T, double>::value && K >= 3 && K <= 4;
    static const int plain_on = (int)env_double("SB200_2D_PLAIN", 1);
    static const int plain_skew = (int)env_double("SB200_2D_SKEW", 1);
    static const int edge_rows = (int)env_double("SB200_2D_EDGE_ROWS", 128);   // cap on the rows of a halo item (0: none): long ones are the tail of the launch (C3b k=4 1058 -> 1216)
    const bool split = HAS_PLAIN && plain_on;
    void (*kern)(const sb::Fused2DParams<T>) = sb::fused2d_kernel<T, BOX, K, FMA, SEP>;
    if constexpr (HAS_PLAIN) {
        if (split)
            kern = plain_skew ? sb::split2d_kernel<BOX, K, FMA, SEP, SB_P2_MINB, true>
                              : sb::split2d_kernel<BOX, K, FMA, SEP, SB_P2_MINB, false>;
    }
    const int smem = sb::fused2d_smem_bytes<T, K>();
    Sched1D* sc = nullptr;
    const int64_t y_lo = range_lo(P), y_hi = range_hi(P);
    for (auto& e : P->sched1d)   // 2D schedules keyed by 1000 + K and the output row range
        if (e.K == 1000 + K && e.comp_lo == y_lo && e.comp_hi == y_hi) sc = &e;
    if (!sc) {
        SB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int occ = 0;
        SB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, sb::F2_WARPS * 32, smem));
        Sched1D e;
        e.K = 1000 + K;
        e.blocks = P->num_sms * std::max(occ, 1);
        const int tiles_x = (int)((P->dims[1] - TL::X0 + TL::TXO - 1) / TL::TXO);
        auto items = guided_schedule_2d(tiles_x, y_hi - y_lo, (int64_t)e.blocks * sb::F2_WARPS, K);
        for (auto& it : items) {
            it.ys0 += (int32_t)y_lo;
            it.ys1 += (int32_t)y_lo;
        }
        if (split) {
            // halo items first (they start with the launch: the general path is slower per row),
            // then the plain ones, each group in guided order
            std::vector<sb::Item2D> plain, edge;
            split_plain_2d<K>(P, items, plain, edge);
            items.clear();
            for (const auto& it : edge) {
                const int32_t step = edge_rows > 0 ? edge_rows : it.ys1 - it.ys0;
                for (int32_t y = it.ys0; y < it.ys1; y += step) {
                    sb::Item2D c = it;
                    c.ys0 = y;
                    c.ys1 = std::min<int32_t>(y + step, it.ys1);
                    c.plain = 0;
                    items.push_back(c);
                }
            }
            for (auto it : plain) {
                it.plain = 1;
                items.push_back(it);
            }
        }
        e.comp_lo = y_lo;
        e.comp_hi = y_hi;
        e.nchunks = (int)items.size();
        const int rc = upload_items(P, items, &e.d_chunks);
        if (rc != SB_OK) return rc;
        P->sched1d.push_back(e);
        sc = &P->sched1d.back();
    }
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
    prm.items = sc->nchunks;
    prm.sched = reinterpret_cast<const sb::Item2D*>(sc->d_chunks);
    const int blocks = std::min(sc->blocks, (prm.items + sb::F2_WARPS - 1) / sb::F2_WARPS);
    prm.total_warps = blocks * sb::F2_WARPS;
    prm.counter = P->d_counter;
    prm.trace = nullptr;
    if (getenv("SB200_TRACE")) {   // debug: per-item trace of the last launch (sb_run writes it out)
        if (!P->d_trace) SB_CUDA(cudaMalloc(&P->d_trace, sizeof(unsigned long long) * 4 * (1 << 20)));
        if (prm.items <= (1 << 20)) prm.trace = P->d_trace;
        P->trace_n = prm.items;
    }
    for (int i = 0; i < 9; i++) prm.w[i] = T(0);
    for (int i = 0; i < P->nw; i++) {
        const int* o = &P->offsets[2 * i];
        prm.w[(o[0] + 1) * 3 + (o[1] + 1)] = (T)P->weights[i];
    }
    if (SEP) {
        double a[3], b[3];
        separable_weights(P, a, b);
        for (int i = 0; i < 3; i++) {
            prm.sa[i] = (T)a[i];
            prm.sb[i] = (T)b[i];
        }
    }
    P->last_kernel = split ? "split2d_kernel" : "fused2d_kernel";
    if (blocks > 0) {
        kern<<<(unsigned)blocks, sb::F2_WARPS * 32, smem, P->stream>>>(prm);
        SB_CUDA(cudaGetLastError());
    }
    return SB_OK;
}

template <typename T, bool BOX, bool FMA, bool SEP = false>
int launch_fused2d_b(sb_plan* P, const T* src, T* dst, int k) {
    switch (k) {
        case 1: return launch_fused2d_k<T, BOX, 1, FMA, SEP>(P, src, dst);
        case 2: return launch_fused2d_k<T, BOX, 2, FMA, SEP>(P, src, dst);
        case 4: return launch_fused2d_k<T, BOX, 4, FMA, SEP>(P, src, dst);
        case 8: return launch_fused2d_k<T, BOX, 8, FMA, SEP>(P, src, dst);
        default: return fail(SB_ERR_ARG, "unsupported 2D fused depth %d", k);
    }
}

template <typename T, bool FMA>
int launch_fused2d_t(sb_plan* P, const T* src, T* dst, int k) {
    if (P->shape == SB_BOX) {
        if constexpr (FMA) {
            double a[3], b[3];
            if (separable_weights(P, a, b)) return launch_fused2d_b<T, true, true, true>(P, src, dst, k);
        }
        return launch_fused2d_b<T, true, FMA>(P, src, dst, k);
    }
    return launch_fused2d_b<T, false, FMA>(P, src, dst, k);
}


// ---- separable composed path (sep2d.cuh)

std::vector<long double> conv_power(const long double w[3], int K) {
    std::vector<long double> c(1, 1.0L);
    for (int s = 0; s < K; s++) {
        std::vector<long double> n(c.size() + 2, 0.0L);
        for (size_t i = 0; i < c.size(); i++)
            for (int j = 0; j < 3; j++) n[i + j] += c[i] * w[j];
        c.swap(n);
    }
    return c;
}

// Band regions of the output rows [r0, r1): the K rows next to a physical y side
// (top / bottom bands, all columns) and the K columns next to the x sides for the
// rest (left / right bands).
std::vector<sb::BandItem> band_items(const sb_plan* P, int64_t r0, int64_t r1, int K) {
    const int64_t ny = P->dims[0], nx = P->dims[1];
    std::vector<sb::BandItem> out;
    const int W = sb::SEP_BW;
    auto rows = [&](int64_t a, int64_t b, bool full) {     // [a, b) intersected with [r0, r1)
        a = std::max(a, r0);
        b = std::min(b, r1);
        if (b <= a) return;
        if (full) {
            for (int64_t x = 0; x < nx; x += W)
                for (int64_t y = a; y < b; y += K)
                    out.push_back({(int32_t)y, (int32_t)x, (int32_t)std::min<int64_t>(K, b - y),
                                   (int32_t)std::min<int64_t>(W, nx - x)});
        } else {
            for (int64_t y = a; y < b; y += W) {
                const int h = (int)std::min<int64_t>(W, b - y);
                out.push_back({(int32_t)y, 0, h, K});
                out.push_back({(int32_t)y, (int32_t)(nx - K), h, K});
            }
        }
    };
    const int64_t ylo = P->phys_lo ? K : 0, yhi = P->phys_hi ? ny - K : ny;
    if (P->phys_lo && P->phys_hi && r0 == 0 && r1 == ny) {
        // whole grid: top and bottom chunks interleaved per column block
        for (int64_t x = 0; x < nx; x += W) {
            const int w = (int)std::min<int64_t>(W, nx - x);
            out.push_back({0, (int32_t)x, K, w});
            out.push_back({(int32_t)(ny - K), (int32_t)x, K, w});
        }
    } else {
        if (P->phys_lo) rows(0, K, true);
        if (P->phys_hi) rows(ny - K, ny, true);
    }
    rows(ylo, yhi, false);
    return out;
}

template <typename T, int K>
int launch_sep2d_k(sb_plan* P, int src_idx) {
    double a[3], b[3];
    separable_weights(P, a, b);
    const int64_t ny = P->dims[0], nx = P->dims[1];
    if (!P->tmp) {
        cudaError_t e = cudaMalloc(&P->tmp, P->buf_elems * P->es);
        if (e != cudaSuccess) return fail(e == cudaErrorMemoryAllocation ? SB_ERR_NOMEM : SB_ERR_CUDA,
                                          "separable scratch allocation failed: %s", cudaGetErrorString(e));
    }
    const int64_t origin = P->g.origin;
    sb::SepParams<T> vp, hp;
    vp.src = reinterpret_cast<const T*>(P->buf[src_idx]) + origin;
    vp.dst = reinterpret_cast<T*>(P->buf[src_idx ^ 1]) + origin;
    vp.tmp = reinterpret_cast<T*>(P->tmp) + origin;
    vp.sy = P->g.sy;
    vp.nx = (int)nx;
    vp.ny = (int)ny;
    // pass rows: K from a physical side, the whole slab on a ghost side (the ghost
    // planes hold the neighbour's rows, depth >= K); intersected with the range
    const int64_t ylo = std::max<int64_t>(P->phys_lo ? K : 0, range_lo(P));
    const int64_t yhi = std::min<int64_t>(P->phys_hi ? ny - K : ny, range_hi(P));
    vp.y0 = (int)ylo;
    vp.y1 = (int)std::max(ylo, yhi);
    vp.row_hi = (int)(ny + P->hhi);
    hp = vp;
    // whole grid (both sides physical, no range): the kernels' fixed-bound form
    const bool wg = P->phys_lo && P->phys_hi && P->zr_hi < 0;
    const long double la[3] = {a[0], a[1], a[2]}, lb[3] = {b[0], b[1], b[2]};
    const auto ca = conv_power(la, K), cb = conv_power(lb, K);
    for (int i = 0; i < 2 * K + 1; i++) {
        vp.c[i] = (T)ca[i];
        hp.c[i] = (T)cb[i];
    }
    // band regions (cached per plan and depth; key -4000 - K)
    Sched1D* sc = nullptr;
    const int64_t rlo = range_lo(P), rhi = range_hi(P);
    for (auto& e : P->sched1d)
        if (e.K == -4000 - K && e.comp_lo == rlo && e.comp_hi == rhi) sc = &e;
    if (!sc) {
        auto items = band_items(P, rlo, rhi, K);
        Sched1D e;
        e.K = -4000 - K;
        e.comp_lo = rlo;
        e.comp_hi = rhi;
        e.nchunks = (int)items.size();
        SB_CUDA(cudaMalloc(&e.d_chunks, sizeof(sb::BandItem) * items.size()));
        SB_CUDA(cudaMemcpyAsync(e.d_chunks, items.data(), sizeof(sb::BandItem) * items.size(),
                                cudaMemcpyHostToDevice, P->stream));
        SB_CUDA(cudaStreamSynchronize(P->stream));
        const int smem = sb::sep_band_smem_bytes<T, K>(K, sb::SEP_BW);
        SB_CUDA(cudaFuncSetAttribute(sb::sep_band_kernel<T, K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        SB_CUDA(cudaFuncSetAttribute(sb::sep_band_kernel<T, K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        P->sched1d.push_back(e);
        sc = &P->sched1d.back();
    }
    sb::SepBandParams<T> bp;
    bp.src = vp.src;
    bp.dst = vp.dst;
    bp.sy = P->g.sy;
    bp.nx = (int)nx;
    bp.ny = (int)ny;
    bp.row_lo = (int)-P->hlo;
    bp.row_hi = (int)(ny + P->hhi);
    bp.fix_lo = P->phys_lo ? -1 : INT_MIN / 2;
    bp.fix_hi = P->phys_hi ? (int)ny : INT_MAX / 2;
    bp.items = reinterpret_cast<const sb::BandItem*>(sc->d_chunks);
    bp.nitems = sc->nchunks;
    for (int i = 0; i < 9; i++) bp.w[i] = T(0);
    for (int i = 0; i < P->nw; i++) {
        const int* o = &P->offsets[2 * i];
        bp.w[(o[0] + 1) * 3 + (o[1] + 1)] = (T)P->weights[i];
    }
    // band: side stream, concurrent with the two passes (disjoint outputs), or
    // (SB200_SEP2D_BAND=1) after them on the main stream
    static const int band_mode = (int)env_double("SB200_SEP2D_BAND", 0);
    if (band_mode == 0 && sc->nchunks > 0) {
        SB_CUDA(cudaEventRecord(P->fork_ev, P->stream));
        SB_CUDA(cudaStreamWaitEvent(P->side_stream, P->fork_ev, 0));
        const unsigned nb = (unsigned)sc->nchunks;
        const int bsm = sb::sep_band_smem_bytes<T, K>(K, sb::SEP_BW);
        if (wg)
            sb::sep_band_kernel<T, K, true><<<nb, sb::SEP_BT, bsm, P->side_stream>>>(bp);
        else
            sb::sep_band_kernel<T, K, false><<<nb, sb::SEP_BT, bsm, P->side_stream>>>(bp);
        SB_CUDA(cudaGetLastError());
        SB_CUDA(cudaEventRecord(P->join_ev, P->side_stream));
    }
    // staged vertical pass at K = 32 (C3a 2492 -> 2778); at K = 16 the direct one
    // measured faster (1881 vs 1449)
    static const int vsmem = (int)env_double("SB200_SEP2D_VSMEM", 1);
    if (vp.y1 <= vp.y0) {
        // no pass rows in this range (band rows only)
    } else if (vsmem && K == 32) {
        constexpr int OUT = sb::SEP_VW * sb::SEP_VB;
        const int smem = sb::sep_vpass_smem_bytes<T, K>();
        static std::atomic<unsigned long long> attr{0};   // one bit per device
        if (!((attr.load() >> (P->device & 63)) & 1ull)) {
            SB_CUDA(cudaFuncSetAttribute(sb::sep_vpass_smem_kernel<T, K, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            SB_CUDA(cudaFuncSetAttribute(sb::sep_vpass_smem_kernel<T, K, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            attr.fetch_or(1ull << (P->device & 63));
        }
        dim3 vg((unsigned)((nx + 31) / 32), (unsigned)((vp.y1 - vp.y0 + OUT - 1) / OUT));
        if (wg)
            sb::sep_vpass_smem_kernel<T, K, true><<<vg, sb::SEP_VW * 32, smem, P->stream>>>(vp);
        else
            sb::sep_vpass_smem_kernel<T, K, false><<<vg, sb::SEP_VW * 32, smem, P->stream>>>(vp);
    } else {
        dim3 vg((unsigned)((nx + sb::SEP_VT - 1) / sb::SEP_VT), (unsigned)((vp.y1 - vp.y0 + sb::SEP_VB - 1) / sb::SEP_VB));
        if (wg)
            sb::sep_vpass_kernel<T, K, true><<<vg, sb::SEP_VT, 0, P->stream>>>(vp);
        else
            sb::sep_vpass_kernel<T, K, false><<<vg, sb::SEP_VT, 0, P->stream>>>(vp);
    }
    SB_CUDA(cudaGetLastError());
    constexpr int TILE = 32 * sb::SEP_HB;
    const int64_t tiles = (nx - 2 * K + TILE - 1) / TILE;
    if (vp.y1 > vp.y0) {
        dim3 hg((unsigned)((tiles + sb::SEP_HW - 1) / sb::SEP_HW), (unsigned)(vp.y1 - vp.y0));
        if (wg)
            sb::sep_hpass_kernel<T, K, true><<<hg, sb::SEP_HW * 32, 0, P->stream>>>(hp);
        else
            sb::sep_hpass_kernel<T, K, false><<<hg, sb::SEP_HW * 32, 0, P->stream>>>(hp);
        SB_CUDA(cudaGetLastError());
    }
    if (band_mode == 0) {
        if (sc->nchunks > 0) SB_CUDA(cudaStreamWaitEvent(P->stream, P->join_ev, 0));
    } else if (sc->nchunks > 0) {
        const unsigned nb = (unsigned)sc->nchunks;
        const int bsm = sb::sep_band_smem_bytes<T, K>(K, sb::SEP_BW);
        if (wg)
            sb::sep_band_kernel<T, K, true><<<nb, sb::SEP_BT, bsm, P->stream>>>(bp);
        else
            sb::sep_band_kernel<T, K, false><<<nb, sb::SEP_BT, bsm, P->stream>>>(bp);
        SB_CUDA(cudaGetLastError());
    }
    P->kernels_launched += 2;   // + the vertical pass counted by launch_one
    P->last_kernel = "sep2d (vertical + horizontal composed passes)";
    return SB_OK;
}

template <typename T>
int launch_sep2d(sb_plan* P, int src_idx, int k) {
    if (k == 16) return launch_sep2d_k<T, 16>(P, src_idx);
    return launch_sep2d_k<T, 32>(P, src_idx);
}

}  // namespace

bool sep2d_ok(const sb_plan* P, int k) {
    static const int enabled = (int)env_double("SB200_SEP2D", 1);
    double a[3], b[3];
    // slab sides need a ghost depth >= k (one launch reads k neighbour rows)
    return enabled && (k == 16 || k == 32) && P->d == 2 && (P->phys_lo || P->hlo >= k) &&
           (P->phys_hi || P->hhi >= k) && P->dims[0] > 2 * k && P->dims[1] > 2 * k && separable_weights(P, a, b);
}

int launch_fused2d(sb_plan* P, int src_idx, int k) {
    if (k >= 16) {
        if (!sep2d_ok(P, k)) return fail(SB_ERR_ARG, "2D depth %d needs the separable composed path", k);
        if (P->dtype == SB_F64) return launch_sep2d<double>(P, src_idx, k);
        return launch_sep2d<float>(P, src_idx, k);
    }
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
