// Launch unit of the fused 3D kernel (K3/K4): TMA descriptors, tile/segment work items.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "plan.hpp"
#include "fused3d.cuh"
#include "compose3d.cuh"
#include "box3d.cuh"

namespace sbh {
namespace {

// ---------------------------------------------------------------- 3D

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// One TMA descriptor per device buffer: a 3D view (cols, rows, planes) of
// the whole allocation; boxes of F3_PW x (region height + 2) x 1, OOB elements zero-filled.
int make_tensor_maps_impl(sb_plan* P, int geo, int box_h, int box_w = sb::F3_PW) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    SB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) return fail(SB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    auto encode = reinterpret_cast<EncodeTiledFn>(fn);
    const int64_t rows = P->dims[1] + 2 * P->r;
    const int64_t planes = P->hlo + P->dims[0] + P->hhi;
    cuuint64_t dims[3] = {(cuuint64_t)P->px, (cuuint64_t)rows, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)(P->px * P->es), (cuuint64_t)(rows * P->px * P->es)};
    cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    const CUtensorMapDataType dt = P->dtype == SB_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    // box3d (geometries 4-6) reads 68-wide boxes that start 16 B before a 128 B line:
    // 64 B promotion fetched 10% fewer DRAM bytes than 128 B (4.89 vs 5.44 GB per C5
    // launch) and ran 1% faster; the other 3D kernels keep 128 B
    static const int promo_env = (int)env_double("SB200_TMA_L2PROMO", -1);
    const int promo = promo_env >= 0 ? promo_env : (geo >= 4 ? 64 : 128);
    const CUtensorMapL2promotion pr = promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                      : promo == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                      : promo == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                                     : CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    for (int b = 0; b < 2; b++) {
        CUresult r = encode(&P->tmap[geo][b], dt, 3, P->buf[b], dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(SB_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    }
    P->tmap_ok[geo] = true;
    return SB_OK;
}

template <typename T, bool BOX, int K, bool FMA, int NTY, int MINB, int RPT = 4>
int launch_fused3d_g(sb_plan* P, int src_idx) {
    using TL = sb::F3Tile<T, K, NTY, RPT>;
    using GEOM = sb::F3Geo<NTY, RPT>;
    static_assert(GEOM::PH == 34 || GEOM::PH == 18, "tensor-map slots exist for plane heights 34 and 18");
    constexpr int GEO = GEOM::PH == 34 ? 0 : 1;   // TMA box height (slot shared by equal heights)
    if (!P->tmap_ok[GEO]) {
        const int rc = make_tensor_maps_impl(P, GEO, GEOM::PH);
        if (rc != SB_OK) return rc;
    }
    auto kern = sb::fused3d_kernel<T, BOX, K, FMA, MINB, NTY, RPT>;
    const int smem = sb::f3_smem_bytes<T, K, NTY, RPT>();
    SB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int occ = 0;
    SB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, GEOM::THREADS, smem));
    occ = std::max(occ, 1);
    sb::Fused3DParams<T> prm;
    prm.src = reinterpret_cast<const T*>(P->buf[src_idx]);
    prm.dst = reinterpret_cast<T*>(P->buf[src_idx ^ 1]);
    prm.origin = P->g.origin;
    prm.sz = P->g.sz;
    prm.sy = P->g.sy;
    prm.nz = (int)P->dims[0];
    prm.ny = (int)P->dims[1];
    prm.nx = (int)P->dims[2];
    prm.ax = (int)(P->g.origin % P->g.sy);
    prm.ry = P->r;
    prm.hz = (int)P->hlo;
    prm.hz_hi = (int)P->hhi;
    prm.phys_lo = P->phys_lo;
    prm.phys_hi = P->phys_hi;
    prm.ghost_lo = P->phys_lo ? 0 : (int)P->hlo;
    prm.ghost_hi = P->phys_hi ? 0 : (int)P->hhi;
    prm.tiles_x = (int)((P->dims[2] - TL::X0 + TL::TXO - 1) / TL::TXO);
    prm.tiles_y = (int)((P->dims[1] + TL::TYO - 1) / TL::TYO);
    const int ctas_max = P->num_sms * occ;
    const int tiles = prm.tiles_x * prm.tiles_y;
    // small uniform z-segments balance best (measured: k=2 10-16 per CTA, k=1 ~32);
    // each item re-computes a 2K-plane warm-up, so not smaller
    const double seg_env = env_double("SB200_3D_ITEMS_PER_CTA", K == 1 ? 32.0 : 12.0);
    const int64_t z_lo = range_lo(P), nzr = range_hi(P) - z_lo;
    int nseg = (int)std::max<int64_t>(1, std::min<int64_t>(nzr, (int64_t)(seg_env * ctas_max / tiles + 0.5)));
    prm.lz = (int)((nzr + nseg - 1) / nseg);
    prm.nseg = (int)((nzr + prm.lz - 1) / prm.lz);
    prm.z0 = (int)z_lo;
    prm.z1 = (int)(z_lo + nzr);
    prm.items = tiles * prm.nseg;
    prm.total_ctas = std::min(ctas_max, prm.items);
    prm.counter = P->d_counter;
    for (int i = 0; i < 27; i++) prm.w[i] = T(0);
    for (int i = 0; i < P->nw; i++) {
        const int* o = &P->offsets[3 * i];
        prm.w[(o[0] + 1) * 9 + (o[1] + 1) * 3 + (o[2] + 1)] = (T)P->weights[i];
    }
    auto fbits = [](double v) -> unsigned long long {
        const float f = (float)v;
        unsigned int u;
        memcpy(&u, &f, 4);
        return u;
    };
    for (int b = 0; b < 3; b++)    // weight pairs of f3_push_pair: (point 0 low, point 1 high)
        for (int dy = 0; dy < 3; dy++)
            for (int c = 1; c <= 2; c++)
                prm.wp[(b * 3 + dy) * 2 + c - 1] = (fbits((double)prm.w[9 * b + dy * 3 + c - 1]) << 32) |
                                                  fbits((double)prm.w[9 * b + dy * 3 + c]);
    P->last_kernel = "fused3d_kernel";
    kern<<<(unsigned)prm.total_ctas, GEOM::THREADS, smem, P->stream>>>(P->tmap[GEO][src_idx], prm);
    SB_CUDA(cudaGetLastError());
    return SB_OK;
}

template <typename T, bool BOX, int K, bool FMA>
int launch_fused3d_k(sb_plan* P, int src_idx) {
    // 1: 128-thread CTAs (64 x 16 regions, 4 per SM: barrier phases of different
    // CTAs decorrelate; measured better at K <= 2), 0: 256-thread CTAs (64 x 32)
    static const int geo = (int)env_double("SB200_3D_GEO", -1);
    // 2: 128-thread CTAs, 3 per SM (more registers per thread).  Measured
    // (fp64, T=24): C4 star k=2 499 (geo 2) vs 479 (geo 1); C5 box k=2 374 vs
    // 392; k=3 both 328-390 vs 247-317.  fp32: geo 1 at k <= 2, geo 0 above.
    // fp32 box, paired FFMA2 path (92 registers): 3 CTAs/SM measured best at k <= 2
    // (C5 fp32 k=2: 626 vs 595 at 4 CTAs/SM; k=1: 568 vs 549)
    const bool geo2 = (sizeof(T) == 8 && K >= 2 && !(BOX && K == 2)) || (sizeof(T) == 4 && BOX && FMA && K <= 2);
    if (geo == 2 || (geo < 0 && geo2)) return launch_fused3d_g<T, BOX, K, FMA, 4, 3>(P, src_idx);
    if (geo == 1 || (geo < 0 && K <= 2)) return launch_fused3d_g<T, BOX, K, FMA, 4, 4>(P, src_idx);
    return launch_fused3d_g<T, BOX, K, FMA, 8, 2>(P, src_idx);
}

// ---- composed two-step star (compose3d.cuh): FMA mode, k = 2

// Two steps of the 7-point star = one step of its 25-point self-convolution
// (away from physical boundaries).  Composed in long double, rounded once.
template <typename T>
void composed_star_weights(const sb_plan* P, T (&w)[125], T (&w7)[7]) {
    long double c[125] = {};
    long double s[3][3][3] = {};
    for (int i = 0; i < P->nw; i++) {
        const int* o = &P->offsets[3 * i];
        s[o[0] + 1][o[1] + 1][o[2] + 1] = (long double)P->weights[i];
    }
    for (int a = 0; a < 27; a++)
        for (int b = 0; b < 27; b++) {
            const int az = a / 9 - 1, ay = a / 3 % 3 - 1, axx = a % 3 - 1;
            const int bz = b / 9 - 1, by = b / 3 % 3 - 1, bx = b % 3 - 1;
            const long double p = s[az + 1][ay + 1][axx + 1] * s[bz + 1][by + 1][bx + 1];
            if (p != 0) c[sb::c3_widx(az + bz, ay + by, axx + bx)] += p;
        }
    for (int i = 0; i < 125; i++) w[i] = (T)c[i];
    for (int i = 0; i < 7; i++) w7[i] = (T)P->weights[i];   // canonical star order
}

// Exact two-step weights of an x-face point p (x = 0: side 0, x = nx-1: side 1;
// y, z off the shell): its neighbour q = p + s*e_x is the held halo, so
// W_s(d) = sum over star pairs o + o' = d with o != s*e_x of w_o w_o', plus
// w_{s e_x} at d = s*e_x (the halo value itself).  Long double, rounded once.
template <typename T>
void xface_weights(const sb_plan* P, T (&wx)[2][125]) {
    long double s3[3][3][3] = {};
    for (int i = 0; i < P->nw; i++) {
        const int* o = &P->offsets[3 * i];
        s3[o[0] + 1][o[1] + 1][o[2] + 1] = (long double)P->weights[i];
    }
    for (int side = 0; side < 2; side++) {
        const int sx = side == 0 ? -1 : 1;
        long double c[125] = {};
        for (int a = 0; a < 27; a++) {
            const int az = a / 9 - 1, ay = a / 3 % 3 - 1, axx = a % 3 - 1;
            if (az == 0 && ay == 0 && axx == sx) continue;                 // the halo neighbour
            for (int b = 0; b < 27; b++) {
                const int bz = b / 9 - 1, by = b / 3 % 3 - 1, bx = b % 3 - 1;
                const long double p = s3[az + 1][ay + 1][axx + 1] * s3[bz + 1][by + 1][bx + 1];
                if (p != 0) c[sb::c3_widx(az + bz, ay + by, axx + bx)] += p;
            }
        }
        c[sb::c3_widx(0, 0, sx)] += s3[1][1][sx + 1];
        for (int i = 0; i < 125; i++) wx[side][i] = (T)c[i];
    }
}

bool compose3d_ok(const sb_plan* P, int k) {
    static const int enabled = (int)env_double("SB200_3D_COMPOSE", 1);
    return enabled && k == 2 && (P->dtype == SB_F64 || enabled == 2) && P->shape == SB_STAR && P->arith == SB_ARITH_FMA && P->nw == 7 &&
           P->dims[0] >= 4 && P->dims[1] >= 4 && P->dims[2] >= 4;
}

// z segments of a persistent 2.5D launch, the same for every xy tile (items are claimed
// tile-fastest, so the CTAs running together work on neighbouring tiles of one z range and
// share halo lines in L2).  Equal segments (`per` per CTA) until 1/guide of the remaining
// planes per CTA is shorter, then guided lengths down to `lmin` planes -- the last items
// are short, so the CTAs finish together (equal segments only, guide = 0: ~7.8 rounds of
// items on C5, 6-8% of the SM cycles idle at the end).  No segment is longer than the equal
// split's: long first items let the CTAs drift apart in z and lose the L2 sharing (C5
// uncapped: fp64 406 -> 393, fp32 704 -> 615 GStencil/s).  Returns the segment count.
int guided_z_segments(int64_t z_lo, int64_t nzr, int tiles, int ctas_max, double per, double guide, int64_t lmin,
                      int* zb, int max_seg) {
    int nb = 0;
    zb[0] = (int)z_lo;
    lmin = std::max<int64_t>(1, lmin);
    // (short ranges -- a block of a streamed sweep -- in segments of at least 32 planes: each
    // segment re-computes a 2K-plane warm-up.  One segment per tile for a 96-plane block --
    // best by CTA fill x warm-up overhead, 0.93 vs ~0.80 -- measured slower, streamed C5
    // sweep 171 vs 156 ms, fp32 146 vs 116: long items let the tiles drift apart in z)
    const int64_t neq = std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(max_seg, std::max<int64_t>(1, nzr / 32)),
                                                              (int64_t)(per * ctas_max / tiles + 0.5)));
    const int64_t lmax = std::max<int64_t>(guide > 0 ? lmin : 1, (nzr + neq - 1) / neq);
    int64_t rem = nzr;
    while (rem > 0) {
        int64_t len = lmax;
        if (guide > 0) {
            len = (int64_t)std::ceil((double)rem * tiles / (guide * ctas_max));
            len = std::min(std::max(len, lmin), lmax);
            if (rem - len < lmin / 2) len = rem;
        }
        if (nb == max_seg - 1) len = rem;
        len = std::min(len, rem);
        zb[nb + 1] = zb[nb] + (int)len;
        nb++;
        rem -= len;
    }
    for (int i = nb + 1; i <= max_seg; i++) zb[i] = zb[nb];
    return nb;
}

template <typename T, int NTY, int MINB>
int launch_compose3d(sb_plan* P, int src_idx) {
    constexpr int GEO = NTY == 8 ? 3 : 2;
    constexpr int VEC = 16 / (int)sizeof(T);
    constexpr int X0 = (2 % VEC == 0) ? 0 : 2 - VEC;   // TMA box start (x0 - 2) 16 B aligned
    if (!P->tmap_ok[GEO]) {
        const int rc = make_tensor_maps_impl(P, GEO, sb::C3Geo<NTY>::PH);
        if (rc != SB_OK) return rc;
    }
    auto kern = sb::compose3d_kernel<T, NTY, MINB>;
    const int smem = sb::c3_smem_bytes<T, NTY>();
    SB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int occ = 0;
    SB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, sb::C3Geo<NTY>::THREADS, smem));
    occ = std::max(occ, 1);
    sb::Compose3DParams<T> prm;
    prm.src = reinterpret_cast<const T*>(P->buf[src_idx]);
    prm.dst = reinterpret_cast<T*>(P->buf[src_idx ^ 1]);
    prm.origin = P->g.origin;
    prm.sz = P->g.sz;
    prm.sy = P->g.sy;
    prm.nz = (int)P->dims[0];
    prm.ny = (int)P->dims[1];
    prm.nx = (int)P->dims[2];
    prm.ax = (int)(P->g.origin % P->g.sy);
    prm.ry = P->r;
    prm.hz = (int)P->hlo;
    prm.hz_hi = (int)P->hhi;
    prm.phys_lo = P->phys_lo;
    prm.phys_hi = P->phys_hi;
    prm.x0_first = X0;
    prm.tiles_x = (int)((P->dims[2] - X0 + sb::C3_CW - 1) / sb::C3_CW);
    prm.tiles_y = (int)((P->dims[1] + sb::C3Geo<NTY>::CH - 1) / sb::C3Geo<NTY>::CH);
    const int ctas_max = P->num_sms * occ;
    const int tiles = prm.tiles_x * prm.tiles_y;
    const double per = env_double("SB200_C3_ITEMS_PER_CTA", 12.0);
    const int64_t z_lo = range_lo(P), z_hi = range_hi(P), nzr = z_hi - z_lo;
    prm.lz = 0;
    prm.nseg = guided_z_segments(z_lo, nzr, tiles, ctas_max, per, env_double("SB200_C3_GUIDE", 0)   /* HBM-bound: the guided tail measured 603 vs 608 */,
                                 (int64_t)env_double("SB200_C3_MIN_PLANES", 12), prm.zb, sb::C3_MAX_SEG);
    prm.z0 = (int)z_lo;
    prm.z1 = (int)z_hi;
    prm.items = tiles * prm.nseg;
    prm.total_ctas = std::min(ctas_max, prm.items);
    prm.counter = P->d_counter;
    T w7[7];
    composed_star_weights<T>(P, prm.w, w7);
    xface_weights<T>(P, prm.wx);

    // physical shell on the side stream (disjoint points; both read only src)
    sb::Shell3DParams<T> sp;
    sp.src = prm.src;
    sp.dst = prm.dst;
    sp.origin = prm.origin;
    sp.sz = prm.sz;
    sp.sy = prm.sy;
    sp.nx = prm.nx;
    sp.ny = prm.ny;
    sp.nz = prm.nz;
    sp.phys_lo = P->phys_lo;
    sp.phys_hi = P->phys_hi;
    sp.hz = (int)P->hlo;
    sp.hz_hi = (int)P->hhi;
    sp.z0 = (int)z_lo;
    sp.z1 = (int)z_hi;
    sp.zf_lo = P->phys_lo && z_lo == 0;
    sp.zf_hi = P->phys_hi && z_hi == P->dims[0];
    const int64_t zi = std::max<int64_t>(0, std::min<int64_t>(z_hi, P->phys_hi ? P->dims[0] - 1 : P->dims[0]) -
                                                std::max<int64_t>(z_lo, P->phys_lo ? 1 : 0));
    sp.nzf = (int64_t)(sp.zf_lo + sp.zf_hi) * prm.nx * prm.ny;
    sp.nyf = 2 * zi * prm.nx;
    sp.nxf = 0;   // x faces: corrected inside compose3d_kernel (E(q) push form)
    for (int i = 0; i < 7; i++) sp.w[i] = w7[i];
    const int64_t shell = sp.nzf + sp.nyf + sp.nxf;
    SB_CUDA(cudaEventRecord(P->fork_ev, P->stream));
    SB_CUDA(cudaStreamWaitEvent(P->side_stream, P->fork_ev, 0));
    const unsigned sblocks = (unsigned)std::min<int64_t>((shell + 255) / 256, (int64_t)P->num_sms * 8);
    sb::compose3d_shell_kernel<T><<<sblocks, 256, 0, P->side_stream>>>(sp);
    SB_CUDA(cudaGetLastError());
    SB_CUDA(cudaEventRecord(P->join_ev, P->side_stream));
    P->kernels_launched++;

    P->last_kernel = "compose3d_kernel";
    if (prm.items > 0) {
        kern<<<(unsigned)prm.total_ctas, sb::C3Geo<NTY>::THREADS, smem, P->stream>>>(P->tmap[GEO][src_idx], prm);
        SB_CUDA(cudaGetLastError());
    }
    SB_CUDA(cudaStreamWaitEvent(P->stream, P->join_ev, 0));   // join
    return SB_OK;
}

template <typename T>
int launch_compose3d_t(sb_plan* P, int src_idx) {
    static const int geo = (int)env_double("SB200_C3_GEO", 2);
    if (geo == 0) return launch_compose3d<T, 8, 2>(P, src_idx);
    if (geo == 2) return launch_compose3d<T, 4, 3>(P, src_idx);
    return launch_compose3d<T, 4, 4>(P, src_idx);
}

// ---- 27-point box, k = 2: output tiles of exactly 64 x TY, ring-only
// level-1 recompute (box3d.cuh)

template <typename T, bool FMA, int NW, int MINB, bool U3 = false>
int launch_box3d(sb_plan* P, int src_idx) {
    using G = sb::B3Geo<T, NW>;
    constexpr int GEO = NW == 4 ? 4 : (NW == 8 ? 5 : 6);   // tensor-map slot of this box geometry
    if (!P->tmap_ok[GEO]) {
        const int rc = make_tensor_maps_impl(P, GEO, G::PH, G::PW);
        if (rc != SB_OK) return rc;
    }
    auto kern = sb::box3d_kernel<T, FMA, NW, MINB, U3>;
    SB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM));
    int occ = 0;
    SB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, G::THREADS, G::SMEM));
    occ = std::max(occ, 1);
    sb::Box3DParams<T> prm;
    prm.src = reinterpret_cast<const T*>(P->buf[src_idx]);
    prm.dst = reinterpret_cast<T*>(P->buf[src_idx ^ 1]);
    prm.origin = P->g.origin;
    prm.sz = P->g.sz;
    prm.sy = P->g.sy;
    prm.nz = (int)P->dims[0];
    prm.ny = (int)P->dims[1];
    prm.nx = (int)P->dims[2];
    prm.ax = (int)(P->g.origin % P->g.sy);
    prm.ry = P->r;
    prm.hz = (int)P->hlo;
    prm.hz_hi = (int)P->hhi;
    prm.phys_lo = P->phys_lo;
    prm.phys_hi = P->phys_hi;
    prm.tiles_x = (int)((P->dims[2] + 63) / 64);
    prm.tiles_y = (int)((P->dims[1] + G::TY - 1) / G::TY);
    const int ctas_max = P->num_sms * occ;
    const int tiles = prm.tiles_x * prm.tiles_y;
    const double per = env_double("SB200_B3_ITEMS_PER_CTA", 6.0);   // (4-6: fp32 771, fp64 417; 8: 763 / 414; 10-12: 754 / 410)
    const int64_t z_lo = range_lo(P), nzr = range_hi(P) - z_lo;
    prm.nseg = guided_z_segments(z_lo, nzr, tiles, ctas_max, per, env_double("SB200_B3_GUIDE", 2.5),
                                 (int64_t)env_double("SB200_B3_MIN_PLANES", 12), prm.zb, sb::B3_MAX_SEG);
    prm.items = tiles * prm.nseg;
    prm.total_ctas = std::min(ctas_max, prm.items);
    prm.counter = P->d_counter;
    for (int i = 0; i < 27; i++) prm.w[i] = T(0);
    for (int i = 0; i < P->nw; i++) {
        const int* o = &P->offsets[3 * i];
        prm.w[(o[0] + 1) * 9 + (o[1] + 1) * 3 + (o[2] + 1)] = (T)P->weights[i];
    }
    for (int i = 0; i < 27; i++) {   // fp32 packed push: (w, w)
        const float f = (float)prm.w[i];
        unsigned int u;
        memcpy(&u, &f, 4);
        prm.wpp[i] = ((unsigned long long)u << 32) | u;
    }
    P->last_kernel = "box3d_kernel";
    if (prm.items > 0) {
        kern<<<(unsigned)prm.total_ctas, G::THREADS, G::SMEM, P->stream>>>(P->tmap[GEO][src_idx], prm);
        SB_CUDA(cudaGetLastError());
    }
    return SB_OK;
}

template <typename T, bool FMA>
int launch_box3d_t(sb_plan* P, int src_idx) {
    // measured (C5, T=100): NW=4 (64 x 16 tiles, 4 CTAs/SM) 402-413 GStencil/s fp64,
    // NW=8 (64 x 32, 2/SM) 403-410, 3 CTAs/SM without a register cap 399-409;
    // rejected: 96-thread CTAs (366-377), a skewed pipeline on mbarriers (390-402),
    // per-die work queues (402), a warp-specialised level split (335); fp32: a split-phase
    // level pipeline (mbarrier arrive after level 1 of plane t, wait before level 2 of plane
    // t - 1, four level-1 planes: 758 vs 770 -- the CTA barrier is not what bounds it); fp64 on
    // the 3x-unrolled loop (no role-rotation moves): 64 x 16 tiles at 3 CTAs/SM (158 registers)
    // 433 vs 440, 64 x 32 at 1 CTA/SM (194 registers) 392, at 2 CTAs/SM it spills (372)
    // (with the guided tail of the z schedule: fp32 3x-unrolled loop 713 -> 761, 64 x 32 tiles
    // 765; fp64 64 x 32 tiles 411 -> 414)
    static const int nw = (int)env_double("SB200_B3_NW", 8);
    static const int minb = (int)env_double("SB200_B3_MINB", 0);
    // fp32: with the scalar dx = 0 term (no input-pair moves) the single-copy loop wins
    // (C5 fp32: 713 vs 691 GStencil/s for the 3x-unrolled, role-renamed one; 5 or 6
    // CTAs/SM, SB200_B3_MINB, measured equal: 700-712)
    static const int u3 = (int)env_double("SB200_B3_U3", 1);
    if constexpr (sizeof(T) == 4 && FMA) {
        if (u3 && nw == 8 && minb == 3) return launch_box3d<T, FMA, 8, 3, true>(P, src_idx);
        if (u3 && nw == 8) return launch_box3d<T, FMA, 8, 2, true>(P, src_idx);
        if (u3 && minb == 6) return launch_box3d<T, FMA, 4, 6, true>(P, src_idx);
        if (u3 && minb == 5) return launch_box3d<T, FMA, 4, 5, true>(P, src_idx);
        if (u3) return launch_box3d<T, FMA, 4, 4, true>(P, src_idx);
    }
    if (nw == 8) return launch_box3d<T, FMA, 8, 2>(P, src_idx);
    if constexpr (sizeof(T) == 4 && FMA) {
        if (minb == 5) return launch_box3d<T, FMA, 4, 5>(P, src_idx);
        if (minb == 6) return launch_box3d<T, FMA, 4, 6>(P, src_idx);
    }
    if (minb == 3) return launch_box3d<T, FMA, 4, 3>(P, src_idx);
    return launch_box3d<T, FMA, 4, 4>(P, src_idx);
}

bool box3d_ok(const sb_plan* P, int k) {
    static const int enabled = (int)env_double("SB200_B3", 1);
    return enabled && k == 2 && P->shape == SB_BOX && P->nw == 27;
}

template <typename T, bool BOX, bool FMA>
int launch_fused3d_b(sb_plan* P, int src_idx, int k) {
    if constexpr (!BOX && FMA) {
        if (compose3d_ok(P, k)) return launch_compose3d_t<T>(P, src_idx);
    }
    if constexpr (BOX) {
        if (box3d_ok(P, k)) return launch_box3d_t<T, FMA>(P, src_idx);
    }
    switch (k) {
        case 1: return launch_fused3d_k<T, BOX, 1, FMA>(P, src_idx);
        case 2: return launch_fused3d_k<T, BOX, 2, FMA>(P, src_idx);
        case 3: return launch_fused3d_k<T, BOX, 3, FMA>(P, src_idx);
        case 4: return launch_fused3d_k<T, BOX, 4, FMA>(P, src_idx);
        default: return fail(SB_ERR_ARG, "unsupported 3D fused depth %d", k);
    }
}

template <typename T, bool FMA>
int launch_fused3d_t(sb_plan* P, int src_idx, int k) {
    if (P->shape == SB_BOX) return launch_fused3d_b<T, true, FMA>(P, src_idx, k);
    return launch_fused3d_b<T, false, FMA>(P, src_idx, k);
}


}  // namespace

int launch_fused3d(sb_plan* P, int src_idx, int k) {
    const bool fma = P->arith == SB_ARITH_FMA;
    if (P->dtype == SB_F64) return fma ? launch_fused3d_t<double, true>(P, src_idx, k) : launch_fused3d_t<double, false>(P, src_idx, k);
    return fma ? launch_fused3d_t<float, true>(P, src_idx, k) : launch_fused3d_t<float, false>(P, src_idx, k);
}

int make_tensor_maps(sb_plan* P, int geo, int box_h) { return make_tensor_maps_impl(P, geo, box_h); }

}  // namespace sbh
