#include <atomic>
// Launch unit of the fused 1D kernel (K1): guided chunk schedule, edge-kernel fork/join.
#include <cstdio>
#include <cstdlib>

#include "plan.hpp"
#include "compose1d.cuh"
#include "fused1d.cuh"

namespace sbh {
namespace {

// Guided chunk schedule for the persistent 1D kernel.  Chunks are claimed in
// list order: first one large chunk per warp (a fraction of the line), then
// chunks shrinking with the remaining work so the tail is balanced, and last
// the two minimum-size chunks touching the physical boundaries (they run the
// slower EDGE path; a large one there was measured to hold a whole launch
// back by ~50%).  S is a multiple of Q; the final chunk overruns n by
// < 32*Q points (covered by the right pad).
std::vector<sb::Chunk1D> guided_schedule_1d(int64_t n, int64_t warps, int Q, int64_t s_min,
                                           bool phys_lo, bool phys_hi, int* n_edge) {
    std::vector<sb::Chunk1D> main, edges;
    auto mk = [&](int64_t start, int64_t S) {
        sb::Chunk1D c;
        c.start = start;
        c.S = (int32_t)S;
        c.pad = 0;
        return c;
    };
    const int64_t edge = 32 * s_min;
    const double frac = env_double("SB200_1D_FIRST_FRAC", 0.7);
    const double div = env_double("SB200_1D_GUIDED_DIV", 2.0);
    const int64_t fixed = (int64_t)env_double("SB200_1D_FIXED_S", 0);
    if (n <= 3 * edge) {  // small line: minimum-size chunks, boundary ones on the edge path
        for (int64_t pos = 0; pos < n; pos += edge) {
            const bool e = (phys_lo && pos == 0) || (phys_hi && pos + edge >= n);
            (e ? edges : main).push_back(mk(pos, s_min));
        }
    } else {
        const int64_t lo = edge, hi = n - edge;
        const int64_t first =
            std::max<int64_t>(s_min, (int64_t)(frac * (double)(hi - lo) / (32.0 * warps)) / Q * Q);
        int64_t pos = lo, issued = 0;
        while (pos < hi) {
            const int64_t rem = hi - pos;
            int64_t S = issued < warps ? first : round_up((int64_t)(rem / (32 * warps * div)), Q);
            if (fixed > 0) S = round_up(fixed, Q);
            S = std::max<int64_t>(S, s_min);
            S = std::min<int64_t>(S, kMaxS1D);
            S = std::min<int64_t>(S, round_up((rem + 31) / 32, Q));
            main.push_back(mk(pos, S));
            pos += 32 * S;
            issued++;
        }
        (phys_lo ? edges : main).push_back(mk(0, s_min));
        if (pos < n) (phys_hi ? edges : main).push_back(mk(pos, round_up((n - pos + 31) / 32, Q)));
    }
    *n_edge = (int)edges.size();
    main.insert(main.end(), edges.begin(), edges.end());
    return main;
}

// ONE_PER_SMSP: one 4-warp CTA per SM (one warp per scheduler: no
// arbitration between warps, up to 255 registers, deep cp.async ring).
template <typename T, int R, int K, bool FMA, int MINB, int NST, bool ONE_PER_SMSP, bool DIAG = false>
int launch_fused1d_k(sb_plan* P, const T* src, T* dst) {
    using SH = sb::Fused1DShape<T, NST>;
    auto kern = sb::fused1d_kernel<T, R, K, FMA, MINB, NST, DIAG>;
    // one CTA per SM is enforced through the shared-memory request
    const int smem = ONE_PER_SMSP ? std::max(SH::SMEM_BYTES, 120 * 1024) : SH::SMEM_BYTES;
    Sched1D* sc = nullptr;
    for (auto& e : P->sched1d)
        if (e.K == K) sc = &e;
    if (!sc) {
        SB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        SB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     (int)cudaSharedmemCarveoutMaxShared));
        int blocks_per_sm = 0;
        SB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, SH::WARPS * 32, smem));
        blocks_per_sm = std::max(blocks_per_sm, 1);
        Sched1D e;
        e.K = K;
        e.blocks = P->num_sms * blocks_per_sm;
        const int64_t warps = (int64_t)e.blocks * SH::WARPS;
        int n_edge = 0;
        auto chunks = guided_schedule_1d(P->g.n[2], warps, SH::Q,
                                         (int64_t)env_double("SB200_1D_SMIN", 12 * SH::Q),
                                         P->phys_lo, P->phys_hi, &n_edge);
        e.nchunks = (int)chunks.size() - n_edge;
        e.nedge = n_edge;
        auto ekern = sb::fused1d_edge_kernel<T, R, K, FMA, NST, DIAG>;
        SB_CUDA(cudaFuncSetAttribute(ekern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (SH::IN_ELEMS + SH::OUT_ELEMS) * (int)sizeof(T)));
        SB_CUDA(cudaMalloc(&e.d_chunks, sizeof(sb::Chunk1D) * chunks.size()));
        SB_CUDA(cudaMemcpyAsync(e.d_chunks, chunks.data(), sizeof(sb::Chunk1D) * chunks.size(),
                           cudaMemcpyHostToDevice, P->stream));
        SB_CUDA(cudaStreamSynchronize(P->stream));
        P->sched1d.push_back(e);
        sc = &P->sched1d.back();
    }
    sb::Fused1DParams<T, R> prm;
    prm.src = src + P->g.origin;
    prm.dst = dst + P->g.origin;
    prm.n = P->g.n[2];
    prm.chunks = reinterpret_cast<const sb::Chunk1D*>(sc->d_chunks);
    prm.nchunks = sc->nchunks;
    prm.total_warps = sc->blocks * SH::WARPS;
    prm.counter = P->d_counter;
    prm.trace = nullptr;
    if (getenv("SB200_TRACE")) {
        if (!P->d_trace) SB_CUDA(cudaMalloc(&P->d_trace, sizeof(unsigned long long) * 4 * (1 << 20)));
        if (sc->nchunks <= (1 << 20)) prm.trace = P->d_trace;
        P->trace_n = sc->nchunks;
    }
    prm.phys_lo = P->phys_lo;
    prm.phys_hi = P->phys_hi;
    for (int i = 0; i < 2 * R + 1; i++) prm.w[i] = (T)P->weights[i];
    if (sc->nedge > 0) {  // fork: boundary chunks on the side stream, concurrently
        SB_CUDA(cudaEventRecord(P->fork_ev, P->stream));
        SB_CUDA(cudaStreamWaitEvent(P->side_stream, P->fork_ev, 0));
        sb::fused1d_edge_kernel<T, R, K, FMA, NST, DIAG><<<(unsigned)sc->nedge, 32,
            (SH::IN_ELEMS + SH::OUT_ELEMS) * (int)sizeof(T), P->side_stream>>>(prm);
        SB_CUDA(cudaGetLastError());
        SB_CUDA(cudaEventRecord(P->join_ev, P->side_stream));
        P->kernels_launched++;
    }
    P->last_kernel = "fused1d_kernel";
    kern<<<(unsigned)sc->blocks, SH::WARPS * 32, smem, P->stream>>>(prm);
    SB_CUDA(cudaGetLastError());
    if (sc->nedge > 0) SB_CUDA(cudaStreamWaitEvent(P->stream, P->join_ev, 0));  // join
    return SB_OK;
}

// Composed-stencil path (FMA mode): the composed (2RK+1)-tap kernel for every
// output at least RK from a physical boundary (main stream) and, on the side
// stream, one exact level-by-level window CTA per physical side for the RK
// outputs next to it (their dependency cone reaches the Dirichlet halo).
std::vector<double> composed_weights(const std::vector<double>& w, int K) {
    std::vector<long double> c(1, 1.0L);
    for (int step = 0; step < K; step++) {
        std::vector<long double> n(c.size() + w.size() - 1, 0.0L);
        for (size_t i = 0; i < c.size(); i++)
            for (size_t j = 0; j < w.size(); j++) n[i + j] += c[i] * (long double)w[j];
        c.swap(n);
    }
    return std::vector<double>(c.begin(), c.end());
}

template <typename T, int R, int K>
int launch_compose1d_k(sb_plan* P, const T* src, T* dst) {
    constexpr int HALF = R * K;
    static_assert(2 * HALF + 1 <= sb::C1_MAXTAPS, "composed depth too large");
    const int64_t n = P->g.n[2];
    Sched1D* sc = nullptr;
    for (auto& e : P->sched1d)
        if (e.K == -K) sc = &e;   // composed schedules keyed by -K
    if (!sc) {
        Sched1D e;
        e.K = -K;
        e.comp_lo = P->phys_lo ? HALF : 0;      // 16 B aligned: HALF % VEC == 0
        e.comp_hi = P->phys_hi ? n - HALF : n;
        e.nchunks = 0;
        e.nedge = (int)P->phys_lo + (int)P->phys_hi;
        auto ck = sb::compose1d_kernel<T, HALF>;
        const int smem = sb::compose1d_smem_bytes<T, HALF>();
        SB_CUDA(cudaFuncSetAttribute(ck, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int occ = 0;
        SB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ck, sb::C1_WARPS * 32, smem));
        e.blocks = P->num_sms * std::max(occ, 1);
        auto cw = composed_weights(P->weights, K);
        e.cw.assign(cw.begin(), cw.end());
        P->sched1d.push_back(e);
        sc = &P->sched1d.back();
    }
    static const int fuse_edges = (int)env_double("SB200_1D_FUSED_EDGES", 1);
    if (sc->nedge > 0 && !fuse_edges) {   // boundary windows: exact level-by-level, side stream
        sb::EdgeWindowParams<T, R> ep;
        ep.src = src + P->g.origin;
        ep.dst = dst + P->g.origin;
        ep.n = n;
        int b = 0;
        if (P->phys_lo) ep.side[b++] = 0;
        if (P->phys_hi) ep.side[b++] = 1;
        for (int i = 0; i < 2 * R + 1; i++) ep.w[i] = (T)P->weights[i];
        SB_CUDA(cudaEventRecord(P->fork_ev, P->stream));
        SB_CUDA(cudaStreamWaitEvent(P->side_stream, P->fork_ev, 0));
        sb::edge_window_kernel<T, R, K, true><<<(unsigned)b, 32, 0, P->side_stream>>>(ep);
        SB_CUDA(cudaGetLastError());
        SB_CUDA(cudaEventRecord(P->join_ev, P->side_stream));
        P->kernels_launched++;
    }
    sb::Compose1DParams<T> cp;
    cp.src = src + P->g.origin;
    cp.dst = dst + P->g.origin;
    cp.lo = sc->comp_lo;
    cp.hi = sc->comp_hi;
    const int64_t tile = 32 * sb::C1_B;
    cp.ntiles = (cp.hi - cp.lo + tile - 1) / tile;
    cp.total_warps = sc->blocks * sb::C1_WARPS;
    cp.counter = P->d_counter;
    cp.taps = 2 * HALF + 1;
    for (int i = 0; i < 2 * HALF + 1; i++) cp.c[i] = (T)sc->cw[i];
    P->last_kernel = "compose1d_kernel";
    if (sc->nedge > 0 && fuse_edges) {
        // boundary windows in the same launch: `nedge` leading CTAs; the composed grid
        // shrinks by as many so the whole launch stays resident
        sb::EdgeWindowParams<T, R> ep;
        ep.src = src + P->g.origin;
        ep.dst = dst + P->g.origin;
        ep.n = n;
        int b = 0;
        if (P->phys_lo) ep.side[b++] = 0;
        if (P->phys_hi) ep.side[b++] = 1;
        for (int i = 0; i < 2 * R + 1; i++) ep.w[i] = (T)P->weights[i];
        const int main_blocks = std::max(1, sc->blocks - sc->nedge);
        cp.total_warps = main_blocks * sb::C1_WARPS;
        auto ck = sb::compose1d_kernel<T, HALF, R>;
        static std::atomic<unsigned long long> attr_set{0};   // per instantiation, one bit per device
        if (!((attr_set.load() >> (P->device & 63)) & 1ull)) {
            SB_CUDA(cudaFuncSetAttribute(ck, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         sb::compose1d_smem_bytes<T, HALF>()));
            attr_set.fetch_or(1ull << (P->device & 63));
        }
        // programmatic dependent launch: CTA scheduling and the launch latency of this
        // step overlap the previous step's tail (the kernel waits on griddepcontrol
        // before reading); short sweeps (C1: one ~10 us launch per step) gain most
        static const int pdl = (int)env_double("SB200_PDL", 1);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(main_blocks + sc->nedge));
        cfg.blockDim = dim3(sb::C1_WARPS * 32);
        cfg.dynamicSmemBytes = sb::compose1d_smem_bytes<T, HALF>();
        cfg.stream = P->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;
        const int nedge = sc->nedge;
        SB_CUDA(cudaLaunchKernelEx(&cfg, ck, cp, ep, nedge));
        return SB_OK;
    }
    if (cp.ntiles > 0) {
        sb::compose1d_kernel<T, HALF><<<(unsigned)sc->blocks, sb::C1_WARPS * 32,
            sb::compose1d_smem_bytes<T, HALF>(), P->stream>>>(cp);
        SB_CUDA(cudaGetLastError());
    }
    if (sc->nedge > 0) SB_CUDA(cudaStreamWaitEvent(P->stream, P->join_ev, 0));
    return SB_OK;
}

template <typename T, int R, bool FMA>
int launch_fused1d_r(sb_plan* P, const T* src, T* dst, int k) {
    static const int mode = (int)env_double("SB200_1D_MODE", 0);
    static const int compose = (int)env_double("SB200_1D_COMPOSE", 1);
    constexpr int VEC = sb::Vec16<T>::n;
    // composed path: FMA mode, depth >= 2, 16 B aligned halo, line long enough
    // (measured: it wins at k = 16 -- 3.6k vs 2.4k GStencil/s on C2 -- and loses at k <= 8,
    //  where the level-by-level kernel's memory pipeline is the better one)
    if (FMA && compose && compose1d_ok(P, k, compose > 1 ? 2 : 16)) {
        switch (k) {
            case 2: return launch_compose1d_k<T, R, 2>(P, src, dst);
            case 4: return launch_compose1d_k<T, R, 4>(P, src, dst);
            case 8: return launch_compose1d_k<T, R, 8>(P, src, dst);
            case 16: return launch_compose1d_k<T, R, 16>(P, src, dst);
            case 32: return launch_compose1d_k<T, R, 32>(P, src, dst);
            case 64:
                if constexpr (R == 1) return launch_compose1d_k<T, R, 64>(P, src, dst);
                break;
            default: break;
        }
    }
    switch (k) {
        case 1: return launch_fused1d_k<T, R, 1, FMA, 1, 3, false>(P, src, dst);
        case 2: return launch_fused1d_k<T, R, 2, FMA, 1, 3, false>(P, src, dst);
        case 4: return launch_fused1d_k<T, R, 4, FMA, 1, 3, false>(P, src, dst);
        case 8:
            if (mode == 1) return launch_fused1d_k<T, R, 8, FMA, 1, 6, true>(P, src, dst);
            if (mode == 2) return launch_fused1d_k<T, R, 8, FMA, 1, 3, false, true>(P, src, dst);
            if (mode == 3) return launch_fused1d_k<T, R, 8, FMA, 1, 4, false>(P, src, dst);
            if (mode == 4) return launch_fused1d_k<T, R, 8, FMA, 1, 5, false>(P, src, dst);
            return launch_fused1d_k<T, R, 8, FMA, 1, 3, false>(P, src, dst);
        case 16:
            if (mode == 1) return launch_fused1d_k<T, R, 16, FMA, 1, 6, true>(P, src, dst);
            if (mode == 2) return launch_fused1d_k<T, R, 16, FMA, 1, 3, false, true>(P, src, dst);
            if (mode == 3) return launch_fused1d_k<T, R, 16, FMA, 1, 4, false>(P, src, dst);
            if (mode == 4) return launch_fused1d_k<T, R, 16, FMA, 1, 5, false>(P, src, dst);
            return launch_fused1d_k<T, R, 16, FMA, 1, 3, false>(P, src, dst);
        default: return fail(SB_ERR_ARG, "unsupported fused depth %d", k);
    }
}

template <typename T, bool FMA>
int launch_fused1d_t(sb_plan* P, const T* src, T* dst, int k) {
    if (P->r == 1) return launch_fused1d_r<T, 1, FMA>(P, src, dst, k);
    return launch_fused1d_r<T, 2, FMA>(P, src, dst, k);
}


}  // namespace

int launch_fused1d(sb_plan* P, int src_idx, int k) {
    const bool fma = P->arith == SB_ARITH_FMA;
    if (P->dtype == SB_F64) {
        auto src = reinterpret_cast<const double*>(P->buf[src_idx]);
        auto dst = reinterpret_cast<double*>(P->buf[src_idx ^ 1]);
        return fma ? launch_fused1d_t<double, true>(P, src, dst, k) : launch_fused1d_t<double, false>(P, src, dst, k);
    }
    auto src = reinterpret_cast<const float*>(P->buf[src_idx]);
    auto dst = reinterpret_cast<float*>(P->buf[src_idx ^ 1]);
    return fma ? launch_fused1d_t<float, true>(P, src, dst, k) : launch_fused1d_t<float, false>(P, src, dst, k);
}

}  // namespace sbh
