// K1 -- fused 1D sweep: K time steps per HBM round trip.
//
// GPU recast of the paper's two 1D devices:
//  * dimension-lifted layout (stencilbench/kernels.py:352-399, transpose.py:
//    316-357): every lane of a warp owns one contiguous substream of S output
//    points, so unit-stride neighbours are the lane's own previous/next
//    values -- no cross-lane reorganisation at all;
//  * time-loop unroll-and-jam (timejam.py:211-304): each lane streams its
//    substream once and advances every value K levels between load and
//    store, keeping a (2R+1)-wide register window per level -- the register
//    pipeline of jam_sweep generalised from k<=2 to any K.
// Substreams overlap by R*K on each side (ghost-zone recompute) so warps and
// lanes never synchronise with each other.
//
// Memory path: global -> shared by cp.async (16 B, L2-only) into a per-warp
// ring of NST stages, each stage holding Q contiguous points of each of the
// 32 substreams (fully used 64 B segments); outputs are staged per lane in
// shared memory and written back as coalesced 16 B vectors.  Shared rows are
// padded to 80 B so the per-lane 16 B reads/writes are conflict-free.
//
// Boundaries: positions outside [0, n) on a physical side are Dirichlet halo
// -- at every level they pass through unchanged (HaloEdges, timejam.py:
// 53-71: the halo is the same at every level).  On a slab side (multi-GPU
// ghost zone) they are computed like interior points; validity then needs
// ghost depth >= R*K.
#pragma once
#include "common.cuh"

namespace sb {

template <typename T> struct Vec16;
template <> struct Vec16<double> { using type = double2; static constexpr int n = 2; };
template <> struct Vec16<float> { using type = float4; static constexpr int n = 4; };

template <typename T, int R>
struct Fused1DParams {
    const T* src;     // interior position 0 of the source buffer
    T* dst;           // interior position 0 of the destination buffer
    int64_t n;        // interior points
    int64_t S;        // outputs per lane (multiple of Q)
    int64_t nlanes;   // lanes with work = ceil(n / S)
    int phys_lo, phys_hi;
    T w[2 * R + 1];   // canonical order: offsets -R..R
};

template <typename T>
struct Fused1DShape {
    static constexpr int VEC = Vec16<T>::n;    // elements per 16 B
    static constexpr int Q = 64 / sizeof(T);   // points per lane per stage (64 B)
    static constexpr int CH = Q / VEC;         // 16 B chunks per lane-stage
    static constexpr int QP = Q + VEC;         // padded shared row (80 B)
    static constexpr int NST = 3;              // input ring depth
    static constexpr int WARPS = 4;            // warps per CTA
    static constexpr int IN_ELEMS = NST * 32 * QP;
    static constexpr int OUT_ELEMS = 2 * 32 * QP;
    static constexpr int SMEM_BYTES = WARPS * (IN_ELEMS + OUT_ELEMS) * (int)sizeof(T);
};

template <int R, int K, int VEC>
struct Fused1DLead {
    static constexpr int RK = R * K;
    static constexpr int LEAD = ((RK + VEC - 1) / VEC) * VEC;   // >= RK, 16 B aligned
    static constexpr int PRE = LEAD + RK;                        // stream index of output 0
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int bytes = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__host__ __device__ constexpr int floor_div(int a, int b) { return (a >= 0) ? a / b : -((-a + b - 1) / b); }
__host__ __device__ constexpr int pos_mod(int a, int b) { return ((a % b) + b) % b; }

template <typename T, int R, int K, bool FMA, bool EDGE>
__device__ __forceinline__ void fused1d_warp(const Fused1DParams<T, R>& P, T* in_s, T* out_s,
                                             int64_t base_lane, int lane) {
    using SH = Fused1DShape<T>;
    using LD = Fused1DLead<R, K, SH::VEC>;
    using V = typename Vec16<T>::type;
    constexpr int Q = SH::Q, VEC = SH::VEC, CH = SH::CH, QP = SH::QP, NST = SH::NST;
    constexpr int W = 2 * R + 1;
    const int64_t S = P.S;
    const int64_t J = LD::PRE + S;
    const int64_t NS = (J + Q - 1) / Q;
    const int64_t a = (base_lane + lane) * S;     // first output of this lane

    auto issue = [&](int64_t st) {
        T* slot = in_s + (int)(st % NST) * 32 * QP;
#pragma unroll
        for (int i = 0; i < CH; i++) {
            const int c = lane + 32 * i;
            const int seg = c / CH, part = c % CH;
            const int64_t lane_g = base_lane + seg;
            const bool valid = (lane_g < P.nlanes) && (st < NS);
            const T* g = P.src + (valid ? (lane_g * S - LD::LEAD + st * Q + part * VEC) : 0);
            cp_async16(slot + seg * QP + part * VEC, g, valid);
        }
        cp_async_commit();
    };

    auto flush = [&](int64_t ob) {
        __syncwarp();
        const T* half = out_s + (int)(ob & 1) * 32 * QP;
#pragma unroll
        for (int i = 0; i < CH; i++) {
            const int c = lane + 32 * i;
            const int seg = c / CH, part = c % CH;
            const int64_t pos = (base_lane + seg) * S + ob * Q + part * VEC;
            const V v = *reinterpret_cast<const V*>(half + seg * QP + part * VEC);
            if (pos + VEC <= P.n) {
                *reinterpret_cast<V*>(P.dst + pos) = v;
            } else {
                const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
                for (int j = 0; j < VEC; j++)
                    if (pos + j < P.n) P.dst[pos + j] = e[j];
            }
        }
    };

    // win[l][i]: level-l values at positions (newest - 2R + i); level 0 = input.
    T win[K][W];
#pragma unroll
    for (int l = 0; l < K; l++)
#pragma unroll
        for (int i = 0; i < W; i++) win[l][i] = T(0);
    T ov[VEC];

#pragma unroll
    for (int st = 0; st < NST - 1; st++) issue(st);

    for (int64_t s = 0; s < NS; s++) {
        cp_async_wait<NST - 2>();
        __syncwarp();
        issue(s + NST - 1);
        const T* row = in_s + (int)(s % NST) * 32 * QP + lane * QP;
        const int64_t p0 = a - LD::LEAD + s * Q;     // position of q = 0
        V xv;
#pragma unroll
        for (int q = 0; q < Q; q++) {
            if (q % VEC == 0) xv = *reinterpret_cast<const V*>(row + q);
            const T x = reinterpret_cast<const T*>(&xv)[q % VEC];
#pragma unroll
            for (int i = 0; i < W - 1; i++) win[0][i] = win[0][i + 1];
            win[0][W - 1] = x;
            T v = T(0);
#pragma unroll
            for (int l = 1; l <= K; l++) {
                const T* c = win[l - 1];
                T acc = acc_first<T, FMA>(P.w[0], c[0]);
#pragma unroll
                for (int i = 1; i < W; i++) acc = acc_term<T, FMA>(acc, P.w[i], c[i]);
                if (EDGE) {
                    const int64_t pos = p0 + q - (int64_t)l * R;
                    const bool halo = (P.phys_lo && pos < 0) || (P.phys_hi && pos >= P.n);
                    acc = halo ? c[R] : acc;
                }
                if (l < K) {
#pragma unroll
                    for (int i = 0; i < W - 1; i++) win[l][i] = win[l][i + 1];
                    win[l][W - 1] = acc;
                } else {
                    v = acc;
                }
            }
            // output index o = s*Q + q - PRE; its residues are compile-time.
            const int oq = pos_mod(q - LD::PRE, Q);
            ov[oq % VEC] = v;
            if (oq % VEC == VEC - 1) {
                const int64_t ob = s + floor_div(q - LD::PRE, Q);
                T* dstrow = out_s + (int)(ob & 1) * 32 * QP + lane * QP + (oq - (VEC - 1));
                V pack;
#pragma unroll
                for (int j = 0; j < VEC; j++) reinterpret_cast<T*>(&pack)[j] = ov[j];
                *reinterpret_cast<V*>(dstrow) = pack;
                if (oq == Q - 1 && ob >= 0 && ob < S / Q) flush(ob);
            }
        }
    }
    cp_async_wait<0>();
}

template <typename T, int R, int K, bool FMA>
__global__ void __launch_bounds__(Fused1DShape<T>::WARPS * 32)
fused1d_kernel(const Fused1DParams<T, R> P) {
    using SH = Fused1DShape<T>;
    using LD = Fused1DLead<R, K, SH::VEC>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* smem = reinterpret_cast<T*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t gwarp = (int64_t)blockIdx.x * SH::WARPS + warp;
    const int64_t base_lane = gwarp * 32;
    if (base_lane >= P.nlanes) return;
    T* in_s = smem + warp * (SH::IN_ELEMS + SH::OUT_ELEMS);
    T* out_s = in_s + SH::IN_ELEMS;
    const int64_t last_lane = min(base_lane + 31, P.nlanes - 1);
    const int64_t J = LD::PRE + P.S;
    const int64_t first_pos = base_lane * P.S - LD::LEAD;
    const int64_t last_pos = last_lane * P.S - LD::LEAD + ((J + SH::Q - 1) / SH::Q) * SH::Q;
    const bool edge = (P.phys_lo && first_pos < 0) || (P.phys_hi && last_pos >= P.n);
    if (edge)
        fused1d_warp<T, R, K, FMA, true>(P, in_s, out_s, base_lane, lane);
    else
        fused1d_warp<T, R, K, FMA, false>(P, in_s, out_s, base_lane, lane);
}

}  // namespace sb
