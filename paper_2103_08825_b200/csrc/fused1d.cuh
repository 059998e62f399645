// K1 -- fused 1D sweep: K time steps per HBM round trip.
//
// GPU recast of the paper's two 1D devices:
//  * dimension-lifted layout (stencilbench/kernels.py:352-399, transpose.py:
//    316-357): every lane of a warp owns one contiguous substream, so
//    unit-stride neighbours are the lane's own previous/next values -- no
//    cross-lane reorganisation at all;
//  * time-loop unroll-and-jam (timejam.py:211-304): each lane streams its
//    substream once and advances every value K levels between load and
//    store -- the register pipeline of jam_sweep generalised from k<=2 to any
//    K.  Substreams overlap by R*K (+alignment) on each side (ghost-zone
//    recompute) so lanes and warps never synchronise with each other.
//
// Accumulation is "push" form: when a level-(l-1) value at position p
// arrives it is folded into the 2R+1 pending level-l sums of outputs
// p-R..p+R.  Each output still receives its terms in canonical offset order
// -R..R (kernels.py:103-108; bit-exact in EXACT mode), but the 2R+1 FMAs an
// arriving value triggers are independent, so the FP64 pipe sees ILP of
// 2R+1 per level instead of one dependent chain.
//
// Work distribution: a persistent grid; each warp repeatedly claims a chunk
// (32 substreams of S points each) from a host-built guided schedule through
// one global atomic, so SMs that run faster take more chunks (the static
// one-wave split left SMs idle for ~1/3 of the launch).  The counter resets
// itself when the last warp leaves, ready for the next launch in the stream.
//
// Memory path: global -> shared by cp.async (16 B, L2-only) into a per-warp
// ring of NST stages, each stage holding Q contiguous points of each of the
// 32 substreams (fully used 64 B segments); outputs are staged per lane in
// shared memory and written back as coalesced 16 B vectors.
//
// Boundaries: positions outside [0, n) on a physical side are Dirichlet halo
// -- the same value at every level (HaloEdges, timejam.py:53-71): an output
// landing there is replaced by the halo value itself.  On a slab side
// (multi-GPU ghost zone) they are computed like interior points; validity
// then needs ghost depth >= R*K.
#pragma once
#include "common.cuh"

namespace sb {

template <typename T> struct Vec16;
template <> struct Vec16<double> { using type = double2; static constexpr int n = 2; };
template <> struct Vec16<float> { using type = float4; static constexpr int n = 4; };

struct Chunk1D {
    int64_t start;   // first output position of substream 0
    int32_t S;       // outputs per substream (multiple of Q)
    int32_t pad;
};

template <typename T, int R>
struct Fused1DParams {
    const T* src;            // interior position 0 of the source buffer
    T* dst;                  // interior position 0 of the destination buffer
    int64_t n;               // interior points
    const Chunk1D* chunks;   // guided schedule
    int32_t nchunks;         // interior chunks (fused1d_kernel); edge chunks follow
    int32_t total_warps;     // warps in the grid (for the counter reset)
    unsigned int* counter;   // [0] next chunk, [1] retired warps
    unsigned long long* trace;  // debug (SB200_TRACE): per chunk {smid|warp, t0, t1}
    int phys_lo, phys_hi;
    T w[2 * R + 1];          // canonical order: offsets -R..R
};

template <typename T, int NST_ = 3>
struct Fused1DShape {
    static constexpr int VEC = Vec16<T>::n;    // elements per 16 B
    static constexpr int Q = 64 / sizeof(T);   // points per lane per stage (64 B)
    static constexpr int CH = Q / VEC;         // 16 B chunks per lane-stage
    static constexpr int QP = Q + VEC;         // padded shared row (80 B)
    static constexpr int NST = NST_;            // input ring depth
    static constexpr int WARPS = 4;            // warps per CTA
    static constexpr int IN_ELEMS = NST * 32 * QP;
    static constexpr int OUT_ELEMS = 2 * 32 * QP;
    static constexpr int SMEM_BYTES = WARPS * (IN_ELEMS + OUT_ELEMS) * (int)sizeof(T);
};

template <int R, int K, int VEC, bool DIAG = false>
struct Fused1DLead {
    static constexpr int RK = R * K;
    static constexpr int LEAD = ((RK + VEC - 1) / VEC) * VEC;   // >= RK, 16 B aligned
    static constexpr int PRE = LEAD + RK + (DIAG ? K - 1 : 0);   // stream step of output 0
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

// One chunk: 32 substreams starting at `start`, S outputs each.
template <typename T, int R, int K, bool FMA, bool EDGE, int NST_, bool DIAG>
__device__ __forceinline__ void fused1d_chunk(const Fused1DParams<T, R>& P, T* in_s, T* out_s,
                                              int64_t start, int64_t S, int lane) {
    using SH = Fused1DShape<T, NST_>;
    using LD = Fused1DLead<R, K, SH::VEC, DIAG>;
    using V = typename Vec16<T>::type;
    constexpr int Q = SH::Q, VEC = SH::VEC, CH = SH::CH, QP = SH::QP, NST = SH::NST;
    constexpr int W = 2 * R + 1;
    const int64_t J = LD::PRE + S;
    const int64_t NS = (J + Q - 1) / Q;
    const int64_t a = start + lane * S;     // first output of this lane

    auto issue = [&](int64_t st) {
        T* slot = in_s + (int)(st % NST) * 32 * QP;
#pragma unroll
        for (int i = 0; i < CH; i++) {
            const int c = lane + 32 * i;
            const int seg = c / CH, part = c % CH;
            const bool valid = st < NS;
            const T* g = P.src + (valid ? (start + seg * S - LD::LEAD + st * Q + part * VEC) : 0);
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
            const int64_t pos = start + seg * S + ob * Q + part * VEC;
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

    // acc[l][j]: pending level-(l+1) sum for the output R-j positions before
    // the next level-l value to be pushed.  pend[l]: the level-l value waiting
    // to be pushed into level l (produced one diagonal earlier).
    T acc[K][W];
    T pend[K];
#pragma unroll
    for (int l = 0; l < K; l++) {
        pend[l] = T(0);
#pragma unroll
        for (int j = 0; j < W; j++) acc[l][j] = T(0);
    }
    T ov[VEC];
    // the 2R physical halo values (read once; EDGE chunks only)
    T halo_lo[R], halo_hi[R];
#pragma unroll
    for (int m = 0; m < R; m++) {
        halo_lo[m] = EDGE && P.phys_lo ? P.src[-1 - m] : T(0);
        halo_hi[m] = EDGE && P.phys_hi ? P.src[P.n + m] : T(0);
    }

#pragma unroll
    for (int st = 0; st < NST - 1; st++) issue(st);

    // Diagonal wavefront: at stream step t, level l pushes its element t-l
    // (the level-0 input of step t, or pend[l] made by level l-1 at step t-1),
    // so the K pushes of one step are mutually independent.
    for (int64_t s = 0; s < NS; s++) {
        cp_async_wait<NST - 2>();
        __syncwarp();
        issue(s + NST - 1);
        const T* row = in_s + (int)(s % NST) * 32 * QP + lane * QP;
        const int64_t p0 = a - LD::LEAD + s * Q;     // position of the step-q input
        V xv;
#pragma unroll
        for (int q = 0; q < Q; q++) {
            if (q % VEC == 0) xv = *reinterpret_cast<const V*>(row + q);
            int rel_lo = 0, rel_hi = 0;
            if (EDGE) {
                const int64_t pq = p0 + q;
                rel_lo = (int)max((int64_t)-(1 << 30), min((int64_t)(1 << 30), pq));
                rel_hi = (int)max((int64_t)-(1 << 30), min((int64_t)(1 << 30), pq - P.n));
            }
            T out = T(0);
#pragma unroll
            for (int li = 0; li < K; li++) {
                // DIAG: levels high-to-low on pend[] (wavefront); else the
                // position-major chain low-to-high through `carry`.
                const int l = DIAG ? K - 1 - li : li;
                const T v = (l == 0) ? reinterpret_cast<const T*>(&xv)[q % VEC] : pend[l];
                T* A = acc[l];
                // the completing term first: the next level waits on it alone
                T done = acc_term<T, FMA>(A[0], P.w[W - 1], v);
#pragma unroll
                for (int j = 1; j < W - 1; j++)
                    A[j] = acc_term<T, FMA>(A[j], P.w[W - 1 - j], v);
                A[W - 1] = acc_first<T, FMA>(P.w[0], v);
                if (EDGE) {
                    // Dirichlet: a halo position keeps its value at every level.
                    // This output sits l + (l+1)R behind the newest input.
                    const int back = (DIAG ? l : 0) + (l + 1) * R;
                    const bool in_lo = P.phys_lo && rel_lo < back;
                    const bool in_hi = P.phys_hi && rel_hi >= back;
                    T h = halo_lo[R - 1];
#pragma unroll
                    for (int m = R - 1; m >= 1; m--) h = (rel_lo == back - m) ? halo_lo[m - 1] : h;
                    T g = halo_hi[R - 1];
#pragma unroll
                    for (int m = R - 2; m >= 0; m--) g = (rel_hi == back + m) ? halo_hi[m] : g;
                    done = in_lo ? h : (in_hi ? g : done);
                }
#pragma unroll
                for (int j = 0; j < W - 1; j++) A[j] = A[j + 1];
                if (l == K - 1) out = done;
                else pend[l + 1] = done;   // DIAG: next step; else: this step, next level
            }
            // out = level K at stream step q - (K-1) = output index s*Q + q - PRE
            const int oq = pos_mod(q - LD::PRE, Q);
            ov[oq % VEC] = out;
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
    __syncwarp();
}

template <typename T, int R, int K, bool FMA, int MINB, int NST_, bool DIAG>
__global__ void __launch_bounds__(Fused1DShape<T, NST_>::WARPS * 32, MINB)
fused1d_kernel(const Fused1DParams<T, R> P) {
    using SH = Fused1DShape<T, NST_>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* smem = reinterpret_cast<T*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    T* in_s = smem + warp * (SH::IN_ELEMS + SH::OUT_ELEMS);
    T* out_s = in_s + SH::IN_ELEMS;
    for (;;) {
        unsigned id = 0;
        if (lane == 0) id = atomicAdd(&P.counter[0], 1u);
        id = __shfl_sync(0xffffffffu, id, 0);
        if (id >= (unsigned)P.nchunks) break;
        const Chunk1D c = P.chunks[id];
        unsigned long long t0 = 0;
        if (P.trace && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        fused1d_chunk<T, R, K, FMA, false, NST_, DIAG>(P, in_s, out_s, c.start, c.S, lane);
        if (P.trace && lane == 0) {
            unsigned long long t1;
            unsigned s32;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            asm volatile("mov.u32 %0, %%smid;" : "=r"(s32));
            P.trace[4 * id + 0] = ((unsigned long long)s32 << 32) | (blockIdx.x * SH::WARPS + warp);
            P.trace[4 * id + 1] = t0;
            P.trace[4 * id + 2] = t1;
            P.trace[4 * id + 3] = ((unsigned long long)c.S << 40) | (unsigned long long)c.start;
        }
    }
    if (lane == 0) {
        const unsigned retired = atomicAdd(&P.counter[1], 1u);
        if (retired == (unsigned)P.total_warps - 1) {   // last warp out resets for the next launch
            atomicExch(&P.counter[0], 0u);
            atomicExch(&P.counter[1], 0u);
        }
    }
}

// Chunks touching a physical boundary (EDGE path), one warp each; launched on
// a side stream concurrently with fused1d_kernel so the interior kernel
// carries no boundary code (registers) and no warp stalls the queue's tail.
template <typename T, int R, int K, bool FMA, int NST_, bool DIAG>
__global__ void __launch_bounds__(32)
fused1d_edge_kernel(const Fused1DParams<T, R> P) {
    using SH = Fused1DShape<T, NST_>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* in_s = reinterpret_cast<T*>(smem_raw);
    T* out_s = in_s + SH::IN_ELEMS;
    const Chunk1D c = P.chunks[P.nchunks + blockIdx.x];
    fused1d_chunk<T, R, K, FMA, true, NST_, DIAG>(P, in_s, out_s, c.start, c.S, threadIdx.x & 31);
}

}  // namespace sb
