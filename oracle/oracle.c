/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the multistep stencil sweep.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the timed CPU baseline; the product path (paper_2103_08825_b200) never
 * links or calls it.
 *
 * This is a plain-C restatement of the reference's scalar oracle:
 *   stencilbench/kernels.py:103-108  _natural_accumulate
 *       out = region(dst); out[...] = 0.0
 *       for off in spec.offsets: out += spec.weights[off] * region(src, off)
 *   stencilbench/kernels.py:120-134  scalar_step (out-of-place, halo read-only)
 *   stencilbench/harness.py:149-157  run_oracle (T steps, ping-pong buffers)
 *   stencilbench/core.py:96-103      canonical (lexicographic) offset order
 *
 * Arithmetic contract (bit-exact with the numpy oracle): per point the
 * accumulator starts at +0.0 and, for every offset in canonical order, one
 * rounded multiply w*x followed by one rounded add.  The file MUST be built
 * with -ffp-contract=off (see oracle/Makefile) so no FMA is formed.
 *
 * Storage convention (the C-ABI's host convention, include/sb200.h): a
 * compact C-order box of shape (n_0+2r, ..., n_{d-1}+2r) holding interior
 * plus an r-deep Dirichlet halo that is read and never written.
 * Parallelised over (row, x-chunk) tasks with OpenMP; results do not depend on the thread
 * count (each point's sum is computed by one thread in canonical order).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int64_t n[3];      /* interior extents, canonicalised to 3D (leading 1s) */
    int64_t s[3];      /* element strides of the storage box */
    int64_t h[3];      /* halo per axis (r on real axes, 0 on padded ones) */
    int64_t total;     /* elements in the storage box */
} geom3;

static int make_geom(int d, int r, const int64_t *dims, geom3 *g) {
    if (d < 1 || d > 3 || r < 1) return -1;
    for (int a = 0; a < 3; a++) { g->n[a] = 1; g->h[a] = 0; }
    for (int a = 0; a < d; a++) {
        if (dims[a] <= 0) return -1;
        g->n[3 - d + a] = dims[a];
        g->h[3 - d + a] = r;
    }
    g->s[2] = 1;
    g->s[1] = g->n[2] + 2 * g->h[2];
    g->s[0] = g->s[1] * (g->n[1] + 2 * g->h[1]);
    g->total = g->s[0] * (g->n[0] + 2 * g->h[0]);
    return 0;
}

/* Linear element offset of each stencil offset, canonical order preserved. */
static int64_t *lin_offsets(int d, int nw, const int32_t *offsets, const geom3 *g) {
    int64_t *lin = (int64_t *)malloc(sizeof(int64_t) * (size_t)nw);
    if (!lin) return NULL;
    for (int i = 0; i < nw; i++) {
        int64_t o = 0;
        for (int a = 0; a < d; a++) o += (int64_t)offsets[i * d + a] * g->s[3 - d + a];
        lin[i] = o;
    }
    return lin;
}

/* Work is split into (row, x-chunk) tasks so 1D lines use every thread too;
 * each point is still computed by one thread in canonical order. */
#define OR_CHUNK 2048   /* 16 KB of `out`: stays in L1 across the per-offset passes */
#define DEFINE_STEP(NAME, T)                                                       \
__attribute__((target_clones("avx2", "default")))                                  \
static void NAME(const T *src, T *dst, const geom3 *g, int nw,                     \
                 const int64_t *lin, const T *w, int nthreads) {                   \
    const int64_t nz = g->n[0], ny = g->n[1], nx = g->n[2];                        \
    const int64_t base0 = g->h[0] * g->s[0] + g->h[1] * g->s[1] + g->h[2];         \
    const int64_t nch = (nx + OR_CHUNK - 1) / OR_CHUNK;                            \
    const int64_t tasks = nz * ny * nch;                                           \
    (void)nthreads;                                                                \
    _Pragma("omp parallel for schedule(static) num_threads(nthreads)")             \
    for (int64_t task = 0; task < tasks; task++) {                                 \
        const int64_t c = task % nch, zy = task / nch;                             \
        const int64_t z = zy / ny, y = zy % ny;                                    \
        const int64_t x0 = c * OR_CHUNK;                                           \
        const int64_t x1 = x0 + OR_CHUNK < nx ? x0 + OR_CHUNK : nx;                \
        const int64_t row = base0 + z * g->s[0] + y * g->s[1];                     \
        T *out = dst + row;                                                        \
        for (int64_t x = x0; x < x1; x++) out[x] = (T)0;                           \
        for (int i = 0; i < nw; i++) {                                             \
            const T wi = w[i];                                                     \
            const T *in = src + row + lin[i];                                      \
            for (int64_t x = x0; x < x1; x++) {                                    \
                T prod = wi * in[x];                                               \
                out[x] = out[x] + prod;                                            \
            }                                                                      \
        }                                                                          \
    }                                                                              \
}

DEFINE_STEP(step_f64, double)
DEFINE_STEP(step_f32, float)

#define DEFINE_SWEEP(NAME, STEP, T)                                                \
int NAME(int d, int r, int nw, const int32_t *offsets, const double *weights,      \
         const int64_t *dims, T *grid, int64_t steps, int nthreads) {              \
    geom3 g;                                                                       \
    if (make_geom(d, r, dims, &g) != 0 || nw < 1 || steps < 0) return -1;          \
    if (nthreads < 1) nthreads = 1;                                                \
    int64_t *lin = lin_offsets(d, nw, offsets, &g);                                \
    T *w = (T *)malloc(sizeof(T) * (size_t)nw);                                    \
    T *other = (T *)malloc(sizeof(T) * (size_t)g.total);                           \
    if (!lin || !w || !other) { free(lin); free(w); free(other); return -2; }      \
    for (int i = 0; i < nw; i++) w[i] = (T)weights[i];                             \
    memcpy(other, grid, sizeof(T) * (size_t)g.total); /* halo in both buffers */   \
    T *a = grid, *b = other;                                                       \
    for (int64_t t = 0; t < steps; t++) {                                          \
        STEP(a, b, &g, nw, lin, w, nthreads);                                      \
        T *tmp = a; a = b; b = tmp;                                                \
    }                                                                              \
    if (a != grid) memcpy(grid, a, sizeof(T) * (size_t)g.total);                   \
    free(lin); free(w); free(other);                                               \
    return 0;                                                                      \
}

/* T oracle steps in place on a compact halo-inclusive box (fp64). */
DEFINE_SWEEP(sbo_sweep_f64, step_f64, double)
/* Same restatement carried out in fp32 (secondary fp32 check only). */
DEFINE_SWEEP(sbo_sweep_f32, step_f32, float)

int sbo_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
