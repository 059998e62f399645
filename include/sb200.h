/*
 * sb200 -- C ABI of the B200-native multistep stencil sweep.
 *
 * Drop-in boundary for the reference package ``stencilbench`` (a pure
 * Python + numpy package; its "plugin interface" is the method registry and
 * the step/sweep call signatures, not an FFI).  Each entry point below names
 * the reference interface it replaces:
 *
 *   sb_plan_create   <- StencilSpec validation + alloc_grid/alloc_like
 *                       (stencilbench/core.py:54-106, core.py:335-373)
 *   sb_upload        <- GridBuffer.set_interior / seeded halo
 *                       (core.py:318-327, harness.py:139-146)
 *   sb_run           <- the T-step loop of harness._execute
 *                       (harness.py:195-201) over scalar_step
 *                       (kernels.py:120-134) and the k-level time jam
 *                       jam_sweep (timejam.py:288-304)
 *   sb_download      <- GridBuffer.natural_interior (core.py:308-316)
 *   sb_step_box      <- scalar_step(..., ranges=...) as driven by the tiled
 *                       runner (tiling.py:353-354)
 *   sb_launch_range  <- (no reference counterpart: slab edge planes first, then
 *                       the interior, overlapping the ghost exchange)
 *   sb_upload_storage / sb_download_storage / sb_layout_convert
 *                    <- the layout conversions of transpose.py:266-357
 *                       (BLOCK_TRANSPOSE / DLT storage), see below
 *   sb_upload_async / sb_download_async / sb_synchronize
 *                    <- (no reference counterpart: stream-ordered transfers
 *                       for overlapping independent grids' sweeps)
 *   sb_plan_destroy  <- (buffers going out of scope)
 *   sb_last_error    <- exception messages of SpecError/GridError
 *                       (core.py:38-43)
 *
 * Host buffers use one convention everywhere: a compact C-order box of the
 * halo-inclusive grid, shape (n_0 + h_lo + h_hi, n_1 + 2r, ..., n_{d-1} + 2r)
 * where h_lo/h_hi are r (physical Dirichlet halo) or the ghost depth of a
 * slab side (multi-GPU).  Halo cells are read, never written, and are
 * preserved bit-for-bit.  Element type is double (SB_F64) or float (SB_F32).
 *
 * Conventions: functions return SB_OK (0) or a negative sb_status; the
 * message is available from sb_last_error() (thread-local).  A plan owns its
 * device memory and stream; one host thread per plan.  There is no CPU
 * fallback: without a CUDA device every compute call fails with SB_ERR_CUDA.
 */
#ifndef SB200_H
#define SB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SB200_ABI_VERSION 1

typedef enum {
    SB_OK = 0,
    SB_ERR_SPEC = -1,   /* invalid stencil (SpecError) */
    SB_ERR_GRID = -2,   /* invalid geometry / buffer size (GridError) */
    SB_ERR_ARG = -3,    /* invalid argument (ValueError) */
    SB_ERR_CUDA = -4,   /* CUDA runtime failure or no device (RuntimeError) */
    SB_ERR_NOMEM = -5,  /* device or host allocation failed (MemoryError) */
    SB_ERR_STATE = -6   /* call out of order, e.g. run before upload */
} sb_status;

typedef enum { SB_F64 = 0, SB_F32 = 1 } sb_dtype;

/* EXACT: per term one rounded multiply then one rounded add, canonical
 * order, accumulator from +0.0 -- bit-identical to the reference oracle
 * (kernels.py:103-108).  FMA: first term a multiply, then fused
 * multiply-adds in canonical order (<= 1e-12 relative vs the oracle). */
typedef enum { SB_ARITH_EXACT = 0, SB_ARITH_FMA = 1 } sb_arith;

typedef enum { SB_STAR = 0, SB_BOX = 1 } sb_shape;

/* AUTO picks the fused temporal-blocking kernel when one exists for the
 * stencil class, else GENERIC (one step per launch, any d/r/shape). */
typedef enum { SB_KERNEL_AUTO = 0, SB_KERNEL_GENERIC = 1, SB_KERNEL_FUSED = 2 } sb_kernel;

typedef struct sb_problem {
    int32_t d;               /* 1, 2 or 3 */
    int32_t r;               /* order (max per-axis distance), >= 1 */
    int32_t shape;           /* sb_shape */
    int32_t nw;              /* number of weights */
    const int32_t *offsets;  /* nw*d offsets, canonical (lexicographic) order */
    const double *weights;   /* nw weights matching offsets */
    int64_t dims[3];         /* interior extents, slowest axis first */
    int32_t dtype;           /* sb_dtype */
    int32_t arith;           /* sb_arith */
    int32_t k;               /* fused steps per launch; 0 = auto */
    int32_t kernel;          /* sb_kernel */
    int32_t device;          /* CUDA device ordinal */
    int32_t ghost_lo;        /* slab side below: 0 = physical halo r; G>0 = G ghost planes */
    int32_t ghost_hi;        /* slab side above: same convention */
} sb_problem;

typedef struct sb_timing {
    double device_ms;        /* CUDA-event time of the whole call on the plan stream */
    double kernel_ms;        /* equal to device_ms: sb_run enqueues kernels only (no copies) */
    int64_t launches;        /* kernels launched by the call */
    int64_t point_updates;   /* interior points x steps (Counters.point_updates) */
    int32_t k_used;          /* fused steps per main launch */
    int32_t reserved;
    char kernel_name[64];    /* main kernel used */
} sb_timing;

typedef struct sb_plan sb_plan;

int sb_plan_create(sb_plan **plan, const sb_problem *problem);
void sb_plan_destroy(sb_plan *plan);

/* Number of elements of the host box (see convention above). */
int sb_host_elems(const sb_plan *plan, int64_t *elems);

/* Host box -> device (both ping-pong buffers; halo/ghost included). */
int sb_upload(sb_plan *plan, const void *host, size_t bytes);
/* Device (current buffer) -> host box, halo included. */
int sb_download(sb_plan *plan, void *host, size_t bytes);

/* The same with the host box given as uniformly pitched rows: row i of the box
 * (sb_host_elems / row-elements rows, slowest axes first) starts at
 * host + i * pitch_bytes, pitch_bytes >= the row's bytes.  A NATURAL
 * GridBuffer.data (stencilbench/core.py:232-373) whose halo equals the stencil
 * order is such a box -- first row at &data[..., halo_unit - r], pitch = one
 * storage row -- so b200_sweep moves it without a compacting host copy;
 * sb_download_pitched writes the box's rows back (the halo cells get the values
 * they already hold, cells outside the box are not touched). */
int sb_upload_pitched(sb_plan *plan, const void *host, size_t pitch_bytes);
int sb_download_pitched(sb_plan *plan, void *host, size_t pitch_bytes);

/* Host box in, `steps` steps, host box out (pitches as above; 0 = compact rows;
 * in and out may be the same memory): upload, run, download in one call.  3D
 * whole-grid plans can overlap the transfers with the sweep (default with pinned
 * host memory on both sides and few launches; SB200_STREAM_SWEEP=1/0 forces it
 * on / off): the grid is cut into blocks of planes, every launch
 * of the sweep runs block by block on ranges shifted down by the reach of the
 * launches before it, so a block's launches start once its planes have arrived
 * and its final planes travel back while later blocks compute -- the same range
 * launches as sb_launch_range, bit-identical to upload + run + download.  Other
 * plans run exactly that sequence.  The grid-in/grid-out call of the drop-in
 * (harness._execute's loop, harness.py:187-201, around one method). */
int sb_sweep_host(sb_plan *plan, const void *host_in, size_t in_pitch_bytes, void *host_out,
                  size_t out_pitch_bytes, int64_t steps);

/* Stream-ordered forms of sb_upload / sb_download on the plan stream: they
 * return once the copy is enqueued.  `host` must stay valid (and should be
 * page-locked, e.g. cudaHostAlloc, for the copy to overlap other work) until
 * sb_synchronize -- used to overlap one grid's transfers with another
 * plan's sweep (pipelined end-to-end sweeps of independent grids). */
int sb_upload_async(sb_plan *plan, const void *host, size_t bytes);
int sb_download_async(sb_plan *plan, void *host, size_t bytes);
/* Wait for everything enqueued on the plan stream; reports kernel errors. */
int sb_synchronize(sb_plan *plan);

/* Advance `steps` time steps, synchronously; fills *timing if non-NULL.
 * Slab plans (ghost_lo/hi > 0) accept steps <= min ghost depth / r. */
int sb_run(sb_plan *plan, int64_t steps, sb_timing *timing);

/* Same, asynchronously on the plan stream (no host sync, no timing). */
int sb_launch(sb_plan *plan, int64_t steps);

/* `repeats` back-to-back sweeps of `steps` steps (sb_launch each), enqueued
 * from native code: short sweeps (C1: one ~10 us launch) are not bound by the
 * caller's per-call overhead.  Asynchronous.  Events are recorded before the
 * first sweep and after the last, and with per_sweep_events != 0 also
 * between sweeps (each costs ~2.5 us of device time between 10 us launches).
 * sb_repeat_times waits and writes up to `cap` durations (ms): one per sweep,
 * or the whole run; returns how many it recorded. */
int sb_launch_repeat(sb_plan *plan, int64_t steps, int32_t repeats, int32_t per_sweep_events);
int sb_repeat_times(sb_plan *plan, float *sweep_ms, int32_t cap);

/* One fused launch of `steps` levels that writes only the slowest-axis
 * interior positions [lo, hi) of the other buffer, reading the current one.
 * A step is split into several range launches (e.g. the slab's edge planes
 * first, then its interior, so the edge planes can be sent to the neighbours
 * while the interior is computed); the call with finish != 0 completes it
 * (swaps buffers).  d >= 2; `steps` a fused depth of the plan (1 for generic
 * plans) and <= the ghost depth / r on slab sides.  Asynchronous on the plan
 * stream. */
int sb_launch_range(sb_plan *plan, int64_t steps, int64_t lo, int64_t hi, int32_t finish);

/* One step restricted to the interior sub-box lo[a] <= i_a < hi[a] (first d
 * entries, slowest axis first): the reference's `ranges` argument
 * (scalar_step, kernels.py:120-134 / _region, kernels.py:88-100).  Writes
 * only the box of the other buffer (the rest of it is stale), then swaps
 * buffers; synchronous.  Whole-grid plans only. */
int sb_step_box(sb_plan *plan, const int64_t *lo, const int64_t *hi);

/* Run on an external stream (e.g. torch's current stream); NULL restores
 * the plan's own stream. */
int sb_set_stream(sb_plan *plan, void *cuda_stream);

/* Device pointer and element strides of the current buffer, for halo
 * exchange by the multi-GPU host layer.  origin = element offset of
 * interior point (0,...,0); strides[0..d-1] in elements. */
int sb_device_view(const sb_plan *plan, int which, void **base,
                   int64_t *origin, int64_t strides[3]);

/* ---- reference storage layouts (stencilbench/transpose.py, core.py:206-229)
 *
 * A reference GridBuffer stores each unit-stride row as
 * [halo_unit | unit_np padded region | halo_unit] (halo_unit = 2r,
 * core.py:35, 260-266); the padded region is NATURAL, BLOCK_TRANSPOSE (every
 * vl x vl block transposed) or DLT (the region viewed as vl x unit_np/vl and
 * transposed).  Cells in [unit_n, unit_np) are Dirichlet padding. */
typedef enum { SB_LAYOUT_NATURAL = 0, SB_LAYOUT_BLOCK_TRANSPOSE = 1, SB_LAYOUT_DLT = 2 } sb_layout;

typedef struct sb_storage {
    int32_t layout;          /* sb_layout */
    int32_t vl;              /* 4 or 8 (SUPPORTED_VL, core.py:31); ignored for NATURAL */
    int64_t unit_n;          /* interior unit-stride extent */
    int64_t unit_np;         /* padded extent: multiple of vl*vl (BLOCK_TRANSPOSE) / vl (DLT) */
    int64_t halo_unit;       /* unit-axis halo cells per side (>= r; the reference uses 2r) */
} sb_storage;

/* Whole reference storage array (GridBuffer.data: rows of unit_np +
 * 2*halo_unit elements, outer axes with their r halo rows, C order) in layout
 * st -> the plan, un-permuted on the device.  Replaces the host-side
 * from_block_transpose / from_dlt + natural_interior path (transpose.py:
 * 303-311, 338-357) of a caller holding a BLOCK_TRANSPOSE or DLT grid (e.g.
 * jam_sweep's, timejam.py:288-304).  Whole-grid plans only. */
int sb_upload_storage(sb_plan *plan, const void *host, size_t bytes, const sb_storage *st);
/* The plan's current grid -> the same storage array, re-permuted on the
 * device into layout st; every cell that is not an interior point keeps the
 * value of the last sb_upload_storage (required first, same geometry). */
int sb_download_storage(sb_plan *plan, void *host, size_t bytes, const sb_storage *st);
/* Device-to-device conversion of `rows` storage rows (unit_np + 2*halo_unit
 * elements each, dtype sb_dtype): to_layout != 0 converts NATURAL `src` to
 * layout st->layout in `dst` (to_block_transpose / to_dlt, transpose.py:
 * 286-301, 314-336); to_layout == 0 is the inverse (from_block_transpose /
 * from_dlt).  Out-of-place, asynchronous on `stream` (NULL = legacy default
 * stream); halo cells are copied unchanged. */
int sb_layout_convert(void *dst, const void *src, int64_t rows, const sb_storage *st, int32_t to_layout,
                      int32_t dtype, void *stream);

/* ---- single-process multi-GPU sweep (grid in, grid out over `ngpu` devices)
 *
 * The interior is split along the slowest axis into `ngpu` balanced slabs,
 * one slab plan per device (`devices[i]`, NULL = 0 .. ngpu-1; a device may
 * repeat, e.g. to emulate the decomposition on one GPU).  Every slab carries
 * G = r*k ghost planes per side facing another slab; between launches of k
 * fused steps the new edge planes are peer-copied (NVLink, copy streams)
 * into the neighbours' ghost planes, overlapped with the slab interiors
 * (2D/3D).  Results are bit-identical to one device.  Host boxes are the
 * GLOBAL compact halo-inclusive box.  Replaces, for a multi-GPU node, the
 * whole-grid sweep of sb_plan_create/sb_upload/sb_run/sb_download.  */
typedef struct sb_multi sb_multi;
int sb_multi_create(sb_multi **multi, const sb_problem *problem, int32_t ngpu, const int32_t *devices);
void sb_multi_destroy(sb_multi *multi);
int sb_multi_upload(sb_multi *multi, const void *host, size_t bytes);
int sb_multi_download(sb_multi *multi, void *host, size_t bytes);
/* Advance `steps` steps (synchronous); timing->device_ms = max over devices. */
int sb_multi_run(sb_multi *multi, int64_t steps, sb_timing *timing);
int sb_multi_info(const sb_multi *multi, int32_t *ngpu, int32_t *k);
/* Slab i: global interior planes [start, end) on `device`. */
int sb_multi_slab(const sb_multi *multi, int32_t i, int64_t *start, int64_t *end, int32_t *device);

/* Fused depth a plan for `problem` would use (host only, no device needed). */
int sb_problem_k(const sb_problem *problem, int32_t *k);

/* Fused depth the plan will use per launch. */
int sb_plan_k(const sb_plan *plan, int32_t *k);

/* Kernels launched by this plan so far (all kernels: main, boundary, generic). */
int sb_kernel_count(const sb_plan *plan, int64_t *count);

const char *sb_last_error(void);
int sb_abi_version(void);
/* Number of CUDA devices visible (0 without a GPU; never fails). */
int sb_device_count(void);

#ifdef __cplusplus
}
#endif

#endif /* SB200_H */
