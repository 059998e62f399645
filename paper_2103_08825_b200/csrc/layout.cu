// Launch unit of the layout-conversion kernels (layout.cuh): reference
// BLOCK_TRANSPOSE / DLT storage rows <-> the plan's natural pitched rows, and
// standalone device conversions (stencilbench/transpose.py:266-357).
#include "plan.hpp"
#include "layout.cuh"

namespace sbh {
namespace {

int check_storage(const sb_storage* st, int64_t* row_elems) {
    if (!st) return fail(SB_ERR_ARG, "NULL storage descriptor");
    if (st->layout < SB_LAYOUT_NATURAL || st->layout > SB_LAYOUT_DLT)
        return fail(SB_ERR_ARG, "unknown layout %d", st->layout);
    if (st->layout != SB_LAYOUT_NATURAL && st->vl != 4 && st->vl != 8)
        return fail(SB_ERR_GRID, "vl must be one of (4, 8), got %d", st->vl);   // core.py:31, 343-344
    if (st->unit_n <= 0 || st->unit_np < st->unit_n || st->halo_unit < 0)
        return fail(SB_ERR_GRID, "bad storage geometry (unit_n %lld, unit_np %lld, halo_unit %lld)",
                    (long long)st->unit_n, (long long)st->unit_np, (long long)st->halo_unit);
    if (st->layout == SB_LAYOUT_BLOCK_TRANSPOSE && st->unit_np % ((int64_t)st->vl * st->vl))
        return fail(SB_ERR_GRID, "unit extent %lld not padded to a multiple of %d", (long long)st->unit_np,
                    st->vl * st->vl);   // transpose.py:283-285
    if (st->layout == SB_LAYOUT_DLT && st->unit_np % st->vl)
        return fail(SB_ERR_GRID, "unit extent %lld not divisible by %d", (long long)st->unit_np, st->vl);
    *row_elems = st->unit_np + 2 * st->halo_unit;
    return SB_OK;
}

template <typename T>
int launch_xfer(const void* src, void* dst, int64_t rows, int64_t nat_stride, int64_t sto_stride, int64_t nat0,
                int64_t sto0, int64_t i_lo, int64_t i_hi, const sb_storage* st, int to_storage, cudaStream_t s) {
    if (rows <= 0 || i_hi <= i_lo) return SB_OK;
    sb::LayoutXfer<T> a;
    a.src = reinterpret_cast<const T*>(src);
    a.dst = reinterpret_cast<T*>(dst);
    a.rows = rows;
    a.nat_stride = nat_stride;
    a.sto_stride = sto_stride;
    a.nat0 = nat0;
    a.sto0 = sto0;
    a.i_lo = i_lo;
    a.i_hi = i_hi;
    a.unit_np = st->unit_np;
    a.layout = st->layout;
    a.vl = st->layout == SB_LAYOUT_NATURAL ? 1 : st->vl;
    a.sub = st->unit_np / a.vl;
    a.tiles = (st->unit_np + sb::LT_S - 1) / sb::LT_S;
    a.to_storage = to_storage;
    dim3 grid((unsigned)(a.tiles + 1), (unsigned)std::min<int64_t>(rows, 65535));
    sb::layout_xfer_kernel<T><<<grid, sb::LT_THREADS, 0, s>>>(a);
    SB_CUDA(cudaGetLastError());
    return SB_OK;
}

int xfer(int dtype, const void* src, void* dst, int64_t rows, int64_t nat_stride, int64_t sto_stride, int64_t nat0,
         int64_t sto0, int64_t i_lo, int64_t i_hi, const sb_storage* st, int to_storage, cudaStream_t s) {
    if (dtype == SB_F64)
        return launch_xfer<double>(src, dst, rows, nat_stride, sto_stride, nat0, sto0, i_lo, i_hi, st, to_storage, s);
    return launch_xfer<float>(src, dst, rows, nat_stride, sto_stride, nat0, sto0, i_lo, i_hi, st, to_storage, s);
}

int check_plan_storage(sb_plan* P, const sb_storage* st, size_t bytes, int64_t* row_elems) {
    if (!P) return fail(SB_ERR_ARG, "NULL plan");
    int rc = check_storage(st, row_elems);
    if (rc != SB_OK) return rc;
    if (!(P->phys_lo && P->phys_hi)) return fail(SB_ERR_GRID, "reference storage needs a whole-grid plan (no ghost sides)");
    if (st->unit_n != P->dims[P->d - 1])
        return fail(SB_ERR_GRID, "storage unit extent %lld, plan has %lld", (long long)st->unit_n,
                    (long long)P->dims[P->d - 1]);
    if (st->halo_unit < P->r) return fail(SB_ERR_GRID, "unit halo %lld < order %d", (long long)st->halo_unit, P->r);
    const size_t want = (size_t)(P->host_rows * *row_elems) * P->es;
    if (bytes != want)
        return fail(SB_ERR_GRID, "storage has %zu bytes, expected %zu (%lld rows x %lld)", bytes, want,
                    (long long)P->host_rows, (long long)*row_elems);
    return SB_OK;
}

}  // namespace
}  // namespace sbh

using namespace sbh;

extern "C" {

int sb_upload_storage(sb_plan* P, const void* host, size_t bytes, const sb_storage* st) {
    int64_t row_elems = 0;
    int rc = check_plan_storage(P, st, bytes, &row_elems);
    if (rc != SB_OK) return rc;
    if (!host) return fail(SB_ERR_ARG, "NULL host storage");
    SB_CUDA(cudaSetDevice(P->device));
    if (P->stage_bytes < bytes) {
        if (P->stage) SB_CUDA(cudaFree(P->stage));
        P->stage = nullptr;
        P->stage_bytes = 0;
        cudaError_t e = cudaMalloc(&P->stage, bytes);
        if (e != cudaSuccess) return fail(e == cudaErrorMemoryAllocation ? SB_ERR_NOMEM : SB_ERR_CUDA,
                                          "staging allocation failed: %s", cudaGetErrorString(e));
        P->stage_bytes = bytes;
    }
    P->stage_row_elems = row_elems;
    SB_CUDA(cudaMemcpyAsync(P->stage, host, bytes, cudaMemcpyHostToDevice, P->stream));
    // every storage row (outer halo rows included) -> the plan's natural row,
    // natural indices [-r, unit_n + r) (storage_col, core.py:290-297)
    char* nat = reinterpret_cast<char*>(P->buf[0]);
    rc = xfer(P->dtype, P->stage, nat, P->host_rows, P->px, row_elems, P->host_dst_offset + P->r, st->halo_unit,
              -P->r, st->unit_n + P->r, st, 0, P->stream);
    if (rc != SB_OK) return rc;
    P->kernels_launched++;
    rc = finish_upload(P);
    if (rc != SB_OK) return rc;
    SB_CUDA(cudaStreamSynchronize(P->stream));
    return SB_OK;
}

int sb_download_storage(sb_plan* P, void* host, size_t bytes, const sb_storage* st) {
    int64_t row_elems = 0;
    int rc = check_plan_storage(P, st, bytes, &row_elems);
    if (rc != SB_OK) return rc;
    if (!host) return fail(SB_ERR_ARG, "NULL host storage");
    if (!P->uploaded) return fail(SB_ERR_STATE, "download before upload");
    if (!P->stage || P->stage_row_elems != row_elems || P->stage_bytes < bytes)
        return fail(SB_ERR_STATE, "download_storage needs a prior upload_storage of the same geometry");
    SB_CUDA(cudaSetDevice(P->device));
    rc = xfer(P->dtype, P->buf[P->cur], P->stage, P->host_rows, P->px, row_elems, P->host_dst_offset + P->r,
              st->halo_unit, -P->r, st->unit_n + P->r, st, 1, P->stream);
    if (rc != SB_OK) return rc;
    P->kernels_launched++;
    SB_CUDA(cudaMemcpyAsync(host, P->stage, bytes, cudaMemcpyDeviceToHost, P->stream));
    SB_CUDA(cudaStreamSynchronize(P->stream));
    return SB_OK;
}

int sb_layout_convert(void* dst, const void* src, int64_t rows, const sb_storage* st, int32_t to_layout,
                      int32_t dtype, void* stream) {
    int64_t row_elems = 0;
    int rc = check_storage(st, &row_elems);
    if (rc != SB_OK) return rc;
    if (!dst || !src) return fail(SB_ERR_ARG, "NULL buffer");
    if (dst == src) return fail(SB_ERR_ARG, "layout conversion is out-of-place: dst and src must differ");
    if (dtype != SB_F64 && dtype != SB_F32) return fail(SB_ERR_ARG, "unknown dtype %d", dtype);
    if (rows < 0) return fail(SB_ERR_ARG, "rows must be >= 0");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    // every cell of every row: halo cells are the identity, the padded region permuted
    rc = xfer(dtype, src, dst, rows, row_elems, row_elems, st->halo_unit, st->halo_unit, -st->halo_unit,
              st->unit_np + st->halo_unit, st, to_layout ? 1 : 0, s);
    return rc;
}

}  // extern "C"
