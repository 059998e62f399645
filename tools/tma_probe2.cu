// TMA probe (development tool): may a 2D/3D tensor-map box start at an
// innermost coordinate that is not 16 B aligned?  fp32 tensor, box 72 x 4,
// start x in {4, 5, 6, 7}: prints whether the load completes and is correct.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tmap, int x, int y, unsigned bytes, float* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(su32(sm)), "l"(&tmap), "r"(x), "r"(y), "r"(0), "r"(su32(&bar)) : "memory");
    }
    __syncthreads();
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(su32(&bar)) : "memory");
    for (int i = threadIdx.x; i < (int)(bytes / 4); i += blockDim.x) out[i] = ((float*)sm)[i];
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int px = 256, rows = 16, planes = 2;
    float* buf;
    cudaMalloc(&buf, px * rows * planes * 4);
    float* h = new float[px * rows * planes];
    for (int i = 0; i < px * rows * planes; i++) h[i] = (float)i;
    cudaMemcpy(buf, h, px * rows * planes * 4, cudaMemcpyHostToDevice);
    void* fn;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap m;
    cuuint64_t dims[3] = {px, rows, planes};
    cuuint64_t str[2] = {px * 4, (cuuint64_t)px * rows * 4};
    cuuint32_t box[3] = {72, 4, 1}, es[3] = {1, 1, 1};
    CUresult r = ((Enc)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode=%d\n", (int)r);
    float* out;
    cudaMalloc(&out, 72 * 4 * 4);
    float res[72 * 4];
    for (int x = 4; x < 8; x++) {
        cudaMemset(out, 0, 72 * 4 * 4);
        probe<<<1, 128, 72 * 4 * 4 + 1024>>>(m, x, 2, 72 * 4 * 4, out);
        cudaError_t e = cudaDeviceSynchronize();
        int bad = -1;
        if (e == cudaSuccess) {
            cudaMemcpy(res, out, sizeof(res), cudaMemcpyDeviceToHost);
            bad = 0;
            for (int yy = 0; yy < 4; yy++)
                for (int xx = 0; xx < 72; xx++)
                    if (res[yy * 72 + xx] != h[(2 + yy) * px + x + xx]) bad++;
        }
        printf("x=%d kernel=%s mismatches=%d\n", x, cudaGetErrorString(e), bad);
        if (e != cudaSuccess) break;
    }
    return 0;
}
