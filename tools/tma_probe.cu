// Standalone TMA probe: 3D tensor-map box loads under different coordinate /
// size regimes (debug aid for the fused 3D kernel).  ./tma_probe <case>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tmap, int x, int y, int z, unsigned bytes, double* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(su32(sm)), "l"(&tmap), "r"(x), "r"(y), "r"(z), "r"(su32(&bar)) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(su32(&bar)) : "memory");
    double s = 0;
    for (int i = threadIdx.x; i < (int)(bytes / 8); i += blockDim.x) s += ((double*)sm)[i];
    atomicAdd(out, s);
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    int c = argc > 1 ? atoi(argv[1]) : 0;
    // tensor: px x rows x planes doubles
    cuuint64_t px = 48, rows = 7, planes = 5;
    cuuint32_t bx = 68, by = 34;
    int x = 16, y = 0, z = 0;
    if (c == 1) { px = 128; rows = 64; planes = 8; bx = 68; by = 34; x = 8; y = 4; z = 2; }   // in bounds
    if (c == 2) { px = 128; rows = 64; planes = 8; bx = 68; by = 34; x = 8; y = -3; z = -1; } // negative coords
    if (c == 3) { px = 48; rows = 7; planes = 5; bx = 68; by = 34; x = 16; y = 0; z = 0; }    // box > tensor
    if (c == 4) { px = 128; rows = 64; planes = 8; bx = 68; by = 34; x = 100; y = 50; z = 7; }// past the end
    double* buf;
    cudaMalloc(&buf, px * rows * planes * 8);
    cudaMemset(buf, 0, px * rows * planes * 8);
    void* fn;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap m;
    cuuint64_t dims[3] = {px, rows, planes};
    cuuint64_t str[2] = {px * 8, px * rows * 8};
    cuuint32_t box[3] = {bx, by, 1}, es[3] = {1, 1, 1};
    CUresult r = ((Enc)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    double* out;
    cudaMalloc(&out, 8);
    cudaMemset(out, 0, 8);
    unsigned bytes = bx * by * 8;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes + 1024);
    probe<<<1, 128, bytes + 1024>>>(m, x, y, z, bytes, out);
    cudaError_t e = cudaDeviceSynchronize();
    printf("case %d encode=%d kernel=%s\n", c, (int)r, cudaGetErrorString(e));
    return 0;
}
