// Microbenchmark (development tool): FFMA2 (fma.rn.f32x2) dependent latency and
// per-SMSP throughput vs independent chains and warps, weights from the constant bank.
#include <cstdio>
#include <cuda_runtime.h>

template <int NCH>
__global__ void ffma2_chains(float* out, int iters, unsigned long long w) {
    unsigned long long a[NCH];
#pragma unroll
    for (int c = 0; c < NCH; c++) a[c] = (unsigned long long)(threadIdx.x + c) * 0x3f8000003f800000ull;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int c = 0; c < NCH; c++) asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(a[c]) : "l"(w));
    }
    long long t1 = clock64();
    unsigned long long s = 0;
#pragma unroll
    for (int c = 0; c < NCH; c++) s ^= a[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(s & 1);
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}

template <int NCH>
void run(int warps, float* d) {
    const int iters = 4096;
    const unsigned long long w = 0x3f7ff0003f7ff000ull;
    ffma2_chains<NCH><<<148, 32 * warps>>>(d, iters, w);
    cudaDeviceSynchronize();
    ffma2_chains<NCH><<<148, 32 * warps>>>(d, iters, w);
    float cyc;
    cudaMemcpy(&cyc, d, 4, cudaMemcpyDeviceToHost);
    const double per_instr = cyc / ((double)iters * NCH);
    printf("chains %2d warps/SM %2d: %.2f cyc per dependent step, SMSP FFMA2 rate %.3f /cyc (FMA lanes/cyc/SMSP %.1f)\n",
           NCH, warps, cyc / iters, warps / 4.0 / per_instr, 64.0 * warps / 4.0 / per_instr);
}

int main() {
    float* d;
    cudaMalloc(&d, 148 * 1024 * 4);
    for (int w : {4, 8, 16}) {
        run<1>(w, d); run<2>(w, d); run<4>(w, d); run<8>(w, d);
    }
    return 0;
}
