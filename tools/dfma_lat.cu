// Microbenchmark (development tool): DFMA / FFMA2 latency and per-warp
// throughput vs independent chains, one CTA per SM, W warps per CTA.
#include <cstdio>
#include <cuda_runtime.h>

template <int NCH>
__global__ void dfma_chains(double* out, int iters, double w) {
    double a[NCH];
#pragma unroll
    for (int c = 0; c < NCH; c++) a[c] = threadIdx.x * 1e-3 + c;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int c = 0; c < NCH; c++) a[c] = fma(a[c], w, 0.5);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < NCH; c++) s += a[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(t1 - t0);
}

template <int NCH>
void run(int warps, double* d) {
    const int iters = 4096;
    dfma_chains<NCH><<<148, 32 * warps>>>(d, iters, 0.999);
    cudaDeviceSynchronize();
    dfma_chains<NCH><<<148, 32 * warps>>>(d, iters, 0.999);
    double cyc;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    const double per_warp = cyc / ((double)iters * NCH);          // cycles per DFMA per warp
    const double smsp_rate = (double)warps / 4.0 / per_warp;      // DFMA warp-instr per cycle per SMSP
    printf("chains %2d warps/SM %2d: %.2f cyc per dependent step, SMSP DFMA rate %.3f /cyc (peak 0.5)\n", NCH,
           warps, cyc / iters, smsp_rate);
}

int main() {
    double* d;
    cudaMalloc(&d, 148 * 1024 * 8);
    for (int w : {4, 8, 12, 16}) {
        run<1>(w, d); run<2>(w, d); run<4>(w, d); run<6>(w, d); run<8>(w, d);
    }
    return 0;
}
