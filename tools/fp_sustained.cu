// Sustained FP64 FMA rate and SM clock under a long DFMA load (development
// tool): back-to-back launches for ~6 s, CUDA-event rate per second of load.
// The burst peak (tools/fp_peak.cu, profiles/fp_peak.json) is measured at the
// maximum SM clock; a sustained DFMA load can hit the board power cap.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS, int ITERS>
__global__ void dfma_loop(double* out, double a, double b) {
    double acc[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; c++) acc[c] = (double)(threadIdx.x + c);
    for (int i = 0; i < ITERS; i++) {
#pragma unroll
        for (int c = 0; c < CHAINS; c++) acc[c] = fma(acc[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; c++) s += acc[c];
    if (s == -12345.0) out[threadIdx.x] = s;
}

int main() {
    double* d;
    cudaMalloc(&d, 1 << 20);
    constexpr int CH = 8, IT = 1 << 14;
    const int blocks = 148 * 4, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int sec = 0; sec < 6; sec++) {
        int n = 0;
        cudaEventRecord(e0);
        float ms = 0;
        while (ms < 1000.f) {
            for (int i = 0; i < 20; i++) dfma_loop<CH, IT><<<blocks, threads>>>(d, 0.999999, 1e-9);
            n += 20;
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        const double flops = 2.0 * CH * IT * (double)blocks * threads * n;
        printf("second %d: %.2f TFLOP/s fp64\n", sec, flops / (ms * 1e-3) / 1e12);
        fflush(stdout);
    }
    return 0;
}
