// Sustained FP64 FMA rate and SM clock under a long DFMA load (development
// tool): back-to-back launches for ~6 s per mode, CUDA-event rate per second.
// The burst peak (tools/fp_peak.cu, profiles/fp_peak.json) is measured at the
// maximum SM clock; a sustained DFMA load can hit the board power cap, and how
// soon depends on the OPERANDS: mode "const" iterates acc = fma(acc, a, b)
// towards its fixed point (operands stop changing: little switching in the
// multiplier array), mode "data" accumulates w[j] * x[i] over register-resident
// random inputs with weights of alternating sign (what a stencil sweep feeds
// the pipe: every multiply sees a new random mantissa), mode "chaos" runs the
// quadratic map acc = fma(acc, acc, c) (both multiplicands change every op).
// Usage: fp_sustained [seconds per mode]; prints TFLOP/s per second of load
// (sample nvidia-smi beside it for clocks and power).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int CHAINS, int ITERS>
__global__ void dfma_const(double* out, double a, double b) {
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

__device__ __forceinline__ double rnd01(unsigned long long& st) {
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    return (double)(st >> 11) * (1.0 / 9007199254740992.0);
}

// acc[c] += w[j] * x[(c + j) % NX]: NX random inputs in registers, 4 weights
// (+, -, +, -: the sums stay bounded), CHAINS independent accumulators
template <int CHAINS, int ITERS>
__global__ void dfma_data(double* out, double w0, double w1, double w2, double w3) {
    constexpr int NX = 8;
    double x[NX], acc[CHAINS];
    unsigned long long st = 0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1);
#pragma unroll
    for (int i = 0; i < NX; i++) x[i] = rnd01(st);
#pragma unroll
    for (int c = 0; c < CHAINS; c++) acc[c] = rnd01(st);
    for (int i = 0; i < ITERS; i += 4) {
#pragma unroll
        for (int c = 0; c < CHAINS; c++) acc[c] = fma(w0, x[c % NX], acc[c]);
#pragma unroll
        for (int c = 0; c < CHAINS; c++) acc[c] = fma(w1, x[(c + 1) % NX], acc[c]);
#pragma unroll
        for (int c = 0; c < CHAINS; c++) acc[c] = fma(w2, x[(c + 2) % NX], acc[c]);
#pragma unroll
        for (int c = 0; c < CHAINS; c++) acc[c] = fma(w3, x[(c + 3) % NX], acc[c]);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; c++) s += acc[c];
    if (s == -12345.0) out[threadIdx.x] = s;
}

template <int CHAINS, int ITERS>
__global__ void dfma_chaos(double* out, double cc) {
    double acc[CHAINS];
    unsigned long long st = 0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1);
#pragma unroll
    for (int c = 0; c < CHAINS; c++) acc[c] = rnd01(st);
    for (int i = 0; i < ITERS; i++) {
#pragma unroll
        for (int c = 0; c < CHAINS; c++) acc[c] = fma(acc[c], acc[c], cc);   // x^2 + c, c = -1.9: chaotic on [-2, 2]
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; c++) s += acc[c];
    if (s == -12345.0) out[threadIdx.x] = s;
}

int main(int argc, char** argv) {
    const int seconds = argc > 1 ? atoi(argv[1]) : 6;
    double* d;
    cudaMalloc(&d, 1 << 20);
    constexpr int CH = 8, IT = 1 << 14;
    const int blocks = 148 * 4, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[3] = {"const", "data", "chaos"};
    for (int mode = 0; mode < 3; mode++) {
        for (int sec = 0; sec < seconds; sec++) {
            int n = 0;
            cudaEventRecord(e0);
            float ms = 0;
            while (ms < 1000.f) {
                for (int i = 0; i < 20; i++) {
                    if (mode == 0) dfma_const<CH, IT><<<blocks, threads>>>(d, 0.999999, 1e-9);
                    else if (mode == 1) dfma_data<CH, IT><<<blocks, threads>>>(d, 0.37, -0.41, 0.29, -0.25);
                    else dfma_chaos<CH, IT><<<blocks, threads>>>(d, -1.9);
                }
                n += 20;
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
            }
            const double flops = 2.0 * CH * IT * (double)blocks * threads * n;
            printf("mode %s second %d: %.2f TFLOP/s fp64\n", names[mode], sec, flops / (ms * 1e-3) / 1e12);
            fflush(stdout);
        }
    }
    return 0;
}
