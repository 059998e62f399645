// Measures the FP64 / FP32 vector-pipe peak of this GPU (FMA throughput),
// the denominator of the stencil roofline's compute side (MEASURED_PEAKS.json
// has HBM and bf16 only).  Prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp_peak fp_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int CHAINS, int ITERS>
__global__ void fma_loop(T* out, T a, T b) {
    T acc[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; c++) acc[c] = (T)(threadIdx.x + c);
    for (int i = 0; i < ITERS; i++) {
#pragma unroll
        for (int c = 0; c < CHAINS; c++) acc[c] = fma(acc[c], a, b);
    }
    T s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; c++) s += acc[c];
    if (s == (T)-12345.0) out[threadIdx.x] = s;  // keep the chain alive
}

// Packed fp32 (FFMA2, fma.rn.f32x2, sm_100+): two FMAs per lane per instruction.
template <int CHAINS, int ITERS>
__global__ void ffma2_loop(float* out, float a, float b) {
    unsigned long long acc[CHAINS];
    const float2 av = make_float2(a, a), bv = make_float2(b, b);
    const unsigned long long A = *reinterpret_cast<const unsigned long long*>(&av);
    const unsigned long long B = *reinterpret_cast<const unsigned long long*>(&bv);
#pragma unroll
    for (int c = 0; c < CHAINS; c++) {
        const float2 x = make_float2((float)(threadIdx.x + c), (float)c);
        acc[c] = *reinterpret_cast<const unsigned long long*>(&x);
    }
    for (int i = 0; i < ITERS; i++) {
#pragma unroll
        for (int c = 0; c < CHAINS; c++) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[c]) : "l"(A), "l"(B));
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; c++) {
        const float2 x = *reinterpret_cast<const float2*>(&acc[c]);
        s += x.x + x.y;
    }
    if (s == -12345.0f) out[threadIdx.x] = s;
}

double measure_ffma2(int blocks_per_sm, int threads) {
    constexpr int CHAINS = 8, ITERS = 1 << 14;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, 4096 * sizeof(float));
    dim3 grid(sms * blocks_per_sm);
    ffma2_loop<CHAINS, ITERS><<<grid, threads>>>(out, 0.999999f, 1e-7f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(e0);
        ffma2_loop<CHAINS, ITERS><<<grid, threads>>>(out, 0.999999f, 1e-7f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFree(out);
    const double fmas = 2.0 * (double)grid.x * threads * CHAINS * (double)ITERS;
    return 2.0 * fmas / (best * 1e-3) / 1e12;
}

template <typename T>
double measure(int blocks_per_sm, int threads) {
    constexpr int CHAINS = 8, ITERS = 1 << 14;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    T* out;
    cudaMalloc(&out, 4096 * sizeof(T));
    dim3 grid(sms * blocks_per_sm);
    fma_loop<T, CHAINS, ITERS><<<grid, threads>>>(out, (T)0.999999, (T)1e-7);  // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(e0);
        fma_loop<T, CHAINS, ITERS><<<grid, threads>>>(out, (T)0.999999, (T)1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFree(out);
    const double fmas = (double)grid.x * threads * CHAINS * (double)ITERS;
    return 2.0 * fmas / (best * 1e-3) / 1e12;  // TFLOP/s (FMA = 2 flops)
}

int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    const double f64 = measure<double>(8, 256);
    const double f32 = measure<float>(8, 256);
    const double f32x2 = measure_ffma2(8, 256);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"fp64_tflops\": %.3f, \"fp32_tflops\": %.3f, \"fp32x2_tflops\": %.3f, "
           "\"clock_khz_attr\": %d, \"how\": \"dependent-chain FMA loops, 8 chains x 2^14 iters, "
           "8 CTAs x 256 threads per SM, best of 5, CUDA events; fp32x2 = packed FFMA2\"}\n",
           prop.name, prop.multiProcessorCount, f64, f32, f32x2, clk);
    return 0;
}
