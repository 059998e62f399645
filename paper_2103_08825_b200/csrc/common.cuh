// Shared device-side definitions for the sb200 stencil kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sb {

// One stencil term accumulation in the two arithmetic modes of sb_arith.
// EXACT restates stencilbench/kernels.py:103-108: acc starts at +0.0 and
// every term is one rounded multiply followed by one rounded add (the
// intrinsics stop nvcc from contracting them into an FMA).
template <typename T> struct Arith;

template <> struct Arith<double> {
    static __device__ __forceinline__ double first(double w, double x, bool fma_mode) {
        return fma_mode ? __dmul_rn(w, x) : __dadd_rn(0.0, __dmul_rn(w, x));
    }
    static __device__ __forceinline__ double term(double acc, double w, double x, bool fma_mode) {
        return fma_mode ? __fma_rn(w, x, acc) : __dadd_rn(acc, __dmul_rn(w, x));
    }
};

template <> struct Arith<float> {
    static __device__ __forceinline__ float first(float w, float x, bool fma_mode) {
        return fma_mode ? __fmul_rn(w, x) : __fadd_rn(0.0f, __fmul_rn(w, x));
    }
    static __device__ __forceinline__ float term(float acc, float w, float x, bool fma_mode) {
        return fma_mode ? __fmaf_rn(w, x, acc) : __fadd_rn(acc, __fmul_rn(w, x));
    }
};

template <typename T, bool FMA>
__device__ __forceinline__ T acc_first(T w, T x) { return Arith<T>::first(w, x, FMA); }
template <typename T, bool FMA>
__device__ __forceinline__ T acc_term(T acc, T w, T x) { return Arith<T>::term(acc, w, x, FMA); }

// Device storage geometry, canonicalised to 3 axes (z, y, x) with x the unit
// stride.  Lower-dimensional problems have leading extents of 1.  `origin`
// is the element offset of interior point (0,0,0) in each buffer.
struct Geom {
    int64_t n[3];        // interior extents (z, y, x)
    int64_t sz, sy;      // element strides of z and y (x stride is 1)
    int64_t origin;      // element offset of interior (0,0,0)
    int slab_axis;       // canonical axis carrying the slab/ghost split (3-d)
};

}  // namespace sb
