// rn.cuh -- explicitly rounded arithmetic.
//
// The reference is built for x86-64 without -mfma, so every `s += a * b` in
// it rounds the product and the sum separately.  Kernels whose results are
// parity-checked bitwise (operator apply, residual, conversions) use these
// helpers so nvcc cannot contract them into FMAs.
#pragma once
#include <cuda_runtime.h>

namespace mpb {

__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }

}  // namespace mpb
